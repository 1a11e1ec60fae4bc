"""GPU velocity-pressure splitting step (sem_pnpn_step) vs
the oracle's O17 (tests/test_oracle_pnpn.py pins it to the exact 2D
Taylor-Green decay).  Both sides solve to tol 1e-12; bars: velocity and
pressure rel-L2 <= 1e-10 (the CG bar), iteration counts within +-1, and the
exact-solution property on the GPU itself."""
import numpy as np
import pytest

import oracle
import semgen
from gpu_common import Case, rel_l2, to_dev, to_np

pytestmark = pytest.mark.gpu


def _tgv(coords, three_d):
    x, y, z = coords
    cz = np.cos(z) if three_d else 1.0
    return np.stack([np.sin(x) * np.cos(y) * cz, -np.cos(x) * np.sin(y) * cz, 0.0 * z])


@pytest.mark.parametrize("kind", ["tgv2d", "tgv3d-deformed"])
def test_pnpn_step_matches_oracle(kind):
    three_d = kind != "tgv2d"
    deform = 0.15 if three_d else 0.0
    c = Case("box", 7, nel=(4, 4, 3), deform=deform)
    nu, dt = 0.05, 0.01
    ul = _tgv(c.ml["coords"], three_d).reshape(3, c.E, -1)
    uo = _tgv(c.mo["coords"], three_d).reshape(3, c.E, -1)
    MJ = oracle.metrics(c.N, c.mo["coords"])
    un_o, p_o, itp_o, itv_o = oracle.pnpn_step(c.N, c.Go, c.Bo, MJ, c.ids, uo, dt, nu, nuniq=c.nuniq, tol=1e-12)
    u = to_dev(ul)
    p = to_dev(np.zeros((c.E, c.lx ** 3)))
    its = c.mesh.pnpn_step(u, p, dt, nu, tol=1e-12, maxit=5000)
    assert abs(its[0] - itp_o) <= 1 and all(abs(a - b) <= 1 for a, b in zip(its[1:], itv_o)), (its, itp_o, itv_o)
    assert rel_l2(to_np(u), un_o) <= 1e-10
    assert rel_l2(to_np(p), p_o) <= 1e-10
    if not three_d:  # the exact solution decays by 1/(1 + 2 nu dt)
        assert rel_l2(to_np(u), ul / (1.0 + 2.0 * nu * dt)) <= 1e-6


def test_pnpn_contract():
    from paper_2405_05640_b200 import sem
    c = Case("box", 3, nel=(3, 3, 3), periodic=(True, False, True))
    u = to_dev(np.zeros((3, c.E, c.lx ** 3)))
    p = to_dev(np.zeros((c.E, c.lx ** 3)))
    with pytest.raises(sem.SemError) as ei:  # walls: out of scope
        c.mesh.pnpn_step(u, p, 0.01, 0.1)
    assert ei.value.status == sem.SEM_EINVAL
    c = Case("box", 3, nel=(3, 3, 3))
    u = to_dev(np.zeros((3, c.E, c.lx ** 3)))
    with pytest.raises(sem.SemError):
        c.mesh.pnpn_step(u, p, -1.0, 0.1)
    its = c.mesh.pnpn_step(u, p, 0.01, 0.1)  # u = 0 stays 0
    assert float(u.abs().max()) == 0.0 and its == [0, 0, 0, 0]


def test_pnpn_step_with_the_papers_pressure_solver():
    """GMRES + hybrid-Schwarz multigrid for the pressure, CG +
    Jacobi for the velocity (pnpn_pressure = gmres, gmres_precond = hsmg) vs
    the oracle's step with its FGMRES + V-cycle (oracle/hsmg.py)."""
    from oracle import hsmg as H
    c = Case("box", 7, nel=(4, 4, 3), deform=0.15)
    nu, dt = 0.05, 0.01
    ul = _tgv(c.ml["coords"], True).reshape(3, c.E, -1)
    uo = _tgv(c.mo["coords"], True).reshape(3, c.E, -1)
    levels = H.setup(c.N, c.mo["coords"], c.mo["bc"], lambda Nl, cl: oracle.lattice_ids((4, 4, 3), Nl, (True,) * 3))

    def psolve(rp):
        x, it, _, _ = H.fgmres(levels, rp, tol=1e-12, maxit=500, restart=30)
        return x, it

    MJ = oracle.metrics(c.N, c.mo["coords"])
    un_o, p_o, itp_o, itv_o = oracle.pnpn_step(c.N, c.Go, c.Bo, MJ, c.ids, uo, dt, nu, nuniq=c.nuniq, tol=1e-12,
                                               pressure_solve=psolve)
    c.mesh.set_options(pnpn_pressure="gmres", gmres_precond="hsmg")
    u = to_dev(ul)
    p = to_dev(np.zeros((c.E, c.lx ** 3)))
    its = c.mesh.pnpn_step(u, p, dt, nu, tol=1e-12, maxit=500)
    assert abs(its[0] - itp_o) <= 1 and all(abs(a - b) <= 1 for a, b in zip(its[1:], itv_o)), (its, itp_o, itv_o)
    assert its[0] < 40  # the multigrid-preconditioned pressure solve
    assert rel_l2(to_np(u), un_o) <= 1e-10
    assert rel_l2(to_np(p), p_o) <= 1e-10
