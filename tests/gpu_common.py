"""Shared set-up of GPU-vs-oracle parity cases.

Each side builds its OWN coordinates from its OWN GLL nodes (oracle.gll vs
the library's sem_gll) through the shared generator module semgen, and its
own numbering (oracle: lattice / geometric ids; library: topology from the
vertex connectivity).  Only seeded fields cross over.
"""
from __future__ import annotations

import numpy as np

import oracle
import semgen


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def to_np(t):
    return t.detach().cpu().numpy()


def to_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


class Case:
    """A mesh on both sides: oracle arrays + a library Mesh."""

    def __init__(self, kind, N, **kw):
        from paper_2405_05640_b200 import sem
        self.kind, self.N = kind, N
        self.lx = N + 1
        xo, _ = oracle.gll(N)
        xl, _ = sem.sem_gll(N)
        if kind == "box":
            nel = kw.get("nel", (3, 3, 3))
            per = kw.get("periodic", (True, True, True))
            deform = kw.get("deform", 0.0)
            lengths = kw.get("lengths", (2 * np.pi,) * 3)
            self.mo = semgen.box_mesh(nel, xo, periodic=per, deform=deform, lengths=lengths)
            self.ml = semgen.box_mesh(nel, xl, periodic=per, deform=deform, lengths=lengths)
            self.ids, self.nuniq = oracle.lattice_ids(nel, N, per)
        elif kind == "cyl":
            args = dict(nc=kw.get("nc", 2), nr=kw.get("nr", 1), nz=kw.get("nz", 3))
            self.mo = semgen.cylinder_mesh(xo, **args)
            self.ml = semgen.cylinder_mesh(xl, **args)
            self.ids, self.nuniq = oracle.geometric_ids(self.mo["coords"], tol=1e-9)
        else:
            raise ValueError(kind)
        self.E = self.mo["conn"].shape[0]
        self.ids = self.ids.reshape(self.E, -1)
        self.mesh = sem.Mesh(self.E, N, self.ml["coords"], self.ml["conn"], self.ml["bc"])
        self.mesh.geom_factors()
        self.Go, self.Bo = oracle.geom(N, self.mo["coords"])
        self.mask = oracle.mask_from_bc(N, self.mo["bc"], self.ids, self.nuniq).reshape(self.E, -1)
        self.mult = oracle.mult(self.ids, self.nuniq).reshape(self.E, -1)

    def field(self, seed):
        return semgen.random_field((self.E, self.lx ** 3), seed)
