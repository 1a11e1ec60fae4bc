"""Thin ctypes binding of libsem_b200.so (include/sem.h).  Argument
marshalling only: every step of the hot path runs in the library's CUDA
kernels.  Device arrays are torch CUDA tensors (PyTorch is used for device
memory, streams and process groups only); host arrays are numpy arrays.

There is NO fallback: if the shared library is missing or fails to load,
importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libsem_b200.so")

SEM_OK, SEM_EINVAL, SEM_ENOMEM, SEM_ECUDA, SEM_ENCCL, SEM_EBREAKDOWN = range(6)
SEM_GS_ADD, SEM_GS_MASK = 0, 1
SEM_CG_STANDARD, SEM_CG_PIPELINED = 0, 1
SEM_PC_JACOBI, SEM_PC_HSMG = 0, 1
SEM_PRESSURE_CG, SEM_PRESSURE_GMRES = 0, 1

# every symbol declared in include/sem.h (checked by tests/test_abi.py)
EXPORTS = [
    "sem_version", "sem_last_error", "sem_gll", "sem_comm_unique_id", "sem_comm_create",
    "sem_comm_create_ex", "sem_comm_status", "sem_comm_destroy", "sem_options_default",
    "sem_mesh_set_options", "sem_mesh_get_options", "sem_mesh_create", "sem_mesh_destroy", "sem_mesh_info",
    "sem_mesh_global_ids", "sem_geom_factors", "sem_geom_get", "sem_mult_mask_get", "sem_ax",
    "sem_gs_op", "sem_ax_dssum", "sem_rhs", "sem_jacobi", "sem_cg_solve", "sem_gmres_solve", "sem_hsmg_apply", "sem_pnpn_step", "sem_cg_solve_host",
    "sem_profile_enable", "sem_profile_get", "sem_iface_candidates", "sem_iface_plan",
]


class SemError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


class MeshInfo(ctypes.Structure):
    _fields_ = [("E", ctypes.c_int64), ("N", ctypes.c_int), ("lx", ctypes.c_int),
                ("n_local", ctypes.c_int64), ("n_unique", ctypes.c_int64),
                ("n_entities", ctypes.c_int64), ("n_masked", ctypes.c_int64),
                ("n_interface", ctypes.c_int64), ("n_boundary_elements", ctypes.c_int64),
                ("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("n_peers", ctypes.c_int),
                ("affine", ctypes.c_int)]


class Options(ctypes.Structure):
    """sem_options_t (include/sem.h)."""
    _fields_ = [("cg_variant", ctypes.c_int), ("affine", ctypes.c_int), ("graph", ctypes.c_int),
                ("pdl", ctypes.c_int), ("gmres_precond", ctypes.c_int), ("hsmg_coarse_iters", ctypes.c_int),
                ("pnpn_pressure", ctypes.c_int), ("cg_layout", ctypes.c_int)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2405_05640_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    sig = {
        "sem_version": ([], ctypes.c_char_p),
        "sem_last_error": ([], ctypes.c_char_p),
        "sem_gll": ([i32, P, P], i32),
        "sem_comm_unique_id": ([P], i32),
        "sem_comm_create": ([P, i32, i32, i32, P], i32),
        "sem_comm_create_ex": ([P, i32, i32, i32, i32, P], i32),
        "sem_comm_status": ([P, P], i32),
        "sem_options_default": ([P], None),
        "sem_mesh_set_options": ([P, P], i32),
        "sem_mesh_get_options": ([P, P], i32),
        "sem_comm_destroy": ([P], None),
        "sem_mesh_create": ([i64, i32, P, P, P, P, P], i32),
        "sem_mesh_destroy": ([P], None),
        "sem_mesh_info": ([P, P], i32),
        "sem_mesh_global_ids": ([P, P], i32),
        "sem_geom_factors": ([P], i32),
        "sem_geom_get": ([P, P, P], i32),
        "sem_mult_mask_get": ([P, P, P], i32),
        "sem_ax": ([P, P, P, P, P, dbl, dbl, P], i32),
        "sem_gs_op": ([P, P, i32, P], i32),
        "sem_ax_dssum": ([P, P, P, P, P, dbl, dbl, P], i32),
        "sem_rhs": ([P, P, P, P], i32),
        "sem_jacobi": ([P, P, P, dbl, dbl, P, P], i32),
        "sem_cg_solve": ([P, P, P, P, P, dbl, dbl, dbl, i32, P, P, P, P], i32),
        "sem_cg_solve_host": ([P, P, P, P, P, dbl, dbl, dbl, i32, P, P, P, P], i32),
        "sem_gmres_solve": ([P, P, P, P, P, dbl, dbl, dbl, i32, i32, P, P, P, P], i32),
        "sem_hsmg_apply": ([P, P, P, dbl, dbl, P], i32),
        "sem_pnpn_step": ([P, P, P, dbl, dbl, dbl, i32, P, P], i32),
        "sem_profile_enable": ([P, i32], i32),
        "sem_profile_get": ([P, P, P, P], i32),
        "sem_iface_candidates": ([i64, i32, P, P, P], i32),
        "sem_iface_plan": ([i64, i32, P, i32, i32, P, P, P, P, P], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


lib = _load()


def _check(st, what=""):
    if st != SEM_OK:
        raise SemError(st, (lib.sem_last_error() or b"").decode() or what)


def _dptr(t):
    """Device pointer of a torch CUDA tensor (float64 contiguous) or None."""
    if t is None:
        return None
    if not t.is_cuda or t.dtype.itemsize != 8 or not t.is_contiguous():
        raise ValueError("expected a contiguous 8-byte CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def _hptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def sem_version():
    return lib.sem_version().decode()


def sem_gll(N: int):
    xi = np.zeros(N + 1)
    w = np.zeros(N + 1)
    _check(lib.sem_gll(N, _hptr(xi), _hptr(w)), "sem_gll")
    return xi, w


def sem_iface_candidates(N: int, conn):
    """Host-only: candidate interface keys [count][4] of a rank's elements."""
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    E = conn.shape[0]
    cnt = ctypes.c_int64(0)
    _check(lib.sem_iface_candidates(E, N, _hptr(conn), ctypes.byref(cnt), None))
    keys = np.zeros((cnt.value, 4), dtype=np.int64)
    _check(lib.sem_iface_candidates(E, N, _hptr(conn), ctypes.byref(cnt), _hptr(keys)))
    return keys


def sem_iface_plan(N: int, conn, rank: int, nranks: int, counts, all_keys):
    """Host-only: (peer_nodes[nranks], n_iface_entities, n_iface_nodes)."""
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    all_keys = np.ascontiguousarray(all_keys, dtype=np.int64)
    peer = np.zeros(nranks, dtype=np.int64)
    ne, nn = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib.sem_iface_plan(conn.shape[0], N, _hptr(conn), rank, nranks, _hptr(counts),
                              _hptr(all_keys), _hptr(peer), ctypes.byref(ne), ctypes.byref(nn)))
    return peer, ne.value, nn.value


def sem_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.sem_comm_unique_id(buf), "sem_comm_unique_id")
    return buf.raw


class Comm:
    def __init__(self, uid: bytes, rank: int, nranks: int, device: int, p2p: bool = True):
        self.h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(uid, 128)
        _check(lib.sem_comm_create_ex(buf, rank, nranks, device, int(bool(p2p)), ctypes.byref(self.h)),
               "sem_comm_create_ex")
        self.rank, self.nranks, self.device = rank, nranks, device

    def status(self):
        """(ok, p2p in use): raises SemError(SEM_ENCCL) once a peer wait timed out."""
        p2p = ctypes.c_int(0)
        _check(lib.sem_comm_status(self.h, ctypes.byref(p2p)), "sem_comm_status")
        return True, bool(p2p.value)

    def close(self):
        if self.h:
            lib.sem_comm_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sem_comm_create(uid: bytes, rank: int, nranks: int, device: int, p2p: bool = True) -> Comm:
    return Comm(uid, rank, nranks, device, p2p)


def sem_options_default() -> Options:
    o = Options()
    lib.sem_options_default(ctypes.byref(o))
    return o


class Mesh:
    """Owns a sem_mesh_t.  Mirrors sem_mesh_create's arguments."""

    def __init__(self, E, N, coords, conn, bc=None, comm: Comm | None = None):
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        conn = np.ascontiguousarray(conn, dtype=np.int64)
        bcarr = None if bc is None else np.ascontiguousarray(bc, dtype=np.int8)
        self.h = ctypes.c_void_p()
        self.E, self.N, self.lx = int(E), int(N), int(N) + 1
        self.n3 = self.lx ** 3
        self.comm = comm
        _check(lib.sem_mesh_create(int(E), int(N), _hptr(coords), _hptr(conn), _hptr(bcarr),
                                   comm.h if comm is not None else None, ctypes.byref(self.h)),
               "sem_mesh_create")

    def close(self):
        if self.h:
            lib.sem_mesh_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- queries ------------------------------------------------------------
    def info(self) -> MeshInfo:
        inf = MeshInfo()
        _check(lib.sem_mesh_info(self.h, ctypes.byref(inf)))
        return inf

    def options(self) -> Options:
        o = Options()
        _check(lib.sem_mesh_get_options(self.h, ctypes.byref(o)))
        return o

    def set_options(self, opt: Options | None = None, **kw):
        """Set sem_options_t fields (cg_variant, affine, graph, pdl,
        gmres_precond, hsmg_coarse_iters, pnpn_pressure, cg_layout); unspecified fields keep their
        current values."""
        o = self.options() if opt is None else opt
        for k, v in kw.items():
            if k == "cg_variant" and isinstance(v, str):
                v = {"standard": SEM_CG_STANDARD, "pipelined": SEM_CG_PIPELINED}[v]
            if k == "gmres_precond" and isinstance(v, str):
                v = {"jacobi": SEM_PC_JACOBI, "hsmg": SEM_PC_HSMG}[v]
            if k == "pnpn_pressure" and isinstance(v, str):
                v = {"cg": SEM_PRESSURE_CG, "gmres": SEM_PRESSURE_GMRES}[v]
            setattr(o, k, int(v))
        _check(lib.sem_mesh_set_options(self.h, ctypes.byref(o)), "sem_mesh_set_options")
        return self

    def global_ids(self):
        ids = np.zeros((self.E, self.n3), dtype=np.int64)
        _check(lib.sem_mesh_global_ids(self.h, _hptr(ids)))
        return ids

    def geom_factors(self):
        _check(lib.sem_geom_factors(self.h), "sem_geom_factors")

    def geom_get(self):
        import torch
        G = torch.empty((self.E, 6, self.n3), dtype=torch.float64, device="cuda")
        B = torch.empty((self.E, self.n3), dtype=torch.float64, device="cuda")
        _check(lib.sem_geom_get(self.h, _dptr(G), _dptr(B)))
        return G, B

    def mult_mask(self):
        import torch
        mult = torch.empty((self.E, self.n3), dtype=torch.float64, device="cuda")
        mask = torch.empty((self.E, self.n3), dtype=torch.float64, device="cuda")
        _check(lib.sem_mult_mask_get(self.h, _dptr(mult), _dptr(mask)))
        return mult, mask

    # -- operators ---------------------------------------------------------------
    def ax(self, u, w, h1=None, h2=None, h1c=1.0, h2c=0.0, stream=None):
        _check(lib.sem_ax(self.h, _dptr(u), _dptr(w), _dptr(h1), _dptr(h2), float(h1c), float(h2c),
                          _stream(stream)))
        return w

    def gs_op(self, u, op=SEM_GS_ADD, stream=None):
        _check(lib.sem_gs_op(self.h, _dptr(u), int(op), _stream(stream)))
        return u

    def ax_dssum(self, u, w, h1=None, h2=None, h1c=1.0, h2c=0.0, stream=None):
        _check(lib.sem_ax_dssum(self.h, _dptr(u), _dptr(w), _dptr(h1), _dptr(h2), float(h1c),
                                float(h2c), _stream(stream)))
        return w

    def rhs(self, f, b, stream=None):
        _check(lib.sem_rhs(self.h, _dptr(f), _dptr(b), _stream(stream)))
        return b

    def jacobi(self, dinv, h1=None, h2=None, h1c=1.0, h2c=0.0, stream=None):
        _check(lib.sem_jacobi(self.h, _dptr(h1), _dptr(h2), float(h1c), float(h2c), _dptr(dinv),
                              _stream(stream)))
        return dinv

    def cg_solve(self, b, x, h1=None, h2=None, h1c=1.0, h2c=0.0, tol=1e-10, maxit=1000,
                 stream=None):
        it, conv = ctypes.c_int(0), ctypes.c_int(0)
        rr = ctypes.c_double(0.0)
        _check(lib.sem_cg_solve(self.h, _dptr(b), _dptr(x), _dptr(h1), _dptr(h2), float(h1c),
                                float(h2c), float(tol), int(maxit), ctypes.byref(it), ctypes.byref(rr),
                                ctypes.byref(conv), _stream(stream)))
        return it.value, rr.value, bool(conv.value)

    def gmres_solve(self, b, x, h1=None, h2=None, h1c=1.0, h2c=0.0, tol=1e-10, maxit=1000, restart=30,
                    stream=None):
        """Restarted right-preconditioned GMRES (sem_gmres_solve): (iters, rel_res, converged)."""
        it, conv = ctypes.c_int(0), ctypes.c_int(0)
        rr = ctypes.c_double(0.0)
        _check(lib.sem_gmres_solve(self.h, _dptr(b), _dptr(x), _dptr(h1), _dptr(h2), float(h1c), float(h2c),
                                   float(tol), int(maxit), int(restart), ctypes.byref(it), ctypes.byref(rr),
                                   ctypes.byref(conv), _stream(stream)))
        return it.value, rr.value, bool(conv.value)

    def hsmg_apply(self, r, z, h1c=1.0, h2c=0.0, stream=None):
        """One hybrid-Schwarz multigrid V-cycle z = M r (sem_hsmg_apply)."""
        _check(lib.sem_hsmg_apply(self.h, _dptr(r), _dptr(z), float(h1c), float(h2c), _stream(stream)),
               "sem_hsmg_apply")

    def pnpn_step(self, u, p, dt, nu, tol=1e-10, maxit=1000, stream=None):
        """One velocity-pressure splitting step (sem_pnpn_step); u [3][E][n3] is
        overwritten.  Returns the iteration counts (pressure, u, v, w)."""
        it = (ctypes.c_int * 4)()
        _check(lib.sem_pnpn_step(self.h, _dptr(u), _dptr(p), float(dt), float(nu), float(tol), int(maxit), it,
                                 _stream(stream)))
        return list(it)

    def cg_solve_host(self, b_host, x_host, h1=None, h2=None, h1c=1.0, h2c=0.0, tol=1e-10,
                      maxit=1000, stream=None):
        """b_host / x_host: host buffers (numpy arrays or pinned torch CPU tensors)."""
        it, conv = ctypes.c_int(0), ctypes.c_int(0)
        rr = ctypes.c_double(0.0)

        def hp(a):
            if hasattr(a, "data_ptr"):
                return ctypes.c_void_p(a.data_ptr())
            return _hptr(a)
        _check(lib.sem_cg_solve_host(self.h, hp(b_host), hp(x_host), _dptr(h1), _dptr(h2),
                                     float(h1c), float(h2c), float(tol), int(maxit),
                                     ctypes.byref(it), ctypes.byref(rr), ctypes.byref(conv),
                                     _stream(stream)))
        return it.value, rr.value, bool(conv.value)

    def profile_enable(self, on=True):
        _check(lib.sem_profile_enable(self.h, int(bool(on))))

    def profile_get(self):
        """(timed operator launches, their summed ms, total kernels launched)."""
        n = ctypes.c_int64(0)
        ms = ctypes.c_double(0.0)
        kl = ctypes.c_int64(0)
        _check(lib.sem_profile_get(self.h, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(kl)))
        return n.value, ms.value, kl.value
