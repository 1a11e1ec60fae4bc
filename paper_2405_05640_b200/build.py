"""Build libsem_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2405_05640_b200.build [--force] [--verbose]

The library links torch's bundled NCCL (nvidia-nccl wheel, 2.28.x) so that a
process that also imports torch loads exactly one libnccl.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsem_b200.so")
# (source, extra flags, object name): the operator kernel is compiled once per
# order (ax_lx.cu, -DSEM_AX_LX=lx) so the orders build in parallel
SOURCES = [(f, [], f + ".o") for f in ["kernels.cu", "ax.cu", "ax_p.cu", "gmres.cu", "pnpn.cu", "hsmg.cu", "hsmg_setup.cpp", "api.cpp", "gsplan.cpp", "topo.cpp",
                                         "basis.cpp", "comm.cpp", "p2p.cu"]]
SOURCES += [("ax_lx.cu", [f"-DSEM_AX_LX={lx}"], f"ax_lx{lx}.o") for lx in range(12, 1, -1)]
HEADERS = ["internal.h", "device_common.cuh", "ax.cuh", "ax_kernel.cuh", "gmres.h", "hsmg.h", os.path.join("..", "..", "include", "sem.h"),
           "p2p.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_paths():
    try:
        import nvidia.nccl as nn  # torch's bundled NCCL
        base = list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    except Exception:
        pass
    return None, None


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    inc, libdir = _nccl_paths()
    deps = [os.path.join(CSRC, s) for s, _, _ in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS] + [__file__]
    if not force and not _stale(LIB, deps):
        return LIB
    objdir = os.path.join(PKG, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    nvcc = _nvcc()
    common = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3",
                     "-I", os.path.join(ROOT, "include")]
    if inc:
        common += ["-DSEM_WITH_NCCL", "-I", inc]
    common += os.environ.get("SEM_NVCC_EXTRA", "").split()  # developer experiments only

    def compile_one(entry):
        src, extra, oname = entry
        obj = os.path.join(objdir, oname)
        cmd = [nvcc, "-c", os.path.join(CSRC, src), "-o", obj] + common + extra
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd = [nvcc, "-x", "cu", "-c", os.path.join(CSRC, src), "-o", obj] + common + extra
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 8)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    link = [nvcc, "-shared", "-o", LIB + ".tmp"] + ARCH + objs + ["-lcudart"]
    if libdir:
        link += ["-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{libdir}"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{' '.join(link)}\n{r.stdout}\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
