"""CPU-side checks of the C-ABI boundary: the library loads, exports every
symbol include/sem.h declares, and rejects bad arguments before touching the
GPU.  No compute call is made here (those are the -m gpu parity tests)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sem.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sem_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def semmod():
    from paper_2405_05640_b200 import build
    build.build()
    from paper_2405_05640_b200 import sem
    return sem


def test_header_symbols_exported(semmod):
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(semmod.lib, name), f"{name} declared in include/sem.h but not exported"
    assert sorted(semmod.EXPORTS) == declared


def test_exports_are_c_symbols():
    # extern "C": no C++ mangling in the dynamic symbol table
    import subprocess
    from paper_2405_05640_b200 import build
    lib = build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    syms = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    for name in _declared():
        assert name in syms


def test_version_and_arch(semmod):
    assert "sm_100a" in semmod.sem_version()


def test_invalid_arguments_fail_cleanly(semmod):
    L = semmod.lib
    out = ctypes.c_void_p()
    coords = np.zeros((3, 1, 8))
    conn = np.arange(8, dtype=np.int64).reshape(1, 8)
    # N out of range -> EINVAL with a message, before any CUDA call
    st = L.sem_mesh_create(1, 0, coords.ctypes.data_as(ctypes.c_void_p),
                           conn.ctypes.data_as(ctypes.c_void_p), None, None, ctypes.byref(out))
    assert st == semmod.SEM_EINVAL and not out.value
    assert b"N must be" in L.sem_last_error()
    st = L.sem_mesh_create(-1, 3, None, None, None, None, ctypes.byref(out))
    assert st == semmod.SEM_EINVAL
    st = L.sem_mesh_create(1, 3, None, None, None, None, ctypes.byref(out))
    assert st == semmod.SEM_EINVAL
    assert L.sem_gs_op(None, None, 0, None) == semmod.SEM_EINVAL
    assert L.sem_cg_solve(None, None, None, None, None, 1.0, 0.0, 1e-8, 10, None, None, None,
                          None) == semmod.SEM_EINVAL
    assert L.sem_gll(0, None, None) == semmod.SEM_EINVAL


def test_no_cpu_fallback_without_library(tmp_path, monkeypatch):
    # the binding must fail loudly when the CUDA library is absent
    import importlib.util
    src = os.path.join(ROOT, "paper_2405_05640_b200", "sem.py")
    fake_pkg = tmp_path / "pkg"
    fake_pkg.mkdir()
    (fake_pkg / "sem.py").write_text(open(src).read())
    spec = importlib.util.spec_from_file_location("sem_nolib", str(fake_pkg / "sem.py"))
    mod = importlib.util.module_from_spec(spec)
    with pytest.raises(ImportError):
        spec.loader.exec_module(mod)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2405_05640_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, flags=re.M), f
                assert "sem_oracle" not in txt and "liboracle" not in txt, f
    # and the oracle never imports the product
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_2405_05640_b200\b", txt, flags=re.M), f
            assert "libsem_b200" not in txt and "#include" not in txt.replace("#include <", ""), f
