"""compute-sanitizer over every kernel of the library (SURVEY 5 auxiliary
subsystems: race detection and memory checking): tests/sanitize_worker.py
under memcheck (out-of-bounds / misaligned accesses, leaks of device
allocations are not counted: torch's caching allocator), racecheck (shared
memory hazards), synccheck (illegal barrier use) and initcheck
(uninitialised global reads).  Each tool must report 0 errors.

Opt-in, ONE tool per process: set SEM_SANITIZE_TOOL=memcheck|racecheck|
synccheck|initcheck (the profiling recipe allows one compute-sanitizer tool
per GPU call: several tools back to back on one box have left the GPU
unusable).  On this build's GPU pool compute-sanitizer is closed (the
wrapper exits 86: "compute-sanitizer is closed on this pool"; log in
profiles/r2_sanitize_memcheck.log); the test then skips with that reason.
test_all_kernels_plain runs the same worker without the sanitizer on every
GPU run: every kernel on small meshes, SEM_OK and finite results."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for c in ("/usr/local/cuda/bin/compute-sanitizer", shutil.which("compute-sanitizer")):
        if c and os.path.exists(c):
            return c
    return None


@pytest.mark.timeout(1500)
def test_compute_sanitizer():
    tool = os.environ.get("SEM_SANITIZE_TOOL")
    if tool not in ("memcheck", "racecheck", "synccheck", "initcheck"):
        pytest.skip("opt-in: SEM_SANITIZE_TOOL=memcheck|racecheck|synccheck|initcheck (one tool per GPU call)")
    cs = _sanitizer()
    if cs is None:
        pytest.skip("compute-sanitizer not found")
    cmd = [cs, f"--tool={tool}", "--error-exitcode=97", "--print-limit=20", "--target-processes=all"]
    if tool == "initcheck":
        cmd += ["--track-unused-memory=no"]
    cmd += [sys.executable, os.path.join(ROOT, "tests", "sanitize_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1400, cwd=ROOT)
    tail = (r.stdout[-3000:] + "\n" + r.stderr[-3000:])
    print(tail)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"sanitize_{tool}.log"), "w") as f:
        f.write(r.stdout + "\n" + r.stderr)
    if r.returncode == 86 and "closed on this pool" in r.stdout + r.stderr:
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert r.returncode == 0, tail
    assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr, tail


@pytest.mark.timeout(600)
def test_all_kernels_plain():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "sanitize_worker.py")], capture_output=True,
                       text=True, timeout=500, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "sanitize worker ok" in r.stdout
