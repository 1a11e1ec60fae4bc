"""Multi-GPU parity (P15): distributed Ax+dssum, gather-scatter
and PCG through the C ABI over NCCL vs the oracle on the global mesh.
Runs tests/mgpu_worker.py under torch.distributed.run on as many GPUs as the
case needs; skipped when the box has fewer GPUs."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("case,nproc", [("box2", 2), ("walled2", 2), ("box4", 4), ("box8", 8)])
def test_multi_gpu_parity(case, nproc):
    if _ngpu() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + nproc}", os.path.join(ROOT, "tests", "mgpu_worker.py"),
           case]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout[-4000:])
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
