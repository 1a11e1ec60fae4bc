"""Multi-GPU parity (P15): distributed Ax+dssum, gather-scatter
and PCG through the C ABI (NVLink peer memory or NCCL) vs the oracle on the global mesh.
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


@pytest.mark.parametrize("case,nproc,p2p", [("box2", 2, "1"), ("walled2", 2, "1"), ("box4", 4, "1"), ("box8", 8, "1"),
                                            ("walled2", 2, "0"), ("box4", 4, "0")])
def test_multi_gpu_parity(case, nproc, p2p):
    # p2p "1": exchange and CG allreduce over NVLink peer memory (default);
    # "0": NCCL send/recv and allreduce (SEM_P2P=0)
    if _ngpu() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + nproc}", os.path.join(ROOT, "tests", "mgpu_worker.py"),
           case]
    env = dict(os.environ, SEM_P2P=p2p)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    print(r.stdout[-4000:])
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
