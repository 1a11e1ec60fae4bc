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


# (case, ranks, worker flags): the peer-memory path (default) and the NCCL
# fallback (--p2p 0), the single-reduction CG, GMRES, FGMRES with the
# hybrid-Schwarz multigrid (levels built across the ranks), repeated solves on
# one communicator, the natural layout of the CG operator output (option
# cg_layout = 0; the default x-planes-last layout runs in every other case)
CASES = [
    ("box2", 2, []), ("walled2", 2, []), ("walled2", 2, ["--p2p", "0"]), ("box2", 2, ["--p2p", "0", "--repeat", "2"]),
    ("box2", 2, ["--variant", "pipelined"]), ("walled2", 2, ["--variant", "pipelined", "--p2p", "0"]),
    ("box2", 2, ["--repeat", "4"]), ("walled2", 2, ["--solver", "gmres"]), ("box2", 2, ["--solver", "gmres"]),
    ("box4", 4, []), ("box4", 4, ["--p2p", "0"]), ("box4", 4, ["--variant", "pipelined", "--repeat", "3"]),
    ("box4", 4, ["--solver", "gmres", "--p2p", "0"]),
    ("walled2", 2, ["--solver", "hsmg"]), ("box2", 2, ["--solver", "hsmg", "--repeat", "2"]),
    ("box4", 4, ["--solver", "hsmg"]), ("box4", 4, ["--solver", "hsmg", "--p2p", "0"]),
    ("walled2", 2, ["--layout", "0"]), ("box4", 4, ["--layout", "0", "--p2p", "0"]),
    ("box8", 8, []),
]


@pytest.mark.parametrize("case,nproc,flags", CASES, ids=[f"{c}-{n}-{'_'.join(f) or 'default'}" for c, n, f in CASES])
def test_multi_gpu_parity(case, nproc, flags):
    if _ngpu() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + nproc}", os.path.join(ROOT, "tests", "mgpu_worker.py"),
           case] + flags
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout[-4000:])
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
