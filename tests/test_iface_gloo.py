"""Multi-rank host logic of the N>1 path on CPU (torch.distributed, gloo):
each rank generates its own element block, computes its interface candidate
keys through the C ABI (host-only entry points), all-gathers them with gloo
and builds the interface plan.  The number of interface nodes exchanged with
every peer must equal the number of unique global nodes the two blocks share
according to the oracle's independent lattice numbering (O6).

Pins: two slabs of a walled 4^3 mesh at N = 7 share
(4*7+1)^2 = 841 nodes; a 2x1x1 mesh on 2 ranks exchanges 64.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import semgen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, nel, N, periodic, grid, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_2405_05640_b200 import sem
        xi = np.linspace(-1.0, 1.0, N + 1)  # node placement is irrelevant to topology
        m = semgen.box_mesh(nel, xi, periodic=periodic, elems=semgen.box_partition(nel, grid, rank))
        keys = sem.sem_iface_candidates(N, m["conn"])
        gathered = [None] * ws
        dist.all_gather_object(gathered, keys)
        counts = np.array([len(k) for k in gathered], dtype=np.int64)
        all_keys = np.concatenate([k.reshape(-1, 4) for k in gathered]) if counts.sum() else np.zeros((0, 4))
        peer, ne, nn = sem.sem_iface_plan(N, m["conn"], rank, ws, counts, all_keys)
        out[rank] = (peer.tolist(), int(ne), int(nn))
    finally:
        dist.destroy_process_group()


def _expected(nel, N, periodic, grid):
    ids, _ = oracle.lattice_ids(nel, N, periodic)
    ws = grid[0] * grid[1] * grid[2]
    sets = []
    lat = {tuple(p): q for q, p in enumerate(semgen.box_partition(nel, (1, 1, 1), 0))}
    for r in range(ws):
        el = [lat[tuple(p)] for p in semgen.box_partition(nel, grid, r)]
        sets.append(set(np.unique(ids[el]).tolist()))
    exp = []
    for r in range(ws):
        peer = [len(sets[r] & sets[s]) if s != r else 0 for s in range(ws)]
        others = set().union(*[sets[s] for s in range(ws) if s != r]) if ws > 1 else set()
        exp.append((peer, len(sets[r] & others)))
    return exp


@pytest.mark.parametrize("nel,N,periodic,grid", [
    ((4, 4, 4), 7, (False, False, False), (2, 1, 1)),   # P15: 841
    ((2, 1, 1), 7, (False, False, False), (2, 1, 1)),   # 64
    ((6, 3, 3), 3, (True, True, True), (2, 1, 1)),      # periodic: both x faces shared
    ((6, 6, 6), 2, (True, True, True), (2, 2, 2)),      # every rank neighbours all 7 others
    ((6, 6, 3), 3, (True, False, True), (2, 2, 1)),
])
def test_interface_plan_matches_oracle(nel, N, periodic, grid):
    ws = grid[0] * grid[1] * grid[2]
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(ws, _free_port(), nel, N, periodic, grid, out), nprocs=ws, join=True)
    exp = _expected(nel, N, periodic, grid)
    for r in range(ws):
        peer, ne, nn = out[r]
        assert peer == exp[r][0], (r, peer, exp[r][0])
        assert nn == exp[r][1]
    if nel == (4, 4, 4):
        assert out[0][2] == 841 and out[0][0][1] == 841
    if nel == (2, 1, 1):
        assert out[0][2] == 64
