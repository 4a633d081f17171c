"""Multi-rank keep-best and local search through the REAL kernels.

* a world-1 NCCL process group around `sharded_argmin` and
  `distributed_local_search` (the collective path bench.py times under torchrun);
* two gloo ranks, both on cuda:0, each evaluating its shard with the GPU
  evaluator: the global answer equals the single-process first strict minimum
  (solver.py:277-279) and the multi-round local search is world-size independent.
"""

from __future__ import annotations

import math
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    import paper_2312_04025_b200 as mp
    from paper_2312_04025_b200 import workloads

    w = workloads.c2(4)
    coarse = mp.gcof(w.raw, w.rules)
    inst = mp.Instance(coarse, w.cluster, mp.effective_bandwidth(w.cluster))
    rows = workloads.placements(11, 50_000, inst.n_ops, inst.K)
    return inst, rows


LS = dict(rounds=3, chains=4096, moves=8, seed=5)


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from paper_2312_04025_b200.distributed import distributed_local_search, sharded_argmin

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst, rows = _problem()
        best = sharded_argmin(inst, rows, rank, world)
        row, ms = distributed_local_search(inst, rows[:8], rank=rank, world=world, **LS)
        q.put((rank, best, row.tobytes(), ms))
        inst.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_world1_real_kernels():
    import torch
    import torch.distributed as dist

    import paper_2312_04025_b200 as mp
    from paper_2312_04025_b200.distributed import distributed_local_search, sharded_argmin

    inst, rows = _problem()
    want = mp.argmin(inst, rows)
    want_ls = distributed_local_search(inst, rows[:8], rank=0, world=1, **LS)  # no process group
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        assert dist.get_backend() == "nccl"
        ms, row = sharded_argmin(inst, rows, 0, 1, device=torch.device("cuda", 0))
        assert (row, ms) == want
        ls_row, ls_ms = distributed_local_search(inst, rows[:8], rank=0, world=1, device=torch.device("cuda", 0),
                                                 **LS)
        assert ls_ms == want_ls[1] and np.array_equal(ls_row, want_ls[0])
    finally:
        dist.destroy_process_group()
        inst.close()


@pytest.mark.gpu
def test_two_gloo_ranks_real_kernels_on_one_gpu():
    import torch.multiprocessing as tmp

    import paper_2312_04025_b200 as mp
    from paper_2312_04025_b200.distributed import distributed_local_search

    inst, rows = _problem()
    want_row, want_ms = mp.argmin(inst, rows)
    want_ls = distributed_local_search(inst, rows[:8], rank=0, world=1, **LS)
    inst.close()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (b, row, ms)) for r, b, row, ms in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        best, row, ms = res[r]
        assert best == (want_ms, want_row)
        assert ms == want_ls[1] and row == want_ls[0].tobytes()
    assert math.isfinite(want_ms)
