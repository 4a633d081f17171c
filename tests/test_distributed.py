"""Multi-process keep-best on CPU (gloo, world size 2): the sharded argmin with a
16-byte all-gather equals the single-process first strict minimum."""

from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as tmp

from paper_2312_04025_b200.distributed import combine_records, encode_record, shard_bounds


def test_shard_bounds_partition():
    for total in (0, 1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - lo for lo, h in spans) - min(h - lo for lo, h in spans) <= 1


def test_combine_is_first_strict_minimum():
    recs = np.concatenate([encode_record(5.0, 9), encode_record(3.0, 40), encode_record(3.0, 12),
                           encode_record(math.inf, -1)])
    assert combine_records(recs) == (3.0, 12)
    assert combine_records(encode_record(math.inf, -1)) == (math.inf, -1)
    # -0.0 never occurs (makespans are sums of non-negative times), +0.0 orders first
    assert combine_records(np.concatenate([encode_record(0.0, 5), encode_record(1e-300, 1)])) == (0.0, 5)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, arrays, rows, q):
    import torch.distributed as dist

    from oracle.oracle import OracleInstance
    from paper_2312_04025_b200.distributed import sharded_argmin

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = OracleInstance(*arrays)

    def evaluate(_inst, r):  # CPU stand-in for the GPU argmin (no GPU here)
        ms, st = orc.eval_batch(r)
        ok = np.where(st == 0)[0]
        if len(ok) == 0:
            return -1, math.inf
        i = int(ok[np.argmin(ms[ok])])
        return i, float(ms[i])

    q.put((rank, sharded_argmin(None, rows, rank, world, evaluate=evaluate)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_argmin_gloo(world, oracle_mod):
    rng = np.random.default_rng(3)
    n, K, m = 12, 3, 20
    cost = rng.uniform(0.5, 8.0, (n, K)).round(3)
    mem = rng.integers(1, 30, n)
    src = np.array([rng.integers(0, j) for j in range(1, n) for _ in range(2)][:m], dtype=np.int32)
    dst = np.array([j for j in range(1, n) for _ in range(2)][:m], dtype=np.int32)
    keep = np.unique(np.stack([src, dst], 1), axis=0)
    src, dst = keep[:, 0].astype(np.int32), keep[:, 1].astype(np.int32)
    pay = rng.integers(1_000_000, 30_000_000, len(src))
    cap = np.array([120, 150, 90])
    bw = rng.uniform(4e6, 4e7, (K, K))
    arrays = (cost, mem, src, dst, pay, cap, bw)
    rows = rng.integers(0, K, (501, n), dtype=np.uint8)
    ms, st = oracle_mod.OracleInstance(*arrays).eval_batch(rows)
    ok = np.where(st == 0)[0]
    want_row = int(ok[np.argmin(ms[ok])])
    want = (float(ms[want_row]), want_row)
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, arrays, rows, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == want for v in got.values()), (got, want)


def _ls_instance():
    rng = np.random.default_rng(11)
    n, K = 10, 3
    cost = rng.uniform(0.5, 8.0, (n, K)).round(3)
    mem = rng.integers(1, 30, n)
    src = np.array([j - 1 - (j % 3 == 0) for j in range(2, n)], dtype=np.int32)
    dst = np.array(list(range(2, n)), dtype=np.int32)
    src = np.concatenate([[0], src]).astype(np.int32)
    dst = np.concatenate([[1], dst]).astype(np.int32)
    pay = rng.integers(1_000_000, 30_000_000, len(src))
    cap = np.array([150, 150, 150])
    bw = rng.uniform(4e6, 4e7, (K, K))
    return (cost, mem, src, dst, pay, cap, bw)


def _ls_worker(rank, world, port, arrays, seeds, q):
    import torch.distributed as dist

    from oracle.oracle import OracleInstance, ls_chains
    from paper_2312_04025_b200.distributed import distributed_local_search

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = OracleInstance(*arrays)

    def search(_inst, s, n, base, moves, rs):  # CPU stand-in for the GPU chains
        row, ms, ch, _ = ls_chains(orc, s, n, base, moves, rs)
        return row, ms, ch

    row, ms = distributed_local_search(None, seeds, rounds=3, chains=24, moves=6, seed=5, rank=rank, world=world,
                                       search=search)
    q.put((rank, (row.tolist(), ms)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_distributed_local_search_is_world_size_independent(world, oracle_mod):
    """Per-round incumbent exchange (16 B all-gather + row broadcast): the result
    equals the single-rank run of the same global chains."""
    from oracle.oracle import OracleInstance, ls_chains

    arrays = _ls_instance()
    seeds = np.random.default_rng(2).integers(0, 3, (4, 10), dtype=np.uint8)
    orc = OracleInstance(*arrays)
    cur, best = seeds, math.inf
    for r in range(3):  # the same rounds without any process group
        row, ms, _, _ = ls_chains(orc, cur, 24, 0, 6, 5 + r)
        best = min(best, ms)
        cur = row.reshape(1, -1)
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ls_worker, args=(r, world, port, arrays, seeds, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v[1] == best for v in got.values()), (got, best)
    assert all(v == got[0] for v in got.values())


def test_local_search_rounds_without_a_process_group(oracle_mod):
    """world=1 without torch.distributed: the same rounds as the reference loop."""
    from oracle.oracle import OracleInstance, ls_chains
    from paper_2312_04025_b200.distributed import distributed_local_search

    arrays = _ls_instance()
    seeds = np.random.default_rng(2).integers(0, 3, (4, 10), dtype=np.uint8)
    orc = OracleInstance(*arrays)

    def search(_inst, s, n, base, moves, rs):
        row, ms, ch, _ = ls_chains(orc, s, n, base, moves, rs)
        return row, ms, ch

    row, ms = distributed_local_search(None, seeds, rounds=3, chains=24, moves=6, seed=5, rank=0, world=1,
                                       search=search)
    cur, best = seeds, math.inf
    for r in range(3):
        w_row, w_ms, _, _ = ls_chains(orc, cur, 24, 0, 6, 5 + r)
        best = min(best, w_ms)
        cur = w_row.reshape(1, -1)
    assert ms == best
    st, rms, *_ = orc.schedule(row)
    assert st == 0 and rms == ms
