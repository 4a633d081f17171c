"""Multi-GPU keep-best: shard placements across ranks, exchange 16-byte records.

Placement evaluation is embarrassingly parallel: rank r owns a
disjoint slice of the placement stream, evaluates it on its own GPU, and the
only collective is one all-gather of a 16-byte record per rank —
(makespan bits, global row index) — followed by a lexicographic minimum.  That
reproduces the reference's first-strict-minimum rule (``solver.py:277-279``)
exactly: the global minimum makespan, lowest global index on ties.  NCCL has no
argmin reduction; the all-gather of G records is latency-bound (~tens of us over
NVLink) and runs once per batch.

The same functions drive ``bench.py`` (NCCL) and tests/test_distributed.py
(gloo, world size 2, on CPU).
"""

from __future__ import annotations

import math

import numpy as np


def shard_bounds(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of ``total`` rows for ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def encode_record(best_ms: float, best_row: int) -> np.ndarray:
    """16-byte record: makespan as int64 bits (non-negative doubles order like
    their bits; +inf marks "no feasible row") and the global row (-1 = none)."""
    if best_row < 0 or not math.isfinite(best_ms):
        return np.array([np.float64(np.inf).view(np.int64), -1], dtype=np.int64)
    return np.array([np.float64(best_ms).view(np.int64), best_row], dtype=np.int64)


def combine_records(records) -> tuple[float, int]:
    """Lexicographic (makespan, row) minimum over gathered records."""
    best = None
    for bits_, row in np.asarray(records, dtype=np.int64).reshape(-1, 2):
        if row < 0:
            continue
        key = (int(bits_), int(row))
        if best is None or key < best:
            best = key
    if best is None:
        return math.inf, -1
    return float(np.int64(best[0]).view(np.float64)), best[1]


def _single(group) -> bool:
    """No process group formed: a single rank (the exchange is the identity)."""
    import torch.distributed as dist

    return not (dist.is_available() and dist.is_initialized())


def allgather_best(best_ms: float, best_row: int, group=None, device=None) -> tuple[float, int]:
    """All-gather every rank's local best (16 B each) and return the global best.
    Uses the default process group's backend (NCCL on GPUs, gloo on CPU); without
    a process group it is the identity (one rank)."""
    import torch
    import torch.distributed as dist

    if _single(group):
        return combine_records(encode_record(best_ms, best_row))

    rec = torch.from_numpy(encode_record(best_ms, best_row))
    if device is not None:
        rec = rec.to(device)
    world = dist.get_world_size(group)
    out = torch.empty(2 * world, dtype=torch.int64, device=rec.device)
    dist.all_gather_into_tensor(out, rec, group=group)
    return combine_records(out.cpu().numpy())


def sharded_argmin(inst, rows_global: np.ndarray, rank: int, world: int, evaluate=None, group=None, device=None):
    """Evaluate this rank's shard and return the global (makespan, row).

    ``evaluate(inst, rows) -> (row, makespan)`` defaults to the GPU
    :func:`paper_2312_04025_b200.argmin`; tests inject the CPU oracle."""
    lo, hi = shard_bounds(len(rows_global), rank, world)
    if evaluate is None:
        from .solver import argmin

        def evaluate(i, r):
            return argmin(i, r)

    local_row, local_ms = evaluate(inst, rows_global[lo:hi]) if hi > lo else (-1, math.inf)
    global_row = lo + local_row if local_row >= 0 else -1
    return allgather_best(local_ms, global_row, group=group, device=device)


def broadcast_row(row: np.ndarray, src: int, group=None, device=None) -> np.ndarray:
    """Broadcast the winning placement row (n_ops bytes) from its owner rank."""
    import torch
    import torch.distributed as dist

    if _single(group):
        return np.ascontiguousarray(row, dtype=np.uint8).copy()

    t = torch.from_numpy(np.ascontiguousarray(row, dtype=np.uint8).copy())
    if device is not None:
        t = t.to(device)
    dist.broadcast(t, src=src, group=group)
    return t.cpu().numpy()


def distributed_local_search(inst, seeds: np.ndarray, *, rounds: int, chains: int, moves: int, seed: int,
                             rank: int, world: int, group=None, device=None, search=None):
    """K5 across GPUs: ``rounds`` rounds of ``chains`` chains in
    total, sharded by contiguous global chain id.  Each round every rank runs its
    chains (global ids ``[lo, hi)``, so proposals depend only on the global id),
    the ranks all-gather a 16-byte ``(makespan bits, global chain)`` record, the
    owner of the lexicographic minimum broadcasts its row, and the next round
    starts every chain from that incumbent.  Results are independent of the world
    size; with ``world=1`` and no process group it is a single-GPU multi-round
    incumbent-improvement loop.  ``search(inst, seeds, chains, chain_base, moves, rng_seed) -> (row, ms,
    chain)`` defaults to the GPU :func:`paper_2312_04025_b200.local_search`; the
    CPU tests inject the oracle's restatement.  Returns ``(row, makespan)``."""
    if search is None:
        from .solver import local_search

        def search(i, s, n, base, mv, rs):
            row, ms, ch, _ = local_search(i, s, chains=n, moves=mv, seed=rs, chain_base=base)
            return row, ms, ch

    cur = np.ascontiguousarray(seeds, dtype=np.uint8)
    best_row, best_ms = None, math.inf
    for r in range(rounds):
        lo, hi = shard_bounds(chains, rank, world)
        if hi > lo:
            row, ms, ch = search(inst, cur, hi - lo, lo, moves, seed + r)
        else:
            row, ms, ch = np.zeros(cur.shape[1], np.uint8), math.inf, -1
        g_ms, g_ch = allgather_best(ms, ch if math.isfinite(ms) else -1, group=group, device=device)
        if g_ch < 0:
            break
        owner = next(k for k in range(world) if shard_bounds(chains, k, world)[0] <= g_ch < shard_bounds(chains, k, world)[1])
        win = broadcast_row(row if owner == rank else np.zeros(cur.shape[1], np.uint8), owner, group=group,
                            device=device)
        if g_ms <= best_ms:
            best_row, best_ms = win, g_ms
        cur = win.reshape(1, -1)
    return best_row, best_ms
