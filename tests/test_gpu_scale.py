"""Evaluation parity at scale: the GPU against the CPU oracle (oracle/moirai_oracle.c,
itself pinned to the reference's goldens by tests/test_oracle.py) on the named
workloads, bit for bit, through the paths the small fixtures do not reach:

* C3 (GPT-3 96 layers, K=8, 48 GB caps): >= 4096 memory-FEASIBLE rows, so the
  memory prefilter, the row compaction and the off-chip group kernel all run on
  thousands of real schedules (97 % of random C3 rows are memory-infeasible);
* C2-K8 (the north-star config) and C4-PCIe: 4096 rows each, every launch shape;
* C5 10 000 and 20 000 ops at K=8: 256 rows each (wide ready sets, off-chip state).

Each checks statuses, makespan bits and the keep-best row (brute_force's first
strict minimum, solver.py:277-279).
"""

from __future__ import annotations

import numpy as np
import pytest
from conftest import bits

import paper_2312_04025_b200 as mp
from paper_2312_04025_b200 import workloads


def _check(inst, orc, rows, shapes=(dict(),)):
    want, wst = orc.eval_batch(rows, threads=16)
    feas = np.flatnonzero(wst == 0)
    want_best = int(feas[np.argmin(want[feas])]) if len(feas) else -1
    for shape in shapes:
        inst.tune(**shape)
        ms, st, _, _ = mp.evaluate_batch(inst, rows, with_detail=True)
        assert np.array_equal(st, wst), shape
        assert np.array_equal(bits(ms), bits(want)), shape
        best, bms = mp.argmin(inst, rows)
        assert best == want_best and (best < 0 or bms == want[best]), shape
    return len(feas)


@pytest.mark.gpu
def test_c3_thousands_of_feasible_rows(oracle_mod):
    w = workloads.c3()
    coarse = mp.gcof(w.raw, w.rules)
    with mp.Instance(coarse, w.cluster, mp.effective_bandwidth(w.cluster)) as inst:
        orc = oracle_mod.OracleInstance.from_instance(inst)
        rows = workloads.placements(w.seed, 1 << 20, inst.n_ops, inst.K)
        # the oracle's memory check is cheap: pick a prefix holding >= 4096 feasible rows
        _, wst = orc.eval_batch(rows[:200_000], threads=16)
        feas_idx = np.flatnonzero(wst == 0)
        assert len(feas_idx) >= 4096
        n = int(feas_idx[4095]) + 1
        sub = np.ascontiguousarray(rows[:n])
        got = _check(inst, orc, sub, shapes=(dict(), dict(group_lanes=16), dict(offchip=True, group_lanes=8)))
        assert got >= 4096
        # and the feasible rows alone (no prefilter rejections around them)
        _check(inst, orc, np.ascontiguousarray(rows[feas_idx[:4096]]))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c2k8", "c4pcie"])
def test_north_star_and_pcie_configs_4096_rows(oracle_mod, name):
    w = {"c2k8": lambda: workloads.c2(8), "c4pcie": lambda: workloads.c4("pcie")}[name]()
    coarse = mp.gcof(w.raw, w.rules)
    with mp.Instance(coarse, w.cluster, mp.effective_bandwidth(w.cluster)) as inst:
        orc = oracle_mod.OracleInstance.from_instance(inst)
        rows = workloads.placements(w.seed, 4096, inst.n_ops, inst.K)
        shapes = (dict(), dict(colo=False), dict(ready_cap=3), dict(tpp=False), dict(tpp_registers=True),
                  dict(group_lanes=8), dict(offchip=True, group_lanes=32, colo=False))
        assert _check(inst, orc, rows, shapes) == 4096


@pytest.mark.gpu
@pytest.mark.parametrize("n", [10_000, 20_000])
def test_c5_large_graphs_256_rows(oracle_mod, n):
    w = workloads.c5(n, 8)
    coarse = mp.gcof(w.raw, w.rules)
    with mp.Instance(coarse, w.cluster, mp.effective_bandwidth(w.cluster)) as inst:
        assert inst.n_ops > n // 2
        orc = oracle_mod.OracleInstance.from_instance(inst)
        rows = workloads.placements(w.seed, 256, inst.n_ops, inst.K)
        assert _check(inst, orc, rows) == 256


@pytest.mark.gpu
def test_streamed_host_batch_with_mostly_overflowing_rows():
    """A host batch large enough to be streamed into one kernel pass (>= 16 x SMs x 512 rows)
    whose ready sets mostly outgrow a forced two-slot capacity: the overflow list must hold
    more than one chunk's worth of rows, and the results equal those of small batches."""
    w = workloads.c1()
    coarse = mp.gcof(w.raw, w.rules)
    with mp.Instance(coarse, w.cluster, mp.effective_bandwidth(w.cluster)) as inst:
        inst.tune(ready_cap=2)
        n = 16 * 148 * 512 + 4096
        rows = workloads.placements(11, n, inst.n_ops, inst.K)
        ms, st, _, _ = mp.evaluate_batch(inst, rows, with_detail=True)
        step = 1 << 16
        for r0 in range(0, n, step):
            m2, s2, _, _ = mp.evaluate_batch(inst, rows[r0:r0 + step], with_detail=True)
            assert np.array_equal(s2, st[r0:r0 + step])
            assert np.array_equal(bits(m2), bits(ms[r0:r0 + step])), r0
