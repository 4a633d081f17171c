"""The callers either side of the evaluator against the
reference's own outputs (tests/golden/aux.json, made by tests/golden/make_golden.py):

* greedy_place (baselines.py:27-86) — GPU warp kernel: same assignment, same
  schedule bits, same InfeasibleMemoryError;
* check_feasibility (simulator.py:179-264) — GPU audit: the same violations in
  the same order with the same messages, on clean and corrupted schedules;
* fuse (fusion.py:251-268) — host graph edit: same graph or the same error.
"""

from __future__ import annotations

import pytest
from conftest import F, cluster_from, golden, golden_node_tuple, graph_from, node_tuple

import paper_2312_04025_b200 as mp


def _sched_from(d):
    return mp.Schedule({int(k): v for k, v in d["assignment"].items()},
                       {int(k): F(v) for k, v in d["starts"].items()},
                       {int(k): F(v) for k, v in d["ends"].items()},
                       {int(k): (tuple(v) if v else None) for k, v in d["channels"].items()},
                       F(d["makespan"]))


def test_fuse_matches_reference():
    cases = golden("aux.json")["fuse"]
    n_ok = n_err = 0
    for case in cases:
        g = graph_from(case["graph"])
        ov = None
        if case["overrides"] is not None:
            ov = mp.CostOverrides({(tuple(s), k): F(t) for s, k, t in case["overrides"]})
        if "error" in case:
            with pytest.raises(getattr(mp, case["error"])):
                mp.fuse(g, case["pred"], case["succ"], ov)
            n_err += 1
            continue
        out, merged = mp.fuse(g, case["pred"], case["succ"], ov)
        want = case["out"]
        assert [node_tuple(n) for n in out.nodes] == [golden_node_tuple(r) for r in want["nodes"]], case["name"]
        assert [(e.src, e.dst, e.payload_bytes) for e in out.edges] == [tuple(e) for e in want["edges"]], case["name"]
        assert merged.id == case["merged"]
        n_ok += 1
    assert n_ok > 50 and n_err >= 2


@pytest.mark.gpu
def test_greedy_matches_reference():
    n = 0
    for case in golden("aux.json")["greedy"]:
        g = graph_from(case["graph"])
        c = cluster_from(case["cluster"])
        mesh = mp.effective_bandwidth(c)
        kind = mp.BaselineKind(case["kind"])
        if "error" in case:
            with pytest.raises(mp.InfeasibleMemoryError) as ei:
                mp.greedy_place(g, c, mesh, kind)
            assert [ei.value.needed, ei.value.available] == case["error"], case["name"]
            continue
        s = mp.greedy_place(g, c, mesh, kind)
        w = case["schedule"]
        assert s.assignment == {int(k): v for k, v in w["assignment"].items()}, (case["name"], kind)
        assert s.makespan_s.hex() == F(w["makespan"]).hex(), case["name"]
        assert {k: v.hex() for k, v in s.starts.items()} == {int(k): F(v).hex() for k, v in w["starts"].items()}
        assert {k: v.hex() for k, v in s.ends.items()} == {int(k): F(v).hex() for k, v in w["ends"].items()}
        n += 1
    assert n > 100


@pytest.mark.gpu
def test_check_feasibility_matches_reference():
    n_clean = n_bad = 0
    for case in golden("aux.json")["audit"]:
        g = graph_from(case["graph"])
        c = cluster_from(case["cluster"])
        mesh = mp.effective_bandwidth(c)
        sched = _sched_from(case["schedule"])
        got = mp.check_feasibility(sched, g, c, mesh, F(case["tol"]))
        want = [(mp.ViolationKind(k), d, tuple(nodes)) for k, d, nodes in case["violations"]]
        assert [(v.kind, v.details, v.nodes) for v in got] == want, case["name"]
        n_clean += not want
        n_bad += bool(want)
    assert n_clean > 20 and n_bad > 40


@pytest.mark.gpu
def test_greedy_seeds_and_audit_on_workload(oracle_mod):
    """C2: the greedy row re-evaluates bit-exactly, seeds the local search, and
    every schedule the GPU produces audits clean."""
    import numpy as np

    from paper_2312_04025_b200 import workloads
    from paper_2312_04025_b200.baselines import greedy_row

    w = workloads.c2(4)
    coarse = mp.gcof(w.raw, w.rules)
    mesh = mp.effective_bandwidth(w.cluster)
    with mp.Instance(coarse, w.cluster, mesh) as inst:
        rows = np.stack([greedy_row(inst, k) for k in mp.BaselineKind])
        ms = mp.evaluate_batch(inst, rows)
        orc = oracle_mod.OracleInstance.from_instance(inst)
        want, _ = orc.eval_batch(rows)
        assert np.array_equal(ms.view(np.uint64), want.view(np.uint64))
        best_row, best_ms, _, _ = mp.local_search(inst, rows, chains=256, moves=64, seed=3)
        assert best_ms <= ms.min()
        sched = mp.schedule_for_assignment(coarse, w.cluster, mesh, inst.decode(best_row))
        assert sched.makespan_s == best_ms
        assert mp.check_feasibility(sched, coarse, w.cluster, mesh) == []
