"""The CPU oracle is pinned against golden vectors produced by the reference.

If these pass, the oracle restates the reference's `_schedule`, `brute_force`
and `gcof` exactly on every fixture, so GPU-vs-oracle parity tests at sizes
beyond the fixtures inherit the reference as their ground truth.
"""

from __future__ import annotations

import numpy as np
import pytest
from conftest import F, cluster_from, golden, golden_node_tuple, graph_from, mesh_from, rules_from, overrides_from

import paper_2312_04025_b200 as mp
from paper_2312_04025_b200.fusion import _Flat


def _flat_instance(oracle_mod, g, c, mesh):
    """Oracle instance from the package's flattening, without touching the GPU."""
    ids = g.node_ids
    devs = c.device_ids
    K = len(devs)
    dg = g.csr()
    cost = np.array([[g.node(i).compute_time[d] for d in devs] for i in ids], dtype=np.float64)
    mem = np.array([g.node(i).mem_bytes for i in ids], dtype=np.int64)
    cap = np.array([c.device(d).mem_bytes for d in devs], dtype=np.int64)
    bw = np.zeros((K, K))
    for a, da in enumerate(devs):
        for b, db in enumerate(devs):
            if a != b:
                bw[a, b] = mesh.bandwidth(da, db)
    return oracle_mod.OracleInstance(cost, mem, dg.esrc, dg.edst, dg.payload, cap, bw)


def test_oracle_schedules_match_reference(oracle_mod):
    n = 0
    for case in golden("schedules.json"):
        g = graph_from(case["graph"])
        c = cluster_from(case["cluster"])
        mesh = mesh_from(case["mesh"], c)
        orc = _flat_instance(oracle_mod, g, c, mesh)
        devs = c.device_ids
        ids = g.node_ids
        flow_ids = [ids[-1] + 1 + f for f in range(len(g.edges))]
        for asg, want in zip(case["assignments"], case["results"]):
            row = np.array([devs.index(asg[str(i)]) for i in ids], dtype=np.uint8)
            st, ms, starts, ends, md, ov = orc.schedule(row)
            if want["status"] == "memory":
                assert st == 1, case["name"]
                assert devs[md] == want["device"] and ov == want["overflow"], case["name"]
                continue
            assert st == 0, case["name"]
            assert ms.hex() == F(want["makespan"]).hex(), case["name"]
            for k, nid in enumerate(ids + flow_ids):
                assert starts[k].hex() == F(want["starts"][str(nid)]).hex(), (case["name"], nid)
                assert ends[k].hex() == F(want["ends"][str(nid)]).hex(), (case["name"], nid)
            n += 1
    assert n > 300


def test_oracle_brute_force_matches_reference(oracle_mod):
    for case in golden("brute_force.json"):
        g = graph_from(case["graph"])
        c = cluster_from(case["cluster"])
        mesh = mp.effective_bandwidth(c)
        orc = _flat_instance(oracle_mod, g, c, mesh)
        ids = g.node_ids
        order = [ids.index(x) for x in mp.topo_order(g)]
        idx, best = orc.enumerate(order)
        if case["status"] == "infeasible":
            assert idx == -1, case["name"]
            continue
        assert best.hex() == F(case["objective"]).hex(), case["name"]
        K = len(c.device_ids)
        digits = []
        x = idx
        for _ in ids:
            digits.append(x % K)
            x //= K
        digits.reverse()
        got = {ids[order[t]]: c.device_ids[d] for t, d in enumerate(digits)}
        assert got == {int(k): v for k, v in case["placement"].items()}, case["name"]


_STATUS = {0: "optimal", 1: "feasible", 2: "infeasible", 3: "budget"}


def test_oracle_solve_exact_matches_reference(oracle_mod):
    """orc_solve_exact restates solve_exact's DFS, bound, drift and node counting:
    status, objective bits and placement equal the reference's under gap and
    node-limit budgets (tests/golden/solve_exact.json)."""
    n = 0
    for case in golden("solve_exact.json"):
        g = graph_from(case["graph"])
        c = cluster_from(case["cluster"])
        mesh = mp.effective_bandwidth(c)
        orc = _flat_instance(oracle_mod, g, c, mesh)
        ids = g.node_ids
        order = [ids.index(x) for x in mp.topo_order(g)]
        st, row, best, _ = orc.solve_exact(order, F(case["gap"]), case["node_limit"])
        assert _STATUS[st] == case["status"], case["name"]
        assert best.hex() == F(case["objective"]).hex(), case["name"]
        if "placement" in case:
            got = {ids[i]: c.device_ids[int(d)] for i, d in enumerate(row)}
            assert got == {int(k): v for k, v in case["placement"].items()}, case["name"]
        n += 1
    assert n == 144


@pytest.mark.parametrize("chunk", range(4))
def test_oracle_gcof_matches_reference(oracle_mod, chunk):
    cases = golden("gcof.json")
    for case in cases[chunk::4]:
        g = graph_from(case["graph"])
        rules = rules_from(case["rules"])
        ov = overrides_from(case.get("overrides"))
        fl = _Flat(g, rules, ov)
        k = fl.keep
        part = oracle_mod.gcof_partition(k[1], k[2], k[3], k[6], k[7], k[10], k[11])
        nodes, edges = oracle_mod.materialize(g, part, ov)
        got = [(i, t, mem, tuple(sorted((kk, float(v).hex()) for kk, v in cost.items())), tuple(members),
                tuple(seq), tag) for i, t, members, seq, tag, mem, cost in nodes]
        want = [golden_node_tuple(r) for r in case["out"]["nodes"]]
        assert got == want, case["name"]
        assert [list(e) for e in edges] == case["out"]["edges"], case["name"]


def test_python_sum_semantics_are_neumaier():
    """Fused costs are sum() over member times (fusion.py:129); on CPython 3.12+
    that is a compensated sum, which the GPU coarsener restates."""
    import math
    import random
    import sys

    if sys.version_info < (3, 12):
        pytest.skip("plain summation before 3.12")
    rng = random.Random(1)

    def neumaier(vals):
        f = 0.0 + vals[0]
        c = 0.0
        for x in vals[1:]:
            t = f + x
            c += ((f - t) + x) if abs(f) >= abs(x) else ((x - t) + f)
            f = t
        if c and math.isfinite(c):
            f += c
        return f

    for _ in range(20000):
        vals = [rng.uniform(0.5, 8.0) * 10 ** rng.randint(-12, 12) for _ in range(rng.randint(1, 5))]
        assert sum(vals).hex() == neumaier(vals).hex()


def test_oracle_schedules_match_reference_simulate_traces(oracle_mod):
    """The oracle's starts/ends equal the event times of the reference's own
    `simulate` (tests/golden/simulate.json), including graphs whose costs are
    missing on devices no op uses (filled with +inf, never read)."""
    n = 0
    for case in golden("simulate.json"):
        g = graph_from(case["graph"])
        c = cluster_from(case["cluster"])
        devs = c.device_ids
        ids = g.node_ids
        for a, want in zip(case["assignments"], case["results"]):
            if want["status"] != "ok":
                continue
            ct = np.array([[g.node(i).compute_time.get(d, np.inf) for d in devs] for i in ids], dtype=np.float64)
            mesh = mp.effective_bandwidth(c)
            K = len(devs)
            bw = np.zeros((K, K))
            for x, dx in enumerate(devs):
                for y, dy in enumerate(devs):
                    if x != y:
                        bw[x, y] = mesh.bandwidth(dx, dy)
            dg = g.csr()
            orc = oracle_mod.OracleInstance(ct, np.array([g.node(i).mem_bytes for i in ids], dtype=np.int64),
                                            dg.esrc, dg.edst, dg.payload,
                                            np.array([c.device(d).mem_bytes for d in devs], dtype=np.int64), bw)
            row = np.array([devs.index(a[str(i)]) for i in ids], dtype=np.uint8)
            s, ms, st, en, _, _ = orc.schedule(row)
            assert s == 0 and ms.hex() == F(want["makespan"]).hex()
            max_id = max(ids)
            node_index = {i: x for x, i in enumerate(ids)}
            node_index.update({max_id + 1 + f: len(ids) + f for f in range(len(g.edges))})
            for t, kind, node, _, _ in want["events"]:
                arr = st if kind.endswith("start") else en
                assert arr[node_index[node]].hex() == F(t).hex(), (case["name"], node, kind)
            n += 1
    assert n >= 95
