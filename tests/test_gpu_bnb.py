"""GPU branch and bound (``solve_exact``, reference solver.py:172-254).

Parity bar:
* gap 0, no limits — status, objective (bits) and placement equal the
  reference's (golden brute_force.json / solve_exact.json, produced by the
  reference itself) and, past the golden sizes, the oracle's restatement of the
  reference's serial branch and bound (oracle/moirai_oracle.c orc_solve_exact,
  pinned by tests/test_oracle.py);
* gap > 0 — the reference's certificate: status OPTIMAL, ``gap`` reported, and
  objective <= optimum / (1 - gap);
* every returned placement re-evaluates (oracle ``_schedule``) to the same bits.
"""

from __future__ import annotations

import math

import numpy as np
import pytest
from conftest import F, cluster_from, golden, graph_from

import paper_2312_04025_b200 as mp

pytestmark = pytest.mark.gpu


def _orc(oracle_mod, g, c):
    from test_oracle import _flat_instance

    return _flat_instance(oracle_mod, g, c, mp.effective_bandwidth(c))


def _row(g, c, placement):
    return np.array([c.device_ids.index(placement[i]) for i in g.node_ids], dtype=np.uint8)


def _reverify(oracle_mod, g, c, sol):
    st, ms, *_ = _orc(oracle_mod, g, c).schedule(_row(g, c, sol.placement))
    assert st == 0 and ms.hex() == sol.objective_s.hex()


def test_gap0_equals_reference_brute_force_golden():
    for case in golden("brute_force.json"):
        g = graph_from(case["graph"])
        c = cluster_from(case["cluster"])
        sol = mp.solve_exact(g, c, mp.effective_bandwidth(c))
        assert sol.status.value == case["status"], case["name"]
        assert sol.objective_s.hex() == F(case["objective"]).hex(), case["name"]
        if "placement" in case:
            assert sol.placement == {int(k): v for k, v in case["placement"].items()}, case["name"]
            assert sol.gap == 0.0


def test_reference_solve_exact_golden(oracle_mod):
    n_exact = n_gap = n_lim = 0
    for case in golden("solve_exact.json"):
        g = graph_from(case["graph"])
        c = cluster_from(case["cluster"])
        mesh = mp.effective_bandwidth(c)
        gap = F(case["gap"])
        budget = mp.SolveBudget(gap=gap, node_limit=case["node_limit"])
        sol = mp.solve_exact(g, c, mesh, budget)
        if case["node_limit"] is None and gap == 0.0:
            assert sol.status.value == case["status"], case["name"]
            assert sol.objective_s.hex() == F(case["objective"]).hex(), case["name"]
            if "placement" in case:
                assert sol.placement == {int(k): v for k, v in case["placement"].items()}, case["name"]
            n_exact += 1
        elif case["node_limit"] is None:
            opt = mp.solve_exact(g, c, mesh)
            assert sol.status.value == case["status"], case["name"]
            if sol.status is mp.Status.OPTIMAL:
                assert sol.gap == gap
                assert sol.objective_s <= opt.objective_s / (1.0 - gap) * (1 + 1e-12), case["name"]
                # the reference's own pick satisfies the same certificate
                assert F(case["objective"]) <= opt.objective_s / (1.0 - gap) * (1 + 1e-12)
            n_gap += 1
        else:
            # a limit may stop the search (FEASIBLE / BUDGET) or the tree may be
            # exhausted within it (OPTIMAL / INFEASIBLE, then it must be the truth)
            if sol.status in (mp.Status.OPTIMAL, mp.Status.INFEASIBLE):
                opt = mp.solve_exact(g, c, mesh, mp.SolveBudget(gap=gap))
                assert sol.status is opt.status, case["name"]
                if gap == 0.0 and opt.schedule is not None:
                    assert sol.objective_s == opt.objective_s and sol.placement == opt.placement
            if case["status"] == "infeasible":
                assert sol.status in (mp.Status.INFEASIBLE, mp.Status.BUDGET), case["name"]
            n_lim += 1
        if sol.schedule is not None:
            _reverify(oracle_mod, g, c, sol)
    assert n_exact == 20 and n_gap == 71 and n_lim == 53


def _random_instance(seed: int, n_ops: int, K: int, tight: bool):
    """Seeded layered DAG with heterogeneous costs, random link bandwidths and
    optional memory pressure (the shape of the reference's random_instance,
    conftest.py:127-154, at sizes past the brute-force guard)."""
    r = np.random.Generator(np.random.PCG64(seed))
    nodes, edges = [], []
    mem = r.integers(1, 40, n_ops)
    for i in range(n_ops):
        nodes.append(mp.OpNode(i + 1, "op", int(mem[i]),
                               {k: float(np.round(r.uniform(0.5, 8.0), 3)) for k in range(K)}))
    seen = set()
    for j in range(1, n_ops):
        for _ in range(int(r.integers(1, 3))):
            i = int(r.integers(max(0, j - 4), j))
            if (i, j) not in seen:
                seen.add((i, j))
                edges.append(mp.FlowEdge(i + 1, j + 1, int(r.integers(1_000_000, 40_000_000))))
    capv = int(mem.sum() * (0.45 if tight else 2))
    c = mp.Cluster([mp.Device(k, capv) for k in range(K)],
                   {(a, b): float(r.uniform(4e6, 4e7)) for a in range(K) for b in range(K) if a != b})
    return mp.CompGraph(nodes, edges), c


@pytest.mark.parametrize("seed", range(7))
def test_gap0_matches_reference_bnb_past_the_guard(oracle_mod, seed):
    """n*log2(K) > 24: brute force refuses; the reference's serial B&B (oracle
    restatement) and the GPU B&B must agree on status, objective and placement.
    (seed 6: 20 ops x 4 devices, 3.9M nodes in the serial search.)"""
    n_ops, K = (14, 4) if seed % 2 == 0 else (18, 3)
    if seed == 6:
        n_ops, K = 20, 4
    g, c = _random_instance(1000 + seed - 5 * (seed == 6), n_ops, K, tight=4 <= seed < 6)
    with pytest.raises(mp.TooLargeError):
        mp.brute_force(g, c, mp.effective_bandwidth(c))
    sol = mp.solve_exact(g, c, mp.effective_bandwidth(c))
    orc = _orc(oracle_mod, g, c)
    ids = g.node_ids
    order = [ids.index(x) for x in mp.topo_order(g)]
    st, row, best, visited = orc.solve_exact(order)
    assert {0: "optimal", 2: "infeasible"}[st] == sol.status.value
    assert sol.objective_s.hex() == best.hex()
    if st == 0:
        assert sol.placement == {ids[i]: c.device_ids[int(d)] for i, d in enumerate(row)}
        _reverify(oracle_mod, g, c, sol)


def test_seeds_do_not_change_the_gap0_answer():
    g, c = _random_instance(77, 12, 4, tight=False)
    mesh = mp.effective_bandwidth(c)
    a = mp.solve_exact(g, c, mesh, seed_chains=0)
    b = mp.solve_exact(g, c, mesh, seed_chains=4096, seed_moves=512)
    assert a.objective_s.hex() == b.objective_s.hex() and a.placement == b.placement
    bf = mp.brute_force(g, c, mesh)
    assert bf.objective_s.hex() == a.objective_s.hex() and bf.placement == a.placement


def test_budgeted_solve_on_coarse_graph_is_clean(oracle_mod):
    """test_acceptance.py:244-263: gap 0.05 with a time budget on the 30-op,
    4-device coarse graph -> OPTIMAL or FEASIBLE, simulator-clean."""
    case = next(x for x in golden("solve_exact.json") if x["name"] == "accept8-nodes500")
    g = graph_from(case["graph"])
    c = cluster_from(case["cluster"])
    assert (len(g.nodes), len(g.edges)) == (30, 57)
    mesh = mp.effective_bandwidth(c)
    sol = mp.solve_exact(g, c, mesh, mp.SolveBudget(gap=0.05, time_limit_s=30.0), seed_chains=1024)
    assert sol.status in (mp.Status.OPTIMAL, mp.Status.FEASIBLE)
    ms, _ = mp.simulate(g, c, mesh, sol.placement)
    assert ms == sol.objective_s
    _reverify(oracle_mod, g, c, sol)
    # no worse than the reference's own best after 5000 nodes
    ref5k = next(x for x in golden("solve_exact.json") if x["name"] == "accept8-nodes5000")
    assert sol.objective_s <= F(ref5k["objective"])


def test_node_and_time_limits():
    g, c = _random_instance(5, 16, 4, tight=False)
    mesh = mp.effective_bandwidth(c)
    s1 = mp.solve_exact(g, c, mesh, mp.SolveBudget(node_limit=1))  # no seed with a limit: the reference's BUDGET
    assert s1.status is mp.Status.BUDGET and s1.schedule is None and math.isinf(s1.objective_s)
    s2 = mp.solve_exact(g, c, mesh, mp.SolveBudget(node_limit=1), seed_chains=1024)  # opt-in seed
    assert s2.status is mp.Status.FEASIBLE and s2.schedule is not None and s2.gap is None
    s3 = mp.solve_exact(g, c, mesh, mp.SolveBudget(time_limit_s=0.0))
    assert s3.status in (mp.Status.FEASIBLE, mp.Status.BUDGET)
