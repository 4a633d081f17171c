"""Host data model of the drop-in surface, mirroring the reference's own tests
(pkg/tests/test_graph.py, test_profiles.py, test_fusion.py helpers)."""

from __future__ import annotations

import itertools
import logging
import random

import pytest

import paper_2312_04025_b200 as mp
from paper_2312_04025_b200 import workloads


def _node(i, t="conv", **kw):
    return mp.OpNode(i, t, kw.pop("mem", 1), kw.pop("times", {0: 1.0}), **kw)


def diamond():
    return mp.CompGraph([_node(i) for i in (1, 2, 3, 4)],
                        [mp.FlowEdge(1, 2, 5), mp.FlowEdge(1, 3, 6), mp.FlowEdge(2, 4, 7), mp.FlowEdge(3, 4, 8)])


def test_opnode_and_edge_validation():
    n = _node(3)
    assert n.members == (3,) and n.type_seq == ("conv",) and n.tag is mp.Tag.PLAIN
    with pytest.raises(ValueError):
        mp.OpNode(1, "x", -1, {})
    with pytest.raises(ValueError):
        mp.OpNode(1, "x", 1, {0: -1.0})
    with pytest.raises(ValueError):
        mp.OpNode(1, "x", 1, {}, members=(1, 1), type_seq=("a", "b"))
    with pytest.raises(ValueError):
        mp.OpNode(1, "x", 1, {}, members=(1, 2), type_seq=("a",))
    with pytest.raises(ValueError):
        mp.FlowEdge(1, 1, 0)
    with pytest.raises(ValueError):
        mp.FlowEdge(1, 2, -5)


def test_compgraph_contract():
    with pytest.raises(ValueError):
        mp.CompGraph([_node(1), _node(1)], [])
    with pytest.raises(mp.DanglingEdgeError):
        mp.CompGraph([_node(1)], [mp.FlowEdge(1, 2, 1)])
    with pytest.raises(ValueError):
        mp.CompGraph([_node(1), _node(2)], [mp.FlowEdge(1, 2, 1), mp.FlowEdge(1, 2, 3)])
    g = mp.CompGraph([_node(3), _node(1), _node(2)], [mp.FlowEdge(3, 1, 1), mp.FlowEdge(1, 2, 1),
                                                       mp.FlowEdge(3, 2, 9)])
    assert g.node_ids == [1, 2, 3]
    assert [(e.src, e.dst) for e in g.edges] == [(3, 1), (1, 2), (3, 2)]  # insertion order
    assert g.succs(3) == [1, 2] and g.preds(2) == [1, 3]
    assert g.edge(3, 2).payload_bytes == 9 and g.edge(2, 3) is None
    assert g == mp.CompGraph(list(g.nodes), list(reversed(g.edges)))
    dg = g.csr()
    assert list(dg.esrc) == [2, 0, 2] and list(dg.edst) == [0, 1, 1]


def test_validate_and_topo():
    g = diamond()
    mp.validate_dag(g)
    assert mp.topo_order(g) == [1, 2, 3, 4]
    cyc = mp.CompGraph([_node(1), _node(2), _node(3)],
                       [mp.FlowEdge(1, 2, 1), mp.FlowEdge(2, 3, 1), mp.FlowEdge(3, 2, 1)])
    with pytest.raises(mp.CycleError) as ei:
        mp.validate_dag(cyc)
    assert ei.value.cycle == [3, 2]  # same witness as the reference (graph.py:234-264)
    with pytest.raises(mp.CycleError):
        mp.topo_order(cyc)


def test_validate_warns_on_disconnected(caplog):
    g = mp.CompGraph([_node(1), _node(2)], [])
    with caplog.at_level(logging.WARNING):
        mp.validate_dag(g)
    assert "not weakly connected" in caplog.text


def test_augment_ids_follow_edge_order():
    g = mp.CompGraph([_node(5), _node(7), _node(9)], [mp.FlowEdge(9, 5, 1), mp.FlowEdge(5, 7, 2)])
    aug = mp.augment(g)
    assert aug.flow_ids == [10, 11]
    assert aug.flow_nodes[10].src == 9 and aug.flow_nodes[11].dst == 7
    assert aug.succs(9) == [10] and aug.preds(5) == [10]
    assert mp.contract(aug) == g


def test_succ_closure():
    c = mp.succ_closure(diamond())
    assert c[1] == frozenset({2, 3, 4}) and c[4] == frozenset()


def _widest_by_paths(c, src, dst):
    best = 0.0
    others = [d for d in c.device_ids if d not in (src, dst)]
    for r in range(len(others) + 1):
        for mids in itertools.permutations(others, r):
            path = (src, *mids, dst)
            w = min(c.links.get((a, b), 0.0) for a, b in zip(path, path[1:]))
            best = max(best, w)
    return best


def test_effective_bandwidth_is_the_widest_path():
    for trial in range(40):
        rng = random.Random(trial)
        n = rng.randint(2, 5)
        ids = list(range(1, n + 1))
        links = {(a, b): float(rng.randint(1, 40)) * 1e6 for a in ids for b in ids if a != b and rng.random() < 0.7}
        for a, b in zip(ids, ids[1:] + ids[:1]):
            links.setdefault((a, b), 2e6)
            links.setdefault((b, a), 2e6)
        c = mp.Cluster([mp.Device(i, 10) for i in ids], links)
        mesh = mp.effective_bandwidth(c)
        for a in ids:
            for b in ids:
                if a != b:
                    assert mesh.bandwidth(a, b) == _widest_by_paths(c, a, b)


def test_cluster_errors_and_comm_time():
    with pytest.raises(ValueError):
        mp.Device(1, 0)
    with pytest.raises(mp.DisconnectedClusterError):
        mp.Cluster([mp.Device(1, 10), mp.Device(2, 10)], {})
    with pytest.raises(mp.DisconnectedClusterError):
        mp.effective_bandwidth(mp.Cluster([mp.Device(1, 10), mp.Device(2, 10)], {(1, 2): 1e6}))
    relay = mp.Cluster([mp.Device(1, 100), mp.Device(2, 100), mp.Device(3, 100)],
                       {(1, 2): 1e7, (2, 1): 1e7, (2, 3): 5e6, (3, 2): 5e6})
    mesh = mp.effective_bandwidth(relay)
    assert mp.comm_time(100_000_000, 1, 3, mesh) == 20.0  # test_acceptance.py:113-118
    assert mp.comm_time(5, 2, 2, mesh) == 0.0


def test_fused_cost_and_overrides():
    n = mp.OpNode(1, "conv∘bn", 1, {0: 5.0}, members=(1, 2), type_seq=("conv", "bn"), tag=mp.Tag.FUSED)
    ov = mp.CostOverrides({(("conv", "bn"), 0): 3.5})
    assert mp.fused_cost(n, 0, ov) == 3.5 and mp.fused_cost(n, 0) == 5.0
    with pytest.raises(mp.MissingProfileError):
        mp.fused_cost(n, 1)
    with pytest.raises(ValueError):
        mp.CostOverrides({(("a",), 0): -1.0})


def test_rules_and_matching():
    rules = workloads.table_rules()
    assert rules.has_pattern(("conv", "bn")) and not rules.has_pattern(("bn", "conv"))
    with pytest.raises(ValueError):
        mp.FusionRule(1, ("a",))
    with pytest.raises(ValueError):
        mp.FusionRuleSet([mp.FusionRule(1, ("a", "b")), mp.FusionRule(1, ("c", "d"))])
    assert mp.match_rule(_node(1, "conv"), _node(2, "bn"), rules) == mp.Match(mp.MatchKind.PREFIX, 2)
    pair = mp.OpNode(1, "conv∘bn", 2, {0: 2.0}, members=(1, 2), type_seq=("conv", "bn"), tag=mp.Tag.BOUND)
    assert mp.match_rule(pair, _node(3, "relu"), rules) == mp.Match(mp.MatchKind.FULL, 2)
    assert mp.match_rule(_node(1, "bn"), _node(2, "conv"), rules) is None


def test_connection_classes():
    g = mp.CompGraph([_node(1), _node(2, "bn"), _node(3, "relu"), _node(4, "add")],
                     [mp.FlowEdge(1, 2, 1), mp.FlowEdge(1, 3, 1), mp.FlowEdge(2, 4, 1), mp.FlowEdge(3, 4, 1)])
    assert mp.classify_connection(g, 1, 2) is mp.ConnKind.MULTI_OUTPUTS
    assert mp.classify_connection(g, 2, 4) is mp.ConnKind.MULTI_INPUTS
    assert not mp.is_valid_conn(g, 1, 3) and mp.is_valid_conn(g, 3, 4)
    with pytest.raises(mp.UnknownEdgeError):
        mp.classify_connection(g, 2, 3)


def test_solve_budget_validation():
    with pytest.raises(ValueError):
        mp.SolveBudget(gap=1.0)
    assert mp.SolveBudget().gap == 0.0


def test_public_surface_names():
    """Every hot-path name of the reference surface exists (opplace/__init__.py:94-112)."""
    for name in ("AugGraph", "Cluster", "CompGraph", "CostOverrides", "CycleError", "Device", "EffectiveMesh",
                 "Event", "EventKind", "FlowEdge", "FlowNode", "FusionRule", "FusionRuleSet", "GenSpec",
                 "MemoryExceededError", "MissingCostError", "OpNode", "Schedule", "Solution", "SolveBudget",
                 "Status", "Tag", "TooLargeError", "augment", "brute_force", "comm_time", "effective_bandwidth",
                 "fused_cost", "gcof", "gen_synthetic", "match_rule", "schedule_for_assignment", "simulate",
                 "solve_exact", "topo_order", "validate_dag"):
        assert hasattr(mp, name), name


def test_mip_start_names_and_values_follow_the_reference_model():
    """x/z/u/S/C values of a schedule in the reference MILP's naming (milp.py:151-160);
    reading them back gives the same assignment, channels and times."""
    from paper_2312_04025_b200.mipstart import mip_start_text

    c = mp.Cluster([mp.Device(0, 100), mp.Device(1, 100)], {(0, 1): 5e6, (1, 0): 5e6})
    g = mp.CompGraph([mp.OpNode(1, "conv", 10, {0: 2.0, 1: 4.0}), mp.OpNode(2, "bn", 10, {0: 1.0, 1: 0.5})],
                     [mp.FlowEdge(1, 2, 10_000_000)])
    s = mp.Schedule({1: 0, 2: 1}, {1: 0.0, 3: 2.0, 2: 4.0}, {1: 2.0, 3: 4.0, 2: 4.5}, {3: (0, 1)}, 4.5)
    text = mip_start_text(s, g, c)
    vals = {ln.split()[0]: float(ln.split()[1]) for ln in text.splitlines() if not ln.startswith("#")}
    assert {k for k, v in vals.items() if k.startswith("x_") and v == 1.0} == {"x_1_0", "x_2_1"}
    assert vals["z_3"] == 1.0 and vals["u_3_0_1"] == 1.0 and vals["u_3_1_0"] == 0.0
    assert (vals["S_2"], vals["C_2"], vals["S_3"], vals["C_3"]) == (4.0, 4.5, 2.0, 4.0)
    import sys
    from pathlib import Path

    ref = Path("/root/reference/pkg/src")
    if ref.exists():  # the reference's own model declares exactly these names (here only)
        sys.path.insert(0, str(ref))
        import opplace

        rc = opplace.Cluster([opplace.Device(0, 100), opplace.Device(1, 100)], {(0, 1): 5e6, (1, 0): 5e6})
        rg = opplace.CompGraph([opplace.OpNode(1, "conv", 10, {0: 2.0, 1: 4.0}),
                                opplace.OpNode(2, "bn", 10, {0: 1.0, 1: 0.5})], [opplace.FlowEdge(1, 2, 10_000_000)])
        mdl = opplace.build_model(rg, rc, opplace.effective_bandwidth(rc))
        names = [v.name for v in mdl.vars]
        assert set(vals) == set(names)  # a complete start: every variable, T included
        x = [vals[nm] for nm in names]
        for row in mdl.rows:  # and a feasible one: every row of the model holds
            lhs = sum(cf * x[v] for cf, v in row.terms)
            assert (lhs <= row.rhs + 1e-9) if row.sense == "<=" else abs(lhs - row.rhs) <= 1e-9, row.name
    assert vals["T"] == 4.5


def test_mip_start_ordering_binaries_follow_the_schedule():
    """dord / dcom exist only for unrelated pairs (milp.py:141-145) and say which
    side runs first (ord1/ord2, milp.py:196-206)."""
    from paper_2312_04025_b200.mipstart import mip_start_values

    c = mp.Cluster([mp.Device(0, 100), mp.Device(1, 100)], {(0, 1): 5e6, (1, 0): 5e6})
    g = mp.CompGraph([mp.OpNode(1, "a", 1, {0: 1.0, 1: 1.0}), mp.OpNode(2, "b", 1, {0: 1.0, 1: 1.0}),
                      mp.OpNode(3, "c", 1, {0: 1.0, 1: 1.0})],
                     [mp.FlowEdge(1, 3, 5_000_000), mp.FlowEdge(2, 3, 5_000_000)])
    # ops 1, 2 unrelated on device 0 (2 first), 3 on device 1; flows 4 (1->3), 5 (2->3)
    s = mp.Schedule({1: 0, 2: 0, 3: 1}, {2: 0.0, 1: 1.0, 5: 1.0, 4: 2.0, 3: 3.0},
                    {2: 1.0, 1: 2.0, 5: 2.0, 4: 3.0, 3: 4.0}, {4: (0, 1), 5: (0, 1)}, 4.0)
    v = mip_start_values(s, g, c)
    assert v["dord_1_2"] == 0.0 and "dord_1_3" not in v and "dord_2_3" not in v
    assert v["dcom_4_5"] == 0.0 and v["T"] == 4.0


def test_bulk_object_construction_restores_the_collector():
    """The GC pause around bulk OpNode creation (gcof, load_graph) restores the
    collector's previous state, also when the body raises."""
    import gc

    from paper_2312_04025_b200.graph import _bulk_objects

    assert gc.isenabled()
    with _bulk_objects():
        assert not gc.isenabled()
    assert gc.isenabled()
    try:
        with _bulk_objects():
            raise ValueError("boom")
    except ValueError:
        pass
    assert gc.isenabled()
    gc.disable()
    try:
        with _bulk_objects():
            pass
        assert not gc.isenabled()
    finally:
        gc.enable()
