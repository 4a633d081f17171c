"""Schema-1 interchange (reference fileio.py): the native graph loader returns the
same CompGraph as the reference procedure, documents it refuses fall back to the
reference's errors, and every save_* writes the reference's document."""

from __future__ import annotations

import json

import pytest
from conftest import golden, graph_from, node_tuple

import paper_2312_04025_b200 as mp
from paper_2312_04025_b200 import fileio


def _same(a, b):
    assert [node_tuple(n) for n in a.nodes] == [node_tuple(n) for n in b.nodes]
    assert [(e.src, e.dst, e.payload_bytes) for e in a.edges] == [(e.src, e.dst, e.payload_bytes) for e in b.edges]


def test_native_loader_round_trips_golden_graphs(tmp_path):
    graphs = [graph_from(c["graph"]) for c in golden("schedules.json")[:40]]
    for c in golden("gcof.json")[:60]:
        graphs.append(graph_from(c["graph"]))
        if "out" in c:
            graphs.append(graph_from(c["out"]))
    graphs.append(mp.gen_synthetic(mp.GenSpec(ops=3000, width=16, density=0.5, devices=(0, 1, 2)), 5))
    n_fused = 0
    for k, g in enumerate(graphs):
        p = tmp_path / f"g{k}.json"
        fileio.save_graph(g, p)
        got = fileio.load_graph(p)
        _same(got, fileio._load_graph_python(p))
        _same(got, g)
        n_fused += any(n.tag is mp.Tag.FUSED for n in got.nodes)
        arr = fileio.load_graph_arrays(p)
        assert arr["id"].tolist() == [n.id for n in g.nodes]
    assert n_fused >= 3  # "∘"-joined op types (\\u2218 escapes) went through the native reader


@pytest.mark.parametrize("mutate, exc", [
    (lambda d: d.update(schema=2), ValueError),
    (lambda d: d.update(kind="rules"), ValueError),
    (lambda d: d["nodes"].append(dict(d["nodes"][0])), ValueError),                      # duplicate id
    (lambda d: d["edges"].append({"src": 1, "dst": 999, "payload_bytes": 1}), mp.DanglingEdgeError),
    (lambda d: d["edges"].append(dict(d["edges"][0])), ValueError),                      # parallel edge
    (lambda d: d["edges"].append({"src": 2, "dst": 2, "payload_bytes": 1}), ValueError),  # self edge
    (lambda d: d["edges"][0].update(payload_bytes=-1), ValueError),
    (lambda d: d["nodes"][0].update(mem_bytes=-5), ValueError),
    (lambda d: d["nodes"][0].update(members=[1, 2, 3]), ValueError),                     # length mismatch
    (lambda d: d["nodes"][0]["compute_time"].update({"0": -1.0}), ValueError),
    (lambda d: d["nodes"][0].update(tag="odd"), ValueError),
])
def test_invalid_documents_raise_the_reference_errors(tmp_path, mutate, exc):
    g = mp.CompGraph([mp.OpNode(1, "conv", 4, {0: 1.0, 1: 2.0}), mp.OpNode(2, "bn", 4, {0: 1.0, 1: 2.0}),
                      mp.OpNode(3, "relu", 4, {0: 1.0, 1: 2.0})],
                     [mp.FlowEdge(1, 2, 10), mp.FlowEdge(2, 3, 10)])
    p = tmp_path / "g.json"
    fileio.save_graph(g, p)
    doc = json.loads(p.read_text())
    mutate(doc)
    p.write_text(json.dumps(doc))
    with pytest.raises(exc):
        fileio.load_graph(p)


def test_other_documents_round_trip(tmp_path):
    rules = mp.FusionRuleSet([mp.FusionRule(1, ("conv", "bn")), mp.FusionRule(2, ("matmul", "add", "gelu"))])
    fileio.save_rules(rules, tmp_path / "r.json")
    assert [(r.id, r.pattern) for r in fileio.load_rules(tmp_path / "r.json")] == [(r.id, r.pattern) for r in rules]
    c = mp.Cluster([mp.Device(0, 100), mp.Device(1, 50)], {(0, 1): 1e9, (1, 0): 2e9})
    fileio.save_cluster(c, tmp_path / "c.json")
    c2 = fileio.load_cluster(tmp_path / "c.json")
    assert c2.device_ids == c.device_ids and dict(c2.links) == dict(c.links)
    ov = mp.CostOverrides({(("conv", "bn"), 0): 3.5})
    fileio.save_overrides(ov, tmp_path / "o.json")
    assert dict(fileio.load_overrides(tmp_path / "o.json").entries) == dict(ov.entries)
    text = (tmp_path / "c.json").read_text()
    assert text.endswith("\n") and json.loads(text)["schema"] == 1 and '"kind": "cluster"' in text


def test_loaded_graph_carries_gcof_arrays_without_objects(tmp_path):
    """load_graph's GCOF input (interned type sequences, tags, memory, cost matrix) is
    built from the native reader's arrays, nodes in any file order and with sparse device
    costs, equal to the object path's; no OpNode is built until someone asks."""
    import random

    import numpy as np

    from paper_2312_04025_b200.fusion import _NodeArrays

    graphs = [graph_from(c["graph"]) for c in golden("gcof.json")[:60]]
    graphs.append(mp.gen_synthetic(mp.GenSpec(ops=2000, width=16, density=0.5, devices=(0, 1, 2)), 7))
    graphs.append(mp.CompGraph([mp.OpNode(5, "conv", 4, {0: 1.0, 3: 2.0}), mp.OpNode(2, "bn", 8, {3: 1.5}),
                                mp.OpNode(9, "relu", 1, {1: 0.5, 0: 0.25}, (9, 10), ("relu", "conv"), mp.Tag.BOUND)],
                               [mp.FlowEdge(5, 2, 10), mp.FlowEdge(2, 9, 10)]))
    rng = random.Random(3)
    for k, g in enumerate(graphs):
        p = tmp_path / f"g{k}.json"
        fileio.save_graph(g, p)
        doc = json.loads(p.read_text())
        rng.shuffle(doc["nodes"])
        p.write_text(json.dumps(doc))
        got = fileio.load_graph(p)
        assert got._nodes_d is None
        na, ref = got._gcof_node_arrays, _NodeArrays(g)
        assert na.types == ref.types and na.devices == ref.devices
        for f in ("seq_beg", "seq", "tag", "mem"):
            assert np.array_equal(getattr(na, f), getattr(ref, f)), (k, f)
        assert na.cost.shape == ref.cost.shape
        assert np.array_equal(np.isnan(na.cost), np.isnan(ref.cost))
        assert np.array_equal(np.nan_to_num(na.cost).view(np.int64), np.nan_to_num(ref.cost).view(np.int64))
        for f in ("esrc", "edst", "payload"):
            assert getattr(got.csr(), f).tolist() == getattr(g.csr(), f).tolist(), (k, f)
        assert got._nodes_d is None  # still no objects
        _same(got, g)
