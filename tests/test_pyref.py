"""The pure-Python reference arm (oracle/pyref.py) reproduces the reference's
makespans on the golden schedule cases, and its multi-process driver returns
rows in order."""

from __future__ import annotations

import numpy as np
from conftest import F, cluster_from, golden, graph_from, mesh_from

from oracle import pyref


def _arrays(g, c, mesh):
    ids = g.node_ids
    devs = c.device_ids
    dg = g.csr()
    K = len(devs)
    bw = np.zeros((K, K))
    for a, da in enumerate(devs):
        for b, db in enumerate(devs):
            if a != b:
                bw[a, b] = mesh.bandwidth(da, db)
    return (np.array([[g.node(i).compute_time[d] for d in devs] for i in ids], dtype=np.float64),
            np.array([g.node(i).mem_bytes for i in ids], dtype=np.int64), dg.esrc, dg.edst, dg.payload,
            np.array([c.device(d).mem_bytes for d in devs], dtype=np.int64), bw)


def test_pyref_matches_golden_makespans():
    n = 0
    for case in golden("schedules.json"):
        g = graph_from(case["graph"])
        c = cluster_from(case["cluster"])
        inst = pyref.Instance.from_arrays(_arrays(g, c, mesh_from(case["mesh"], c)))
        devs = c.device_ids
        for asg, want in zip(case["assignments"], case["results"]):
            a = {k: devs.index(asg[str(i)]) for k, i in enumerate(g.node_ids)}
            if want["status"] == "memory":
                try:
                    pyref.schedule(inst, a)
                    raise AssertionError("expected memory overflow")
                except pyref.MemoryExceeded as e:
                    assert (devs[e.device], e.overflow) == (want["device"], want["overflow"])
                continue
            assert pyref.schedule(inst, a).hex() == F(want["makespan"]).hex(), case["name"]
            n += 1
    assert n > 300


def test_pyref_all_cores_preserves_order():
    case = golden("schedules.json")[0]
    g = graph_from(case["graph"])
    c = cluster_from(case["cluster"])
    arrays = _arrays(g, c, mesh_from(case["mesh"], c))
    rows = np.random.default_rng(0).integers(0, len(c.device_ids), (37, len(g)), dtype=np.uint8)
    _, ms, procs = pyref.time_all_cores(arrays, rows, processes=3)
    assert procs == 3
    assert ms == pyref.eval_rows(pyref.Instance.from_arrays(arrays), rows)
