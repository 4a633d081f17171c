"""Shared helpers: golden-fixture loading and conversion to the package's types.

Tests marked ``gpu`` need a B200 (run with ``-m gpu``); everything else runs on
CPU.  GPU tests are never skipped silently: on a box without a GPU they fail.
"""

from __future__ import annotations

import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import paper_2312_04025_b200 as mp  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@lru_cache(maxsize=None)
def golden(name: str):
    return json.loads((GOLDEN / name).read_text())


def F(h: str) -> float:
    return float.fromhex(h)


def graph_from(d) -> mp.CompGraph:
    nodes = [mp.OpNode(i, t, mem, {int(k): F(v) for k, v in ct.items()}, tuple(members), tuple(seq), mp.Tag(tag))
             for i, t, mem, ct, members, seq, tag in d["nodes"]]
    return mp.CompGraph(nodes, [mp.FlowEdge(a, b, p) for a, b, p in d["edges"]])


def cluster_from(d) -> mp.Cluster:
    return mp.Cluster([mp.Device(i, m) for i, m in d["devices"]], {(a, b): F(h) for a, b, h in d["links"]})


def mesh_from(d, c=None) -> mp.EffectiveMesh:
    bw = {(a, b): F(h) for a, b, h in d}
    ids = sorted({a for a, _ in bw} | {b for _, b in bw}) if bw else (c.device_ids if c else [])
    if c is not None:
        ids = c.device_ids
    return mp.EffectiveMesh(ids, bw)


def rules_from(d) -> mp.FusionRuleSet:
    return mp.FusionRuleSet([mp.FusionRule(i, tuple(p)) for i, p in d])


def overrides_from(d):
    if d is None:
        return None
    return mp.CostOverrides({(tuple(s), k): F(t) for s, k, t in d})


def node_tuple(n):
    """Everything observable about an output node, floats as exact hex."""
    return (n.id, n.op_type, n.mem_bytes, tuple(sorted((k, float(v).hex()) for k, v in n.compute_time.items())),
            tuple(n.members), tuple(n.type_seq), n.tag.value)


def golden_node_tuple(row):
    i, t, mem, ct, members, seq, tag = row
    return (i, t, mem, tuple(sorted((int(k), F(v).hex()) for k, v in ct.items())), tuple(members), tuple(seq), tag)


def bits(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float64).view(np.uint64)


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle

    oracle.build()
    return oracle
