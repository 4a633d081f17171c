"""The named benchmark workloads C1-C5 (BASELINE.json configs).

All inputs are synthetic and deterministic: graphs are built from seeded
templates (no checkpoints or traces exist offline), clusters follow Table III
of the paper (``PAPER.md:850-870``; Gbps converted to bytes/s as Gbps*1e9/8),
placements are ``numpy.random.Generator(PCG64(seed)).integers(0, K, (P, n_ops),
dtype=uint8)`` with seed = config index.

* C1 Inception-v4-sized: ``gen_synthetic(490 ops, width 4, density 0.5)``,
  Table-I rules, K=2 inter-server devices A (RTX 2080 Ti) / B (T4).
* C2 BERT-large: embed + 24 encoder layers x 20 ops (481 raw ops, 265/360
  after GCOF), K=4 intra-server V100, V100, P100, P100 (Table III) or the K=8
  variant of two such quads joined by 100 Gbps InfiniBand.
* C3 GPT-3-style: embed + 96 pre-LN decoder layers + final LN + LM head at
  hidden 12288; per-op weight bytes; K=8 with 48 GB caps (memory-infeasible
  placements occur).
* C4 ViT-L/16: patch-embed conv + the C2 encoder x 24 + head; K=8 (4 fast, 4
  1.6x slower devices) with an NVLink-5 or a PCIe Gen5 table.
* C5: ``gen_synthetic(n, width 32, density 0.5)`` sweep, K in {2, 4, 8}.
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass

import numpy as np

from .fusion import FusionRule, FusionRuleSet
from .graph import CompGraph, FlowEdge, OpNode
from .profiles import Cluster, Device
from .synth import GenSpec, gen_synthetic

GB = 1_000_000_000
MiB = 1 << 20
GBPS = 1e9 / 8.0  # bytes/s per Gbit/s


def table_rules() -> FusionRuleSet:
    """Table I conv-rooted family (reference test fixture ``conftest.py:27-33``)."""
    return FusionRuleSet([
        FusionRule(1, ("conv", "bn")),
        FusionRule(2, ("conv", "bn", "relu")),
        FusionRule(3, ("conv", "bn", "add", "relu")),
    ])


def transformer_rules() -> FusionRuleSet:
    """Rules of the transformer templates."""
    return FusionRuleSet([
        FusionRule(1, ("matmul", "add")),
        FusionRule(2, ("matmul", "add", "gelu")),
        FusionRule(3, ("add", "layernorm")),
    ])


# ---- clusters ------------------------------------------------------------------
def inter_server_2() -> Cluster:
    """Table III inter-server A (2080 Ti, 11 GB) and B (T4, 16 GB)."""
    return Cluster([Device(0, 11 * GB), Device(1, 16 * GB)],
                   {(0, 1): 44.26 * GBPS, (1, 0): 42.39 * GBPS})


_INTRA = {  # Table III intra-server average Gbps, row = source
    (0, 1): 1170.04, (0, 2): 626.10, (0, 3): 610.56,
    (1, 0): 1148.16, (1, 2): 618.98, (1, 3): 581.09,
    (2, 0): 630.43, (2, 1): 609.82, (2, 3): 571.96,
    (3, 0): 622.67, (3, 1): 575.08, (3, 2): 581.35,
}
_INTRA_MEM = (32 * GB, 32 * GB, 16 * GB, 16 * GB)


def intra_server_4() -> Cluster:
    return Cluster([Device(k, _INTRA_MEM[k]) for k in range(4)],
                   {pair: g * GBPS for pair, g in _INTRA.items()})


def intra_server_8() -> Cluster:
    """Two Table-III quads; every cross-quad pair is bottlenecked by 100 Gbps IB."""
    links = {}
    for q in (0, 4):
        for (a, b), g in _INTRA.items():
            links[(a + q, b + q)] = g * GBPS
    for a in range(4):
        for b in range(4, 8):
            links[(a, b)] = 100.0 * GBPS
            links[(b, a)] = 100.0 * GBPS
    return Cluster([Device(k, _INTRA_MEM[k % 4]) for k in range(8)], links)


def uniform_cluster(k: int, mem: int, bw: float) -> Cluster:
    return Cluster([Device(d, mem) for d in range(k)],
                   {(a, b): bw for a in range(k) for b in range(k) if a != b})


# ---- transformer templates -----------------------------------------------------
@dataclass
class _Builder:
    rng: random.Random
    speed: tuple[float, ...]
    nodes: list
    edges: list
    next_id: int = 1

    def op(self, t: str, lo: float, hi: float, mem: int) -> int:
        base = math.exp(self.rng.uniform(math.log(lo), math.log(hi)))
        times = {k: base * s * math.exp(self.rng.uniform(-0.1, 0.1)) for k, s in enumerate(self.speed)}
        nid = self.next_id
        self.next_id += 1
        self.nodes.append(OpNode(nid, t, mem, times))
        return nid

    def edge(self, a: int, b: int, payload: int):
        self.edges.append(FlowEdge(a, b, payload))


# per-op-type cost ranges (seconds at speed 1.0) for a 512-token sequence
_MM = (0.8e-4, 2.0e-4)
_EW = (0.5e-5, 3.0e-5)
_ATT = (0.5e-4, 1.5e-4)


def _encoder_layer(b: _Builder, x: int, hidden: int, heads: int, seq: int, ffn: int, pre_ln: bool) -> int:
    act = seq * hidden * 2
    scores = heads * seq * seq * 2
    inter = seq * ffn * 2
    wq = hidden * hidden * 2
    wf = hidden * ffn * 2
    bias = hidden * 2
    src = x
    if pre_ln:
        src = b.op("layernorm", *_EW, 4 * hidden)
        b.edge(x, src, act)
    q_mm = b.op("matmul", *_MM, wq)
    q_add = b.op("add", *_EW, bias)
    k_mm = b.op("matmul", *_MM, wq)
    k_add = b.op("add", *_EW, bias)
    v_mm = b.op("matmul", *_MM, wq)
    v_add = b.op("add", *_EW, bias)
    qk = b.op("matmul", *_ATT, 0)
    sm = b.op("softmax", *_EW, 0)
    av = b.op("matmul", *_ATT, 0)
    o_mm = b.op("matmul", *_MM, wq)
    o_add = b.op("add", *_EW, bias)
    res1 = b.op("add", *_EW, 0)
    ln1 = b.op("layernorm", *_EW, 4 * hidden)
    f1_mm = b.op("matmul", *_MM, wf)
    f1_add = b.op("add", *_EW, ffn * 2)
    gelu = b.op("gelu", *_EW, 0)
    f2_mm = b.op("matmul", *_MM, wf)
    f2_add = b.op("add", *_EW, bias)
    res2 = b.op("add", *_EW, 0)
    ln2 = b.op("layernorm", *_EW, 4 * hidden)
    for t in (q_mm, k_mm, v_mm):
        b.edge(src, t, act)
    b.edge(x, res1, act)
    b.edge(q_mm, q_add, act)
    b.edge(k_mm, k_add, act)
    b.edge(v_mm, v_add, act)
    b.edge(q_add, qk, act)
    b.edge(k_add, qk, act)
    b.edge(qk, sm, scores)
    b.edge(sm, av, scores)
    b.edge(v_add, av, act)
    b.edge(av, o_mm, act)
    b.edge(o_mm, o_add, act)
    b.edge(o_add, res1, act)
    b.edge(res1, ln1, act)
    b.edge(ln1, f1_mm, act)
    b.edge(ln1, res2, act)
    b.edge(f1_mm, f1_add, inter)
    b.edge(f1_add, gelu, inter)
    b.edge(gelu, f2_mm, inter)
    b.edge(f2_mm, f2_add, act)
    b.edge(f2_add, res2, act)
    b.edge(res2, ln2, act)
    return ln2


SPEED_4 = (1.0, 1.0, 1.6, 1.6)        # V100, V100, P100, P100
SPEED_8 = SPEED_4 + SPEED_4


def bert_large(speed=SPEED_4, layers: int = 24, seed: int = 2) -> CompGraph:
    """BERT-large encoder: embed + ``layers`` x 20 ops, 24 edges per layer (raw)."""
    b = _Builder(random.Random(seed), tuple(speed), [], [])
    x = b.op("embed", *_EW, 30522 * 1024 * 2)
    for _ in range(layers):
        x = _encoder_layer(b, x, 1024, 16, 512, 4096, pre_ln=False)
    return CompGraph(b.nodes, b.edges)


def gpt3_decoder(speed=SPEED_8, layers: int = 96, seed: int = 3, hidden: int = 12288) -> CompGraph:
    """GPT-3-style pre-LN decoder stack with an LM head (raw graph)."""
    b = _Builder(random.Random(seed), tuple(speed), [], [])
    seq, heads, ffn = 2048, 96, 4 * hidden
    x = b.op("embed", *_EW, 50257 * hidden * 2)
    for _ in range(layers):
        x = _encoder_layer(b, x, hidden, heads, seq, ffn, pre_ln=True)
    lnf = b.op("layernorm", *_EW, 4 * hidden)
    b.edge(x, lnf, seq * hidden * 2)
    head = b.op("matmul", *_MM, 50257 * hidden * 2)
    b.edge(lnf, head, seq * hidden * 2)
    return CompGraph(b.nodes, b.edges)


def vit_large(speed=(1.0,) * 4 + (1.6,) * 4, seed: int = 4) -> CompGraph:
    """ViT-L/16: patch-embed conv + 24 encoder layers + layernorm + head."""
    b = _Builder(random.Random(seed), tuple(speed), [], [])
    hidden, seq = 1024, 197
    x = b.op("conv", *_MM, 16 * 16 * 3 * hidden * 2)
    for _ in range(24):
        x = _encoder_layer(b, x, hidden, 16, seq, 4096, pre_ln=False)
    head = b.op("matmul", *_EW, hidden * 1000 * 2)
    b.edge(x, head, hidden * 2)
    return CompGraph(b.nodes, b.edges)


# ---- named configs ---------------------------------------------------------------
@dataclass
class Workload:
    name: str
    raw: CompGraph
    rules: FusionRuleSet
    cluster: Cluster
    placements: int
    seed: int


def c1() -> Workload:
    g = gen_synthetic(GenSpec(ops=490, width=4, density=0.5, devices=(0, 1),
                              mem_range=(1_000_000, 64_000_000)), seed=2312)
    return Workload("C1-inception-v4-490ops-K2", g, table_rules(), inter_server_2(), 4096, 1)


def c2(k: int = 4) -> Workload:
    if k == 4:
        return Workload("C2-bert-large-K4", bert_large(SPEED_4), transformer_rules(), intra_server_4(), 1 << 20, 2)
    return Workload("C2-bert-large-K8", bert_large(SPEED_8), transformer_rules(), intra_server_8(), 1 << 20, 2)


def c3() -> Workload:
    return Workload("C3-gpt3-96L-K8-48GB", gpt3_decoder(), transformer_rules(),
                    uniform_cluster(8, 48 * GB, 900e9), 1 << 20, 3)


def c4(link: str = "nvlink") -> Workload:
    bw = 900e9 if link == "nvlink" else 64e9
    return Workload(f"C4-vit-large-K8-{link}", vit_large(), transformer_rules(),
                    uniform_cluster(8, 180 * GB, bw), 1 << 24, 4)


def c5(n: int, k: int) -> Workload:
    g = gen_synthetic(GenSpec(ops=n, width=32, density=0.5, devices=tuple(range(k))), seed=0)
    rng = random.Random(0)
    links = {(a, b): rng.uniform(4e6, 4e7) for a in range(k) for b in range(k) if a != b}
    c = Cluster([Device(d, 10 ** 15) for d in range(k)], links)
    return Workload(f"C5-synth-{n}ops-K{k}", g, table_rules(), c, 0, 5)


def placements(seed: int, P: int, n_ops: int, K: int) -> np.ndarray:
    """The survey's placement stream: PCG64(seed) uint8 device indices."""
    g = np.random.Generator(np.random.PCG64(seed))
    return g.integers(0, K, (P, n_ops), dtype=np.uint8)
