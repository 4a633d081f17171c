"""Fusion rules and GCOF coarsening (``pkg/src/opplace/fusion.py``).

Rule types and the single-pair helpers (``match_rule``, ``classify_connection``,
``is_valid_conn``) are small host utilities of the API.  :func:`gcof` — the hot
path — runs on the GPU through ``mp_coarsen`` (K1/K2, csrc/mp_coarsen.cu): the
graph, the interned type sequences and the rules are flattened here, the
partition, fused costs and quotient edges come back as arrays, and the output
``CompGraph`` is assembled from them (singleton groups reuse the input node
objects exactly as ``materialize`` does, ``fusion.py:233-235``).
"""

from __future__ import annotations

import ctypes as C
import sys
from itertools import chain
from operator import attrgetter
from dataclasses import dataclass
from enum import Enum
from typing import Iterable, Iterator

import numpy as np

from . import _native as N
from .errors import CycleCreationError, CycleError, UnknownEdgeError
from .graph import CompGraph, FlowEdge, OpNode, Tag, _bulk_objects, find_cycle, validate_dag
from .profiles import CostOverrides

FUSE_JOINER = "∘"  # joins member types in a fused node's op_type (fusion.py:23)


class ConnKind(Enum):
    DIRECT = "direct"
    MULTI_OUTPUTS = "multi_outputs"
    MULTI_INPUTS = "multi_inputs"


@dataclass(frozen=True)
class FusionRule:
    """A type sequence that may become one kernel (``fusion.py:32-43``)."""

    id: int
    pattern: tuple[str, ...]

    def __post_init__(self):
        if len(self.pattern) < 2:
            raise ValueError(f"rule {self.id}: pattern needs at least two op types")
        if not all(self.pattern):
            raise ValueError(f"rule {self.id}: empty op type in pattern")


class FusionRuleSet:
    """Rules with unique ids (``fusion.py:46-63``)."""

    def __init__(self, rules: Iterable[FusionRule]):
        self.rules = list(rules)
        ids = [r.id for r in self.rules]
        if len(ids) != len(set(ids)):
            raise ValueError("duplicate rule ids")
        self._patterns = frozenset(r.pattern for r in self.rules)

    def has_pattern(self, seq: tuple[str, ...]) -> bool:
        return seq in self._patterns

    def __iter__(self) -> Iterator[FusionRule]:
        return iter(self.rules)

    def __len__(self) -> int:
        return len(self.rules)


class MatchKind(Enum):
    FULL = "full"
    PREFIX = "prefix"


@dataclass(frozen=True)
class Match:
    kind: MatchKind
    rule_id: int


def classify_connection(g: CompGraph, src: int, dst: int) -> ConnKind:
    """Edge class by endpoint degrees (``fusion.py:77-85``)."""
    if g.edge(src, dst) is None:
        raise UnknownEdgeError(src, dst)
    if g.out_degree(src) > 1:
        return ConnKind.MULTI_OUTPUTS
    return ConnKind.MULTI_INPUTS if g.in_degree(dst) > 1 else ConnKind.DIRECT


def is_valid_conn(g: CompGraph, src: int, dst: int) -> bool:
    return classify_connection(g, src, dst) is not ConnKind.MULTI_OUTPUTS


def match_sequences(pred_seq, succ_seq, rules: FusionRuleSet) -> Match | None:
    """Strict-prefix matches beat full ones; lowest rule id (``fusion.py:93-104``)."""
    t = tuple(pred_seq) + tuple(succ_seq)
    n = len(t)
    pref = [r.id for r in rules if len(r.pattern) > n and r.pattern[:n] == t]
    if pref:
        return Match(MatchKind.PREFIX, min(pref))
    full = [r.id for r in rules if r.pattern == t]
    return Match(MatchKind.FULL, min(full)) if full else None


def match_rule(pred: OpNode, succ: OpNode, rules: FusionRuleSet) -> Match | None:
    return match_sequences(pred.type_seq, succ.type_seq, rules)


_TAG_CODE = {Tag.PLAIN: 0, Tag.FUSED: 1, Tag.BOUND: 2}
_CODE_TAG = {0: Tag.PLAIN, 1: Tag.FUSED, 2: Tag.BOUND}


_A_SEQ, _A_TAG, _A_MEM, _A_CT = (attrgetter("type_seq"), attrgetter("tag"), attrgetter("mem_bytes"),
                                  attrgetter("compute_time"))


class _NodeArrays:
    """Graph-intrinsic part of the flat coarsening input, cached on the (immutable)
    CompGraph: interned node type sequences (node types get the first ids, in node
    order — exactly as the per-call interning numbers them), tags, memory and the
    cost matrix over the devices the nodes name."""

    __slots__ = ("types", "seq_beg", "seq", "tag", "mem", "cost", "devices")

    def __init__(self, g: CompGraph):
        nodes = g.nodes
        V = len(nodes)
        seqs = list(map(_A_SEQ, nodes))
        flat_types = list(chain.from_iterable(seqs))
        self.types = {t: k for k, t in enumerate(dict.fromkeys(flat_types))}
        lens = np.fromiter(map(len, seqs), dtype=np.int32, count=V)
        self.seq_beg = np.zeros(V + 1, np.int32)
        np.cumsum(lens, out=self.seq_beg[1:])
        total = int(self.seq_beg[-1])
        self.seq = np.fromiter(map(self.types.__getitem__, flat_types), dtype=np.int32, count=total)
        self.tag = np.fromiter(map(_TAG_CODE.__getitem__, map(_A_TAG, nodes)), dtype=np.int32, count=V)
        self.mem = np.fromiter(map(_A_MEM, nodes), dtype=np.int64, count=V)
        cts = list(map(_A_CT, nodes))
        keys = list(map(tuple, cts))
        first = keys[0] if keys else ()
        uniform = keys.count(first) == len(keys)
        devs = set(first) if uniform else set().union(*cts)
        self.devices = sorted(devs)
        D = len(self.devices)
        if uniform and V and list(first) == self.devices:
            cost = np.fromiter(chain.from_iterable(map(dict.values, cts)), dtype=np.float64,
                               count=V * D).reshape(V, max(D, 1))
        else:
            dindex = {d: i for i, d in enumerate(self.devices)}
            cost = np.full((V, max(D, 1)), np.nan)
            for i, ct in enumerate(cts):
                for k, t in ct.items():
                    cost[i, dindex[k]] = float(t)
        self.cost = np.ascontiguousarray(cost)

    @classmethod
    def from_file_arrays(cls, a: dict, order: np.ndarray) -> "_NodeArrays":
        """The same arrays from the native reader's output (file order, ``order`` =
        ascending-id permutation), vectorised: no OpNode objects needed."""
        na = cls.__new__(cls)
        strs = a["strings"]
        V = len(order)
        sb = a["seq_beg"].astype(np.int64)
        lens = (sb[1:] - sb[:-1])[order]
        na.seq_beg = np.zeros(V + 1, np.int32)
        np.cumsum(lens, out=na.seq_beg[1:])
        total = int(na.seq_beg[-1])
        # flattened type sequences in ascending-id node order (string-table indices)
        starts = np.repeat(sb[:-1][order] - na.seq_beg[:-1], lens)
        flat = a["seq"].astype(np.int64)[np.arange(total) + starts] if total else np.zeros(0, np.int64)
        # type ids by first appearance (dict.fromkeys order of the object path)
        uniq, first = np.unique(flat, return_index=True)
        by_first = uniq[np.argsort(first, kind="stable")]
        na.types = {strs[int(x)]: k for k, x in enumerate(by_first.tolist())}
        remap = np.zeros(max(len(strs), 1), np.int32)
        remap[by_first] = np.arange(len(by_first), dtype=np.int32)
        na.seq = remap[flat].astype(np.int32) if total else np.zeros(0, np.int32)
        na.tag = a["tag"].astype(np.int32)[order]  # the reader's codes are _TAG_CODE's
        na.mem = a["mem"].astype(np.int64)[order]
        cdev = a["ct_dev"]
        na.devices = sorted(set(np.unique(cdev).tolist()))
        D = len(na.devices)
        cost = np.full((V, max(D, 1)), np.nan)
        if len(cdev):
            inv = np.empty(V, np.int64)
            inv[order] = np.arange(V)
            cb = a["ct_beg"].astype(np.int64)
            node_of = np.repeat(inv, cb[1:] - cb[:-1])
            col = np.searchsorted(np.asarray(na.devices, dtype=np.int64), cdev)
            cost[node_of, col] = a["ct_val"]
        na.cost = np.ascontiguousarray(cost)
        return na

    @staticmethod
    def of(g: CompGraph) -> "_NodeArrays":
        na = getattr(g, "_gcof_node_arrays", None)
        if na is None:
            na = _NodeArrays(g)
            g._gcof_node_arrays = na
        return na


class _Flat:
    """Array form of a coarsening problem (mp_coarsen_input)."""

    def __init__(self, g: CompGraph, rules: FusionRuleSet, overrides: CostOverrides | None):
        na = _NodeArrays.of(g)
        dg = g.csr()
        V = len(g)
        types = dict(na.types)
        for r in rules:
            for t in r.pattern:
                types.setdefault(t, len(types))
        if overrides is not None:
            for (sq, _k) in overrides.entries:
                for t in sq:
                    types.setdefault(t, len(types))
        total = int(na.seq_beg[-1])
        devices = na.devices
        cost = na.cost
        if overrides is not None:
            extra = sorted({k for (_, k) in overrides.entries} - set(devices))
            if extra:  # override-only devices: NaN columns (no member has a time there)
                devices = sorted(set(devices) | set(extra))
                full = np.full((V, len(devices)), np.nan)
                pos = [devices.index(d) for d in na.devices]
                if na.devices:
                    full[:, pos] = na.cost[:, :len(na.devices)]
                cost = full
        self.devices = devices
        dindex = {d: i for i, d in enumerate(self.devices)}
        D = len(self.devices)
        rb = np.zeros(len(rules) + 1, np.int32)
        rt = []
        rid = np.empty(len(rules), np.int32)
        for r, rule in enumerate(rules):
            rid[r] = rule.id
            rt.extend(types[t] for t in rule.pattern)
            rb[r + 1] = len(rt)
        ob = [0]
        ot = []
        odev = []
        otime = []
        if overrides is not None:
            for (sq, k), t in overrides.entries.items():
                ot.extend(types[x] for x in sq)
                ob.append(len(ot))
                odev.append(dindex[k])
                otime.append(float(t))
        self.keep = [
            dg.ids, na.seq_beg, na.seq if total else np.zeros(1, np.int32), na.tag, na.mem,
            np.ascontiguousarray(cost), dg.esrc, dg.edst, dg.payload, rid, rb, np.asarray(rt or [0], np.int32),
            np.asarray(ob, np.int32), np.asarray(ot or [0], np.int32), np.asarray(odev or [0], np.int32),
            np.asarray(otime or [0.0], np.float64),
        ]
        k = self.keep
        self.cin = N.mp_coarsen_input(
            V, len(dg.esrc), max(D, 1), N.ptr(k[0]), N.ptr(k[1]), N.ptr(k[2]), N.ptr(k[3]), N.ptr(k[4]),
            N.ptr(k[5]), N.ptr(k[6]), N.ptr(k[7]), N.ptr(k[8]), len(rules), N.ptr(k[9]), N.ptr(k[10]),
            N.ptr(k[11]), len(otime), N.ptr(k[12]), N.ptr(k[13]), N.ptr(k[14]), N.ptr(k[15]),
            1 if sys.version_info >= (3, 12) else 0)


# diagnostics of the last gcof call: ordered_replay = the graph had DFS-order
# hazards and the ordered replay ran (False: chains resolved in parallel)
LAST_GCOF: dict = {}


def gcof(g: CompGraph, rules: FusionRuleSet, overrides: CostOverrides | None = None,
         device: int = 0) -> CompGraph:
    """GCOF coarsening on the GPU (``fusion.py:271-304``).

    Same output as the reference, node by node (ids, op types, members, type
    sequences, tags, memory, fp64 costs bit for bit) and edge list order
    (sorted by ``(u, v)``); ``CycleError`` on cyclic input.
    """
    if len(g) == 0:
        return CompGraph([], [])
    with _bulk_objects():
        flat = _Flat(g, rules, overrides)
    out = N.mp_coarsen_output()
    err = N.mp_error()
    lib = N.lib()
    code = lib.mp_coarsen(C.byref(flat.cin), device, C.byref(out), C.byref(err))
    if code == N.MP_ERR_CYCLE:
        ids = g.node_ids
        raise CycleError(find_cycle(ids, {i: g.succs(i) for i in ids}))
    N.check(code, err, "mp_coarsen")
    LAST_GCOF["ordered_replay"] = bool(out.ordered_replay)
    try:
        # views of the native buffers (freed below, after the result no longer needs them;
        # everything kept is converted to lists / owned arrays while building it)
        ng, ne = out.n_groups, out.n_edges
        D = len(flat.devices)
        view = np.ctypeslib.as_array
        grp_tag = view(out.grp_tag, (ng,)) if ng else np.zeros(0, np.int32)
        mbeg = view(out.mem_beg, (ng + 1,))
        members = view(out.members, (int(mbeg[-1]),)) if mbeg[-1] else np.zeros(0, np.int32)
        gmem = view(out.grp_mem, (ng,)) if ng else np.zeros(0, np.int64)
        gcost = view(out.grp_cost, (ng * max(D, 1),)).reshape(ng, max(D, 1)) if ng else np.zeros((0, 1))
        esrc = view(out.out_src, (ne,)).copy() if ne else np.zeros(0, np.int32)
        edst = view(out.out_dst, (ne,)).copy() if ne else np.zeros(0, np.int32)
        epay = view(out.out_payload, (ne,)).copy() if ne else np.zeros(0, np.int64)
        return _gcof_result(g, flat, ng, D, mbeg, members, gmem, gcost, grp_tag, esrc, edst, epay)
    finally:
        lib.mp_coarsen_free(C.byref(out))


def _gcof_result(g, flat, ng, D, mbeg, members, gmem, gcost, grp_tag, esrc, edst, epay) -> CompGraph:
    """The coarsened CompGraph from the native output arrays (node by node as the
    reference builds it; unfused nodes are the input objects themselves).  The node
    ids and the edge arrays are ready at once; the OpNode objects are built on first
    use (the next stage — an Instance — reads the cost / memory arrays attached as
    ``_gcof_cost_arrays`` instead).  ``mbeg``..``grp_tag`` may be views of native
    buffers: everything kept is copied here."""
    ids_in = np.asarray(g.csr().ids)
    if ng:
        mb = np.array(mbeg[: ng + 1], dtype=np.int64)
        mem_idx = np.array(members[: int(mb[-1])], dtype=np.int64)
        ids = ids_in[np.minimum.reduceat(mem_idx, mb[:-1])]  # id = the smallest member id (int64 array)
    else:
        mb, mem_idx, ids = np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64)
    cost = np.array(gcost, dtype=np.float64).reshape(ng, max(D, 1))
    gmem_c = np.array(gmem, dtype=np.int64)
    tag_c = np.array(grp_tag, dtype=np.int32)
    devices = flat.devices

    def build() -> dict:
        with _bulk_objects():
            return _gcof_nodes(g.nodes, ng, D, devices, mb, mem_idx, gmem_c, cost, tag_c)

    out = CompGraph._from_lazy(ids, build, esrc, edst, epay)
    out._gcof_cost_arrays = (devices, cost, gmem_c)
    return out


def _gcof_nodes(nodes_in, ng, D, devices, mbeg, members, gmem, gcost, grp_tag) -> dict:
    """{id: OpNode} of the coarsened graph (fusion.py:221-240 node by node)."""
    new_nodes = {}
    mb = mbeg.tolist()
    mlist = members.tolist()
    cost_rows = gcost.tolist()
    partial = np.isnan(gcost).any(axis=1).tolist() if ng else []  # a device some member lacks
    mem_l = gmem.tolist()
    tag_l = grp_tag.tolist()
    join = FUSE_JOINER.join
    tags = [_CODE_TAG[c] for c in range(3)]
    op_types: dict = {}  # fused type sequences repeat (one per layer kind): join once
    new = object.__new__
    setattr_ = object.__setattr__  # OpNode is frozen: install its __dict__ in one call
    for z in range(ng):
        b, e = mb[z], mb[z + 1]
        if e - b == 1:
            n = nodes_in[mlist[b]]
            new_nodes[n.id] = n
            continue
        if e - b == 2:
            p0, p1 = nodes_in[mlist[b]], nodes_in[mlist[b + 1]]
            seq = p0.type_seq + p1.type_seq
            mids = p0.members + p1.members
            gid = p0.id if p0.id < p1.id else p1.id
        else:
            idx = mlist[b:e]
            parts = [nodes_in[m] for m in idx]
            seq = tuple(chain.from_iterable([p.type_seq for p in parts]))
            mids = tuple(chain.from_iterable([p.members for p in parts]))
            # nodes_in is in ascending id order: the smallest member index has the smallest id
            gid = nodes_in[min(idx)].id
        row = cost_rows[z]
        cost = ({devices[k]: row[k] for k in range(D) if row[k] == row[k]} if partial[z]
                else dict(zip(devices, row)))
        ot = op_types.get(seq)
        if ot is None:
            ot = op_types[seq] = join(seq)
        n = new(OpNode)
        setattr_(n, "__dict__", {"id": gid, "op_type": ot, "mem_bytes": mem_l[z], "compute_time": cost,
                                 "members": mids, "type_seq": seq, "tag": tags[tag_l[z]]})
        new_nodes[gid] = n
    return new_nodes


def _combined_cost(parts, seq, overrides):
    """Per-device time of a fused node (``fusion.py:117-130``): override, else
    the builtin ``sum`` of the member times in member order."""
    common = set(parts[0].compute_time)
    for p in parts[1:]:
        common &= set(p.compute_time)
    devices = set(common)
    if overrides is not None:
        devices |= overrides.devices_for(seq)
    cost = {}
    for k in sorted(devices):
        ov = overrides.get(seq, k) if overrides is not None else None
        cost[k] = ov if ov is not None else sum(p.compute_time[k] for p in parts)
    return cost


def fuse(g: CompGraph, pred: int, succ: int, overrides: CostOverrides | None = None) -> tuple[CompGraph, OpNode]:
    """Fuse one edge (``fusion.py:251-268``): the merged node (id = min of the
    two, members / type sequence concatenated pred first, memory summed, costs
    summed or overridden, tag FUSED) takes the union of both endpoints' external
    edges; the edge list comes back sorted by ``(u, v)`` as the reference's
    ``materialize``.  ``UnknownEdgeError`` when the edge is missing,
    ``CycleCreationError`` when another pred ~> succ path would close a cycle.
    A single graph edit, not a data-parallel path: it runs on the host."""
    if g.edge(pred, succ) is None:
        raise UnknownEdgeError(pred, succ)
    validate_dag(g)
    frontier = [n for n in g.succs(pred) if n != succ]
    seen = set(frontier)
    while frontier:
        n = frontier.pop()
        if n == succ:
            raise CycleCreationError(pred, succ)
        for m in g.succs(n):
            if m not in seen:
                seen.add(m)
                frontier.append(m)
    a, b = g.node(pred), g.node(succ)
    seq = a.type_seq + b.type_seq
    gid = min(pred, succ)
    merged = OpNode(gid, FUSE_JOINER.join(seq), a.mem_bytes + b.mem_bytes, _combined_cost([a, b], seq, overrides),
                    a.members + b.members, seq, Tag.FUSED)
    nodes = [merged if n.id == gid else n for n in g.nodes if n.id not in (pred, succ) or n.id == gid]
    where = {pred: gid, succ: gid}
    payload: dict[tuple[int, int], int] = {}
    for e in g.edges:
        gu, gv = where.get(e.src, e.src), where.get(e.dst, e.dst)
        if gu != gv:
            payload[(gu, gv)] = payload.get((gu, gv), 0) + e.payload_bytes
    out = CompGraph(sorted(nodes, key=lambda n: n.id), [FlowEdge(u, v, payload[(u, v)]) for (u, v) in sorted(payload)])
    return out, out.node(gid)
