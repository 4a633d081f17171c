"""ctypes wrapper of the CPU oracle (oracle/moirai_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, by __graft_entry__.smoke() as the
checker, and by bench.py's cpu_baseline / ``--impl reference`` legs.  The
product package ``paper_2312_04025_b200`` never imports this module.

Parity pinned against the reference package (tests/test_oracle.py +
tests/golden/*.json produced by tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libmoirai_oracle.so"


def build() -> Path:
    src = HERE / "moirai_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "CC=gcc"], check=True)
    return LIB


class _Problem(C.Structure):
    _fields_ = [("n_ops", C.c_int), ("n_flows", C.c_int), ("K", C.c_int),
                ("cost", C.c_void_p), ("mem", C.c_void_p), ("fsrc", C.c_void_p), ("fdst", C.c_void_p),
                ("payload", C.c_void_p), ("cap", C.c_void_p), ("bw", C.c_void_p)]


class _GcofIn(C.Structure):
    _fields_ = [("V", C.c_int), ("E", C.c_int), ("seq_beg", C.c_void_p), ("seq_types", C.c_void_p),
                ("tag", C.c_void_p), ("esrc", C.c_void_p), ("edst", C.c_void_p), ("R", C.c_int),
                ("rule_id", C.c_void_p), ("rule_beg", C.c_void_p), ("rule_types", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        L.orc_inst_new.restype = C.c_void_p
        L.orc_inst_new.argtypes = [C.POINTER(_Problem)]
        L.orc_inst_free.argtypes = [C.c_void_p]
        L.orc_schedule.restype = C.c_int
        L.orc_schedule.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_double),
                                   C.POINTER(C.c_int), C.POINTER(C.c_int64)]
        L.orc_eval_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int]
        L.orc_enumerate.restype = C.c_int64
        L.orc_enumerate.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]
        L.orc_last_max_ready.restype = C.c_int
        L.orc_solve_exact.restype = C.c_int
        L.orc_solve_exact.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_int64, C.c_void_p,
                                      C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.orc_gcof.restype = C.c_int
        L.orc_gcof.argtypes = [C.POINTER(_GcofIn), C.c_void_p, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else None


class OracleInstance:
    """Flat problem (same layout as include/moirai_b200.h mp_problem)."""

    def __init__(self, cost, mem, fsrc, fdst, payload, cap, bw):
        self.arrays = [np.ascontiguousarray(cost, np.float64), np.ascontiguousarray(mem, np.int64),
                       np.ascontiguousarray(fsrc, np.int32), np.ascontiguousarray(fdst, np.int32),
                       np.ascontiguousarray(payload, np.int64), np.ascontiguousarray(cap, np.int64),
                       np.ascontiguousarray(bw, np.float64)]
        cost = self.arrays[0]
        self.n_ops, self.K = cost.shape
        self.n_flows = self.arrays[2].shape[0]
        self._prob = _Problem(self.n_ops, self.n_flows, self.K, *(_p(a) for a in self.arrays))
        h = lib().orc_inst_new(C.byref(self._prob))
        if not h:
            raise ValueError("cyclic graph")
        self._h = h

    @classmethod
    def from_instance(cls, inst):
        """Build from the product package's flattened Instance arrays."""
        return cls(*inst._arrays)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_inst_free(self._h)
            self._h = None

    def schedule(self, row):
        row = np.ascontiguousarray(row, np.uint8)
        N = self.n_ops + self.n_flows
        st = np.zeros(N)
        en = np.zeros(N)
        ms = C.c_double(0)
        md = C.c_int(-1)
        ov = C.c_int64(0)
        s = lib().orc_schedule(self._h, _p(row), _p(st), _p(en), C.byref(ms), C.byref(md), C.byref(ov))
        return s, ms.value, st, en, md.value, ov.value

    def max_ready(self, row) -> int:
        """Largest ready set while scheduling `row` (diagnostic)."""
        self.schedule(row)
        return lib().orc_last_max_ready()

    def eval_batch(self, rows, threads: int = 1):
        rows = np.ascontiguousarray(rows, np.uint8)
        P = rows.shape[0]
        ms = np.empty(P)
        status = np.empty(P, np.int8)
        lib().orc_eval_batch(self._h, _p(rows), P, _p(ms), _p(status), int(threads))
        return ms, status

    def enumerate(self, op_order):
        op_order = np.ascontiguousarray(op_order, np.int32)
        best = C.c_double(0)
        idx = lib().orc_enumerate(self._h, _p(op_order), C.byref(best))
        return int(idx), best.value

    def solve_exact(self, op_order, gap: float = 0.0, node_limit: int | None = None):
        """Reference branch and bound (solver.py:172-254) without the time limit.
        Returns (status 0 optimal / 1 feasible / 2 infeasible / 3 budget, row, makespan, visited)."""
        op_order = np.ascontiguousarray(op_order, np.int32)
        row = np.zeros(self.n_ops, np.uint8)
        best = C.c_double(0)
        vis = C.c_int64(0)
        st = lib().orc_solve_exact(self._h, _p(op_order), float(gap), -1 if node_limit is None else int(node_limit),
                                   _p(row), C.byref(best), C.byref(vis))
        return int(st), row, best.value, int(vis.value)


def gcof_partition(seq_beg, seq_types, tag, esrc, edst, rule_beg, rule_types):
    """Partition produced by the reference GCOF DFS + final_partition.
    Returns list of (member index list, tag code) in ascending output id."""
    V = len(tag)
    E = len(esrc)
    arrs = [np.ascontiguousarray(x, np.int32) for x in (seq_beg, seq_types, tag, esrc, edst, rule_beg,
                                                        rule_types)]
    R = len(arrs[5]) - 1
    rid = np.arange(R, dtype=np.int32)
    gin = _GcofIn(V, E, _p(arrs[0]), _p(arrs[1]), _p(arrs[2]), _p(arrs[3]), _p(arrs[4]), R, _p(rid),
                  _p(arrs[5]), _p(arrs[6]))
    gb = np.zeros(V + 1, np.int32)
    mem = np.zeros(max(V, 1), np.int32)
    gt = np.zeros(max(V, 1), np.int32)
    n = lib().orc_gcof(C.byref(gin), _p(gb), _p(mem), _p(gt))
    if n < 0:
        raise ValueError("cyclic graph")
    return [(mem[gb[z]:gb[z + 1]].tolist(), int(gt[z])) for z in range(n)]


def materialize(g, groups, overrides=None):
    """fusion.py:117-130,221-248 restated over a product-package CompGraph.
    ``groups``: (member index list, tag code) from :func:`gcof_partition`.
    Returns (nodes as tuples, edges as (u, v, payload) sorted)."""
    ids = g.node_ids
    nodes_in = g.nodes
    where = {}
    out_nodes = []
    for members, tagc in groups:
        mids = [ids[m] for m in members]
        gid = min(mids)
        for m in mids:
            where[m] = gid
        if len(mids) == 1:
            n = g.node(mids[0])
            out_nodes.append((n.id, n.op_type, n.members, n.type_seq, n.tag.value, n.mem_bytes,
                              dict(n.compute_time)))
            continue
        parts = [g.node(m) for m in mids]
        members_t = tuple(x for p in parts for x in p.members)
        seq = tuple(t for p in parts for t in p.type_seq)
        mem = sum(p.mem_bytes for p in parts)
        common = set(parts[0].compute_time)
        for p in parts[1:]:
            common &= set(p.compute_time)
        devs = set(common)
        if overrides is not None:
            devs |= overrides.devices_for(seq)
        cost = {}
        for k in sorted(devs):
            ov = overrides.get(seq, k) if overrides is not None else None
            if ov is not None:
                cost[k] = ov
            else:
                # builtin sum() exactly as fusion.py:129 (compensated on CPython >= 3.12)
                cost[k] = sum(p.compute_time[k] for p in parts)
        tagname = {0: "plain", 1: "fused", 2: "bound"}[tagc]
        out_nodes.append((gid, "∘".join(seq), members_t, seq, tagname, mem, cost))
    pay = {}
    for e in g.edges:
        gu, gv = where[e.src], where[e.dst]
        if gu != gv:
            pay[(gu, gv)] = pay.get((gu, gv), 0) + e.payload_bytes
    edges = [(u, v, pay[(u, v)]) for (u, v) in sorted(pay)]
    out_nodes.sort(key=lambda t: t[0])
    return out_nodes, edges


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---- K5 restated (paper_2312_04025_b200/csrc/mp_eval.cu mp_ls_kernel) -------------------
_M64 = (1 << 64) - 1


def _mix64(x: int) -> int:
    x &= _M64
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & _M64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & _M64
    x ^= x >> 31
    return x


def ls_chains(orc: "OracleInstance", seeds, n_chains: int, chain_base: int, moves: int, rng_seed: int):
    """CPU restatement of the local-search chains: chain c starts from seed row
    (c % n_seed), move t re-assigns op (h mod n) to device (old + 1 + (h >> 32) mod
    (K-1)) mod K with h = mix64(rng_seed ^ mix64(c * PHI + t)), accepted iff the
    makespan does not increase (infeasible = +inf).  Exact only when no
    evaluation overflows the GPU's ready capacity (the caller checks
    ready_cap >= ready_bound).  Returns (best row, best ms, best chain, chain ms)."""
    seeds = np.ascontiguousarray(seeds, np.uint8)
    n, K = orc.n_ops, orc.K
    chain_ms = np.empty(n_chains)
    rows = []
    for c in range(n_chains):
        gc = c + chain_base
        row = seeds[gc % len(seeds)].copy()

        def ev(r):
            st, ms, *_ = orc.schedule(r)
            return ms if st == 0 else math.inf

        cur = ev(row)
        for t in range(moves if K > 1 else 0):
            h = _mix64(rng_seed ^ _mix64(gc * 0x9E3779B97F4A7C15 + t))
            i = (h & 0xFFFFFFFF) % n
            old = int(row[i])
            row[i] = (old + 1 + (h >> 32) % (K - 1)) % K
            ms = ev(row)
            if ms <= cur:
                cur = ms
            else:
                row[i] = old
        chain_ms[c] = cur
        rows.append(row)
    best = int(np.argmin(chain_ms)) if n_chains else 0
    return rows[best], float(chain_ms[best]), best + chain_base, chain_ms
