"""Pure-Python restatement of the reference evaluation loop — the CPU reference arm.

TEST / BASELINE INFRASTRUCTURE ONLY (see oracle/oracle.py header).

The reference (`opplace`) is pure Python and is not available on the GPU box,
so bench.py's ``--impl reference`` and ``cpu_baseline`` legs time this
restatement instead.  It keeps the reference's data structures — dicts keyed
by node id, a Python list as the ready set scanned with tuple keys — so its
cost per evaluation tracks the reference's (tests/test_pyref.py pins its
results to the golden vectors; DESIGN.md §6 records its speed against the real
package in this container).

    Instance  ~ solver.py:42-77  (_Instance; flattened from the product's arrays)
    schedule  ~ solver.py:80-148 (_schedule), returns the makespan or raises
    MemoryExceeded
"""

from __future__ import annotations

import os
import time


class MemoryExceeded(Exception):
    def __init__(self, device, overflow):
        self.device, self.overflow = device, overflow


class Instance:
    """Shared tables of one problem, built once (the `_Instance` role)."""

    def __init__(self, cost, mem, esrc, edst, payload, cap, bw):
        n, K = len(cost), len(cap)
        self.devices = list(range(K))
        self.ops = list(range(n))
        self.flows = list(range(n, n + len(esrc)))
        self.flow_set = set(self.flows)
        self.cap = {k: int(cap[k]) for k in self.devices}
        self.mem = {i: int(mem[i]) for i in self.ops}
        self.p = {i: {k: float(cost[i][k]) for k in self.devices} for i in self.ops}
        self.fsrc = {n + f: int(esrc[f]) for f in range(len(esrc))}
        self.fdst = {n + f: int(edst[f]) for f in range(len(edst))}
        self.payload = {n + f: int(payload[f]) for f in range(len(payload))}
        self.bw = {(a, b): float(bw[a][b]) for a in self.devices for b in self.devices if a != b}
        succ = {x: [] for x in self.ops + self.flows}
        pred = {x: [] for x in self.ops + self.flows}
        for q in self.flows:
            succ[self.fsrc[q]].append(q)
            pred[q].append(self.fsrc[q])
            succ[q].append(self.fdst[q])
            pred[self.fdst[q]].append(q)
        self.succs, self.preds = succ, pred
        # a topological order of the augmented graph (Kahn)
        indeg = {x: len(pred[x]) for x in succ}
        order = [x for x in sorted(succ) if indeg[x] == 0]
        head = 0
        while head < len(order):
            x = order[head]
            head += 1
            for y in succ[x]:
                indeg[y] -= 1
                if indeg[y] == 0:
                    order.append(y)
        self.topo = order
        self.rev_topo = order[::-1]

    @classmethod
    def from_arrays(cls, arrays):
        cost, mem, esrc, edst, payload, cap, bw = arrays
        return cls(cost.tolist(), mem.tolist(), esrc.tolist(), edst.tolist(), payload.tolist(), cap.tolist(),
                   bw.tolist())


def schedule(inst: Instance, assign: dict) -> float:
    """List-schedule one assignment {op index: device index}; returns the makespan."""
    load = dict.fromkeys(inst.devices, 0)
    for i in inst.ops:
        load[assign[i]] += inst.mem[i]
    for k in inst.devices:
        if load[k] > inst.cap[k]:
            raise MemoryExceeded(k, load[k] - inst.cap[k])
    dur = {}
    chan = {}
    for i in inst.ops:
        dur[i] = inst.p[i][assign[i]]
    for q in inst.flows:
        ka, kb = assign[inst.fsrc[q]], assign[inst.fdst[q]]
        if ka == kb:
            dur[q] = 0.0
            chan[q] = None
        else:
            dur[q] = inst.payload[q] / inst.bw[(ka, kb)]
            chan[q] = (ka, kb)
    rank = {}
    for x in inst.rev_topo:
        top = 0.0
        for y in inst.succs[x]:
            if rank[y] > top:
                top = rank[y]
        rank[x] = dur[x] + top
    npred = {x: len(inst.preds[x]) for x in inst.topo}
    est = dict.fromkeys(inst.topo, 0.0)
    ready = [x for x in inst.topo if npred[x] == 0]
    op_free = dict.fromkeys(inst.devices, 0.0)
    out_free = dict.fromkeys(inst.devices, 0.0)
    in_free = dict.fromkeys(inst.devices, 0.0)
    ends = {}
    while ready:
        pick = None
        for x in ready:
            if x in inst.flow_set:
                c = chan[x]
                e = est[x] if c is None else max(est[x], out_free[c[0]], in_free[c[1]])
            else:
                e = max(est[x], op_free[assign[x]])
            key = (e, -rank[x], x)
            if pick is None or key < pick:
                pick = key
        e, _, x = pick
        end = e + dur[x]
        ends[x] = end
        if x in inst.flow_set:
            c = chan[x]
            if c is not None:
                out_free[c[0]] = end
                in_free[c[1]] = end
        else:
            op_free[assign[x]] = end
        ready.remove(x)
        for y in inst.succs[x]:
            npred[y] -= 1
            if est[y] < end:
                est[y] = end
            if npred[y] == 0:
                ready.append(y)
    return max(ends[i] for i in inst.ops)


def eval_rows(inst: Instance, rows) -> list:
    out = []
    for row in rows:
        assign = {i: int(k) for i, k in enumerate(row)}
        try:
            out.append(schedule(inst, assign))
        except MemoryExceeded:
            out.append(float("inf"))
    return out


# ---- multi-process timing (the reference arm uses every host core) ------------------
_G = {}


def _worker_init(arrays):
    _G["inst"] = Instance.from_arrays(arrays)


def _worker_rows(rows):
    return eval_rows(_G["inst"], rows)


def time_all_cores(arrays, rows, processes: int | None = None):
    """Evaluate `rows` across `processes` forked workers (one Instance each,
    built outside the timer); returns (seconds, makespans, processes)."""
    import multiprocessing as mpc

    procs = processes or os.cpu_count() or 1
    chunks = [rows[i::procs] for i in range(procs)]
    ctx = mpc.get_context("fork")
    with ctx.Pool(procs, initializer=_worker_init, initargs=(arrays,)) as pool:
        pool.map(_worker_rows, [c[:1] for c in chunks])  # warm every worker
        t0 = time.perf_counter()
        parts = pool.map(_worker_rows, chunks)
        dt = time.perf_counter() - t0
    ms = [None] * len(rows)
    for i, part in enumerate(parts):
        for j, v in enumerate(part):
            ms[i + j * procs] = v
    return dt, ms, procs
