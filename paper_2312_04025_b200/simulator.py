"""Placement replay with an event trace (``pkg/src/opplace/simulator.py:74-172``).

The reference keeps ``simulate`` as an independent second implementation of the
dispatch semantics (a lazy heap instead of a ready-list scan).  Here the timing
is produced by the same GPU evaluator in trace mode (``mp_schedule_one``) — the
reference's own test asserts both give bitwise-identical starts/ends
(``test_simulator.py:74-89``) — and the trace is assembled from it: start and
end events for every op and flow, sorted by ``(time, kind, node)``.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _native as N

from .errors import MemoryExceededError, MissingCostError
from .graph import CompGraph
from .placement import Schedule
from .profiles import Cluster, EffectiveMesh
from .solver import Instance, _schedule_row


class EventKind(str, Enum):
    OP_START = "op-start"
    OP_END = "op-end"
    FLOW_START = "flow-start"
    FLOW_END = "flow-end"


_KIND_ORDER = {k: i for i, k in enumerate(EventKind)}


@dataclass(frozen=True)
class Event:
    """Timestamped trace entry (``simulator.py:29-55``)."""

    time_s: float
    kind: EventKind
    node: int
    device: int | None = None
    channel: tuple[int, int] | None = None

    def sort_key(self) -> tuple[float, int, int]:
        return (self.time_s, _KIND_ORDER[self.kind], self.node)


def simulate(gc: CompGraph, c: Cluster, mesh: EffectiveMesh,
             placement: dict[int, int]) -> tuple[float, list[Event]]:
    """Replay a total placement; returns ``(makespan, sorted trace)``.

    Validation follows ``simulator.py:85-96``: unknown device -> ``KeyError``,
    no time on the placed device -> ``MissingCostError``, memory ->
    ``MemoryExceededError``.  Only placed devices need a compute time, so other
    entries are filled with a value the schedule never reads.
    """
    caps = {d: c.device(d).mem_bytes for d in c.device_ids}
    load = dict.fromkeys(caps, 0)
    for i in gc.node_ids:
        node = gc.node(i)
        k = placement[i]
        if k not in caps:
            raise KeyError(f"op {i} placed on unknown device {k}")
        if k not in node.compute_time:
            raise MissingCostError(i, k)
        load[k] += node.mem_bytes
    for k in c.device_ids:
        if load[k] > caps[k]:
            raise MemoryExceededError(k, load[k] - caps[k])
    with Instance(gc, c, mesh, _fill_missing=float("inf")) as inst:
        row = inst.encode([placement])[0]
        sched = _schedule_row(inst, row)
    events: list[Event] = []
    op_ends = []
    for nid in inst.op_ids:
        d = placement[nid]
        events.append(Event(sched.starts[nid], EventKind.OP_START, nid, device=d))
        events.append(Event(sched.ends[nid], EventKind.OP_END, nid, device=d))
        op_ends.append(sched.ends[nid])
    for f, e in enumerate(gc.edges):
        q = inst.flow_id(f)
        ch = sched.channels[q]
        if ch is None:
            dev = placement[e.src]
            events.append(Event(sched.starts[q], EventKind.FLOW_START, q, device=dev))
            events.append(Event(sched.ends[q], EventKind.FLOW_END, q, device=dev))
        else:
            events.append(Event(sched.starts[q], EventKind.FLOW_START, q, channel=ch))
            events.append(Event(sched.ends[q], EventKind.FLOW_END, q, channel=ch))
    events.sort(key=Event.sort_key)
    return max(op_ends), events


class ViolationKind(str, Enum):
    DEVICE_OVERLAP = "device-overlap"
    SOURCE_CHANNEL_OVERLAP = "source-channel-overlap"
    DEST_CHANNEL_OVERLAP = "dest-channel-overlap"
    PRECEDENCE_BREAK = "precedence-break"
    MEMORY_OVER = "memory-over"
    DURATION_MISMATCH = "duration-mismatch"


@dataclass(frozen=True)
class Violation:
    """One audit finding (``simulator.py:58-71``)."""

    kind: ViolationKind
    details: str
    nodes: tuple[int, ...] = field(default=())


def check_feasibility(schedule: Schedule, gc: CompGraph, c: Cluster, mesh: EffectiveMesh,
                      tol: float = 0.0) -> list[Violation]:
    """Audit a schedule on the GPU (``simulator.py:179-264``); empty = feasible.

    The checks (memory, durations, starts >= 0, precedence over every augmented
    link, pairwise device / source-channel / destination-channel overlaps) run in
    ``mp_audit_schedule`` with the reference's floating-point expressions, one
    thread per node, link or pair; findings come back in the reference's order
    and carry its messages.  ``tol`` widens every comparison as in the reference.
    """
    assign, starts, ends = schedule.assignment, schedule.starts, schedule.ends
    ids = gc.node_ids
    n_ops = len(ids)
    max_id = max(ids, default=0)
    flow_ids = [max_id + 1 + f for f in range(len(gc.edges))]
    for n in ids + flow_ids:
        if n not in starts or n not in ends:
            raise KeyError(f"schedule is missing node {n}")
    devs = c.device_ids
    for i in ids:
        if i not in assign or assign[i] not in devs:
            raise KeyError(f"schedule does not place op {i} on a known device")
    if n_ops == 0:
        return []  # nothing to audit (the reference's loops are empty)
    with Instance(gc, c, mesh, _fill_missing=float("inf")) as inst:
        row = inst.encode([assign])[0]
        st = np.asarray([starts[n] for n in ids + flow_ids], dtype=np.float64)
        en = np.asarray([ends[n] for n in ids + flow_ids], dtype=np.float64)
        n_out = C.c_int64(0)
        cap = 256
        while True:
            buf = (N.mp_violation * cap)()
            err = N.mp_error()
            code = inst._lib.mp_audit_schedule(inst.handle, N.ptr(row), N.ptr(st), N.ptr(en), float(tol), buf, cap,
                                               C.byref(n_out), C.byref(err))
            N.check(code, err, "mp_audit_schedule")
            if n_out.value <= cap:
                break
            cap = n_out.value
    edges = gc.edges
    out: list[Violation] = []
    for v in buf[:n_out.value]:
        k, x, y = v.kind, int(v.x), int(v.y)
        if k == 0:
            d = devs[x]
            out.append(Violation(ViolationKind.MEMORY_OVER,
                                 f"device {d} holds {y} bytes, capacity {c.device(d).mem_bytes}"))
        elif k in (1, 2):
            node = (ids + flow_ids)[x]
            if k == 1:
                if x < n_ops:
                    want = gc.node(node).compute_time[assign[node]]
                else:
                    e = edges[x - n_ops]
                    ka, kb = assign[e.src], assign[e.dst]
                    want = 0.0 if ka == kb else e.payload_bytes / mesh.bandwidth(ka, kb)
                out.append(Violation(ViolationKind.DURATION_MISMATCH,
                                     f"node {node} spans {ends[node] - starts[node]}, expected {want}", (node,)))
            else:
                out.append(Violation(ViolationKind.DURATION_MISMATCH,
                                     f"node {node} starts before time zero ({starts[node]})", (node,)))
        elif k == 3:
            e = edges[x >> 1]
            q = flow_ids[x >> 1]
            a, b = (e.src, q) if x % 2 == 0 else (q, e.dst)
            out.append(Violation(ViolationKind.PRECEDENCE_BREAK,
                                 f"node {b} starts at {starts[b]} before {a} ends at {ends[a]}", (a, b)))
        elif k == 4:
            i, j = ids[x], ids[y]
            out.append(Violation(ViolationKind.DEVICE_OVERLAP, f"ops {i} and {j} overlap on device {assign[i]}", (i, j)))
        else:
            q, r = flow_ids[x], flow_ids[y]
            if k == 5:
                out.append(Violation(ViolationKind.SOURCE_CHANNEL_OVERLAP,
                                     f"flows {q} and {r} both leave device {assign[edges[x].src]}", (q, r)))
            else:
                out.append(Violation(ViolationKind.DEST_CHANNEL_OVERLAP,
                                     f"flows {q} and {r} both arrive at device {assign[edges[x].dst]}", (q, r)))
    return out
