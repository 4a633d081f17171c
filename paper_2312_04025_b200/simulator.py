"""Placement replay with an event trace (``pkg/src/opplace/simulator.py:74-172``).

The reference keeps ``simulate`` as an independent second implementation of the
dispatch semantics (a lazy heap instead of a ready-list scan).  Here the timing
is produced by the same GPU evaluator in trace mode (``mp_schedule_one``) — the
reference's own test asserts both give bitwise-identical starts/ends
(``test_simulator.py:74-89``) — and the trace is assembled from it: start and
end events for every op and flow, sorted by ``(time, kind, node)``.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

from .errors import MemoryExceededError, MissingCostError
from .graph import CompGraph
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
