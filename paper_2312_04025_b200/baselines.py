"""Greedy placement baselines on the GPU (``pkg/src/opplace/baselines.py:27-86``).

``greedy_place`` keeps the reference's signature, scoring and tie rules: ops in
``topo_order(gc)``, each committed to the device with the smallest
``(score, device id)`` where the score is the op's earliest finish (or start)
with its in-flows timed in flow order against the committed channel clocks.
The choice runs as one warp (``mp_greedy_place``: lane k scores device k), the
final timing is the exact schedule of the chosen assignment
(``mp_schedule_one``), as the reference's closing ``_schedule`` call.  The
rows double as local-search / branch-and-bound seeds.
"""

from __future__ import annotations

import ctypes as C
from enum import Enum

import numpy as np

from . import _native as N
from .graph import CompGraph, topo_order
from .placement import Schedule
from .profiles import Cluster, EffectiveMesh
from .solver import Instance, _schedule_row


class BaselineKind(str, Enum):
    EARLIEST_FINISH = "earliest-finish"
    EARLIEST_START = "earliest-start"


def greedy_row(inst: Instance, kind: BaselineKind = BaselineKind.EARLIEST_FINISH) -> np.ndarray:
    """The greedy assignment as a placement row (uint8 device indices)."""
    kind = BaselineKind(kind)
    pos = {nid: i for i, nid in enumerate(inst.op_ids)}
    op_order = np.asarray([pos[x] for x in topo_order(inst.gc)], dtype=np.int32)
    row = np.zeros(inst.n_ops, dtype=np.uint8)
    err = N.mp_error()
    code = inst._lib.mp_greedy_place(inst.handle, N.ptr(op_order), 0 if kind is BaselineKind.EARLIEST_FINISH else 1,
                                     N.ptr(row), C.byref(err))
    N.check(code, err, "mp_greedy_place")
    return row


def greedy_place(gc: CompGraph, c: Cluster, mesh: EffectiveMesh,
                 kind: BaselineKind = BaselineKind.EARLIEST_FINISH) -> Schedule:
    """Single-pass greedy placement; raises ``InfeasibleMemoryError`` when no
    device can hold the next op (``baselines.py:75-77``)."""
    with Instance(gc, c, mesh) as inst:
        return _schedule_row(inst, greedy_row(inst, kind))
