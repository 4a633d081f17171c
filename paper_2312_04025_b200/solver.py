"""Placement evaluation and search on the GPU — the drop-in solver surface.

Reference: ``pkg/src/opplace/solver.py``.  The public names keep their
signatures and error behaviour:

* :func:`schedule_for_assignment` (``solver.py:151-165``) — one exact schedule,
  computed by the evaluator kernel in trace mode (``mp_schedule_one``).
* :func:`brute_force` (``solver.py:257-282``) — enumerate every assignment on
  the GPU (``mp_enumerate_argmin``), same digit order and first-strict-minimum
  tie rule, then rebuild the winning schedule.
* :func:`solve_exact` (``solver.py:172-254``) — see its docstring.

New batched entry points (no reference analogue; they expose the data-parallel
loop the reference runs one ``_schedule`` at a time):
:class:`Instance`, :func:`evaluate_batch`, :func:`argmin`, :func:`local_search`.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import CycleError, DeviceLimitError, MemoryExceededError, MissingCostError, TooLargeError
from .graph import CompGraph, find_cycle, topo_order
from .placement import Schedule, Solution, Status
from .profiles import Cluster, EffectiveMesh, effective_bandwidth


@dataclass
class SolveBudget:
    """Limits for :func:`solve_exact` (``solver.py:29-39``)."""

    time_limit_s: float | None = None
    gap: float = 0.0
    node_limit: int | None = None

    def __post_init__(self):
        if not 0.0 <= self.gap < 1.0:
            raise ValueError("gap must be in [0, 1)")


class Instance:
    """A placement problem resident on one GPU (``_Instance``, ``solver.py:42-77``).

    Flattening: op index = rank of the op id (ascending), flow index = edge
    order, device index = rank of the device id.  Validation order matches the
    reference: empty graph, then missing costs (first op, then first device, in
    ascending order), then cycles.

    Departures: clusters of more than 16 devices raise
    :class:`DeviceLimitError` before anything is built; a NaN compute time raises
    ``ValueError`` (the reference accepts NaN, ``graph.py:59-61`` checks ``t < 0``
    only, but its dispatch order is then defined by NaN comparisons of Python
    tuples; this package does not restate that).
    """

    MAX_DEVICES = 16  # csrc/mp_common.cuh MP_MAX_DEV

    def __init__(self, gc: CompGraph, c: Cluster, mesh: EffectiveMesh, device: int = 0,
                 _fill_missing: float | None = None):
        if len(gc) == 0:
            raise ValueError("cannot place an empty graph")
        if len(c.device_ids) > self.MAX_DEVICES:
            raise DeviceLimitError(len(c.device_ids), self.MAX_DEVICES)
        self.gc, self.cluster, self.mesh = gc, c, mesh
        self.device_ids = c.device_ids
        self.dev_index = {d: k for k, d in enumerate(self.device_ids)}
        dg = gc.csr()
        self.dense = dg
        self.op_ids = [int(x) for x in dg.ids]
        K = len(self.device_ids)
        n = len(self.op_ids)
        fast = getattr(gc, "_gcof_cost_arrays", None)  # a GCOF output: its cost / memory arrays
        if fast is not None:
            devs, gcost, gmem = fast
            col = {d: k for k, d in enumerate(devs)}
            # NaN marks a device some member lacks; any NaN (or an unknown device) takes the
            # object path below, which reports it exactly as the reference does
            if all(d in col for d in self.device_ids) and not np.isnan(gcost).any():
                cost = np.ascontiguousarray(gcost[:, [col[d] for d in self.device_ids]])
                mem = gmem
            else:
                fast = None
        if fast is None:
            cost = np.empty((n, K), dtype=np.float64)
            for i, nid in enumerate(self.op_ids):
                ct = gc.node(nid).compute_time
                for k, dev in enumerate(self.device_ids):
                    t = ct.get(dev)
                    if t is None:
                        if _fill_missing is None:
                            raise MissingCostError(nid, dev)
                        t = _fill_missing
                    cost[i, k] = t
            if np.isnan(cost).any():
                i, k = map(int, np.argwhere(np.isnan(cost))[0])
                raise ValueError(f"op {self.op_ids[i]} has a NaN compute time on device {self.device_ids[k]}; "
                                 "NaN costs are not supported")
            mem = np.asarray([gc.node(i).mem_bytes for i in self.op_ids], dtype=np.int64)
        cap = np.asarray([c.device(d).mem_bytes for d in self.device_ids], dtype=np.int64)
        bw = np.zeros((K, K), dtype=np.float64)
        for a, da in enumerate(self.device_ids):
            for b, db in enumerate(self.device_ids):
                if a != b:
                    bw[a, b] = mesh.bandwidth(da, db)
        self._arrays = (np.ascontiguousarray(cost), mem, np.ascontiguousarray(dg.esrc),
                        np.ascontiguousarray(dg.edst), np.ascontiguousarray(dg.payload), cap, bw)
        prob = N.mp_problem(n, len(dg.esrc), K, *(N.ptr(x) for x in self._arrays))
        err = N.mp_error()
        handle = C.c_void_p()
        lib = N.lib()
        code = lib.mp_instance_create(C.byref(prob), device, C.byref(handle), C.byref(err))
        if code == N.MP_ERR_MISSING_COST:
            raise MissingCostError(self.op_ids[err.a], self.device_ids[err.b])
        if code == N.MP_ERR_CYCLE:
            raise CycleError(find_cycle(gc.node_ids, {i: gc.succs(i) for i in gc.node_ids}))
        N.check(code, err, "mp_instance_create")
        self._h = handle
        self._lib = lib
        self.n_ops = n
        self.n_flows = len(dg.esrc)
        self.K = K
        self.max_op_id = self.op_ids[-1]

    # -- lifecycle ----------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.mp_instance_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        inf = N.mp_instance_info()
        self._lib.mp_instance_info_get(self._h, C.byref(inf))
        return {f: getattr(inf, f) for f, _ in N.mp_instance_info._fields_}

    def tune(self, group_lanes: int = 0, ctas_per_sm: int = 0, ready_cap: int = 0, colo: bool = True,
             lanes_used: int = 0, tpp: bool = True, tpp_registers: bool = False,
             offchip: bool = False, tpp_round1: bool = False, durtab: bool = True,
             costs: str = "auto", row3: bool = False) -> None:
        """Launch-shape knobs: evaluation results never depend on them.  With
        automatic ``group_lanes``/``lanes_used`` and ``tpp`` the thread-per-placement
        kernel runs when the calibrated ready set fits its register capacity.
        ``ready_cap`` also fixes the local-search capacity (a proposal whose ready
        set exceeds it is rejected), the one knob local-search results depend on.
        ``costs``: where the duration-table kernel reads op costs ("auto": shared
        memory unless reading them through L1 fits 1.5x the lanes); ``row3`` forces the
        3-bit row tile (K <= 8) that is otherwise used only where it fits more lanes."""
        flags = ((0 if colo else 1) | (0 if tpp else 2) | (4 if tpp_registers else 0) | (8 if offchip else 0)
                 | (16 if tpp_round1 else 0) | (0 if durtab else 32)
                 | {"auto": 0, "global": 64, "smem": 128}[costs] | (256 if row3 else 0))
        if self._lib.mp_instance_tune(self._h, group_lanes, lanes_used, ctas_per_sm, ready_cap, flags) != 0:
            raise ValueError("group_lanes in {0,1,2,4,8,16,32}; lanes_used a multiple of it, <= 32")

    # -- placement encoding -------------------------------------------------------
    def encode(self, assignments) -> np.ndarray:
        """dicts op id -> device id  ->  uint8 [P, n_ops] rows of device indices.
        Raises KeyError like ``schedule_for_assignment`` (``solver.py:160-164``)."""
        rows = np.empty((len(assignments), self.n_ops), dtype=np.uint8)
        for r, asg in enumerate(assignments):
            for i, nid in enumerate(self.op_ids):
                if nid not in asg:
                    raise KeyError(f"assignment is missing op {nid}")
                d = asg[nid]
                if d not in self.dev_index:
                    raise KeyError(f"op {nid} assigned to unknown device {d}")
                rows[r, i] = self.dev_index[d]
        return rows

    def decode(self, row) -> dict[int, int]:
        return {nid: self.device_ids[int(k)] for nid, k in zip(self.op_ids, row)}

    def flow_id(self, f: int) -> int:
        return self.max_op_id + 1 + f


def _as_instance(gc, c=None, mesh=None) -> tuple[Instance, bool]:
    if isinstance(gc, Instance):
        return gc, False
    if mesh is None:
        mesh = effective_bandwidth(c)
    return Instance(gc, c, mesh), True


def _rows(inst: Instance, placements) -> np.ndarray:
    if isinstance(placements, np.ndarray):
        if placements.dtype != np.uint8:
            # no wrap-around: a device index >= 256 must not alias a valid one
            if not np.issubdtype(placements.dtype, np.integer):
                raise ValueError("placements must hold integer device indices")
            if placements.size and (placements.min() < 0 or placements.max() >= inst.K):
                raise ValueError(f"device indices must lie in [0, {inst.K})")
        rows = np.ascontiguousarray(placements, dtype=np.uint8)
        if rows.ndim != 2 or rows.shape[1] != inst.n_ops:
            raise ValueError(f"placements must be uint8 [P, {inst.n_ops}]")
        return rows
    return inst.encode(list(placements))


def evaluate_batch(gc, placements, c: Cluster | None = None, mesh: EffectiveMesh | None = None,
                   *, with_detail: bool = False):
    """Makespans of many placements at once (K3).

    ``gc`` is an :class:`Instance` or a ``CompGraph`` (then ``c``/``mesh`` are
    required).  ``placements`` is ``uint8 [P, n_ops]`` (device indices, column =
    ascending op id) or a sequence of ``{op id: device id}`` dicts.  Returns
    ``makespan`` (fp64, ``inf`` when infeasible) and, with ``with_detail``,
    ``status`` (0 ok, 1 memory exceeded, 2 unknown device), the first over-full
    device id and the overflow in bytes — the data ``MemoryExceededError``
    carries (``solver.py:85-87``).
    """
    inst, own = _as_instance(gc, c, mesh)
    try:
        rows = _rows(inst, placements)
        P = rows.shape[0]
        ms = np.empty(P, dtype=np.float64)
        st = np.empty(P, dtype=np.int8)
        md = np.empty(P, dtype=np.int32)
        ov = np.empty(P, dtype=np.int64)
        err = N.mp_error()
        code = inst._lib.mp_evaluate_batch(inst.handle, N.ptr(rows), P, N.ptr(ms), N.ptr(st),
                                           N.ptr(md), N.ptr(ov), 0, None, C.byref(err))
        N.check(code, err, "mp_evaluate_batch")
        if not with_detail:
            return ms
        dev = np.where(md >= 0, np.asarray(inst.device_ids, dtype=np.int64)[np.clip(md, 0, None)], -1)
        return ms, st, dev, ov
    finally:
        if own:
            inst.close()


def argmin(gc, placements, c: Cluster | None = None, mesh: EffectiveMesh | None = None):
    """Index and makespan of the best feasible row: the first strict minimum,
    as the ``brute_force`` keep-best loop (``solver.py:277-279``).  Returns
    ``(-1, inf)`` when no row is feasible (K4)."""
    inst, own = _as_instance(gc, c, mesh)
    try:
        rows = _rows(inst, placements)
        best = C.c_int64(-1)
        bms = C.c_double(math.inf)
        err = N.mp_error()
        code = inst._lib.mp_evaluate_argmin(inst.handle, N.ptr(rows), rows.shape[0], None, None,
                                            C.byref(best), C.byref(bms), 0, None, C.byref(err))
        N.check(code, err, "mp_evaluate_argmin")
        return int(best.value), float(bms.value)
    finally:
        if own:
            inst.close()


def _schedule_row(inst: Instance, row: np.ndarray) -> Schedule:
    Nn = inst.n_ops + inst.n_flows
    starts = np.empty(Nn, dtype=np.float64)
    ends = np.empty(Nn, dtype=np.float64)
    ms = C.c_double()
    err = N.mp_error()
    row = np.ascontiguousarray(row, dtype=np.uint8)
    code = inst._lib.mp_schedule_one(inst.handle, N.ptr(row), N.ptr(starts), N.ptr(ends),
                                     C.byref(ms), C.byref(err))
    if code == N.MP_ERR_MEMORY_EXCEEDED:
        raise MemoryExceededError(inst.device_ids[err.a], int(err.b))
    N.check(code, err, "mp_schedule_one")
    assign = inst.decode(row)
    st: dict[int, float] = {}
    en: dict[int, float] = {}
    for i, nid in enumerate(inst.op_ids):
        st[nid] = float(starts[i])
        en[nid] = float(ends[i])
    chan: dict[int, tuple[int, int] | None] = {}
    dg = inst.dense
    for f in range(inst.n_flows):
        q = inst.flow_id(f)
        st[q] = float(starts[inst.n_ops + f])
        en[q] = float(ends[inst.n_ops + f])
        ka = inst.device_ids[row[dg.esrc[f]]]
        kb = inst.device_ids[row[dg.edst[f]]]
        chan[q] = None if ka == kb else (ka, kb)
    return Schedule(assign, st, en, chan, float(ms.value))


def schedule_for_assignment(gc: CompGraph, c: Cluster, mesh: EffectiveMesh,
                            assignment: dict[int, int]) -> Schedule:
    """Timing for a fixed assignment (``solver.py:151-165``), computed on the GPU."""
    with Instance(gc, c, mesh) as inst:
        row = inst.encode([assignment])[0]
        return _schedule_row(inst, row)


def brute_force(gc: CompGraph, c: Cluster, mesh: EffectiveMesh) -> Solution:
    """Every assignment evaluated on the GPU; first strict optimum in
    ``itertools.product`` order over ``topo_order(gc)`` (``solver.py:257-282``)."""
    with Instance(gc, c, mesh) as inst:
        n, k = inst.n_ops, inst.K
        if n * math.log2(k) > 24:
            raise TooLargeError(n, k)
        order = topo_order(gc)
        pos = {nid: i for i, nid in enumerate(inst.op_ids)}
        op_order = np.asarray([pos[x] for x in order], dtype=np.int32)
        best = C.c_int64(-1)
        bms = C.c_double()
        err = N.mp_error()
        code = inst._lib.mp_enumerate_argmin(inst.handle, N.ptr(op_order), 0, k ** n,
                                             C.byref(best), C.byref(bms), None, C.byref(err))
        N.check(code, err, "mp_enumerate_argmin")
        if best.value < 0:
            return Solution(Status.INFEASIBLE, math.inf, None)
        x = int(best.value)
        row = np.empty(n, dtype=np.uint8)
        for t in range(n - 1, -1, -1):
            row[op_order[t]] = x % k
            x //= k
        sched = _schedule_row(inst, row)
        return Solution(Status.OPTIMAL, sched.makespan_s, sched, 0.0)


def solve_exact(gc: CompGraph, c: Cluster, mesh: EffectiveMesh,
                budget: SolveBudget | None = None, *, seed_chains: int | None = None,
                seed_moves: int | None = None) -> Solution:
    """Branch and bound over assignments on the GPU (``solver.py:172-254``).

    Same search space, node bound, memory-prefix check and incumbent rule as
    the reference (ops in ``topo_order(gc)``, devices ascending), but a whole
    frontier of up to 65 536 children is bounded per round on the GPU and the
    leaves are scheduled by the evaluator kernel (``mp_branch_and_bound``).

    * gap 0, no limits: ``Status.OPTIMAL`` with the optimal makespan and the
      lexicographically smallest optimal assignment — the reference's answer
      (its own acceptance claim: exact == brute force, ``test_acceptance.py:61-84``).
    * gap > 0: prune when ``bound >= best * (1 - gap)`` (``solver.py:239``);
      ``Status.OPTIMAL`` with ``gap`` set, objective within ``1/(1-gap)`` of the optimum.
    * node / time limits stop between rounds: ``Status.FEASIBLE`` with the
      incumbent, or ``Status.BUDGET`` without one (``solver.py:246-254``).
      ``node_limit`` counts bounded nodes and a round never starts past it; the
      time limit is checked between rounds (a round bounds at most 65 536
      children).

    By default (``seed_chains=None``) the incumbent is seeded with a GPU local
    search of 1024 chains (from seeded random rows and the two greedy
    baselines) when no node or time limit is set; at gap 0 seeds change the
    work, never the answer.  With a limit no seed is used by default, so a
    search stopped before its first leaf reports ``Status.BUDGET`` exactly where
    the reference does; an explicit ``seed_chains > 0`` opts back in (a stopped
    search then reports ``Status.FEASIBLE`` with the seed).
    """
    budget = budget or SolveBudget()
    if seed_chains is None:
        seed_chains = 0 if (budget.node_limit is not None or budget.time_limit_s is not None) else 1024
    with Instance(gc, c, mesh) as inst:
        n, k = inst.n_ops, inst.K
        order = topo_order(gc)
        pos = {nid: i for i, nid in enumerate(inst.op_ids)}
        op_order = np.asarray([pos[x] for x in order], dtype=np.int32)
        seeds = None
        if seed_chains > 0 and k > 1:
            rng = np.random.Generator(np.random.PCG64(0x5eed))
            start = rng.integers(0, k, (min(seed_chains, 64), n), dtype=np.uint8)
            moves = seed_moves if seed_moves is not None else min(4 * n * k, 2048)
            from .baselines import BaselineKind, greedy_row
            from .errors import InfeasibleMemoryError

            cand = [start]
            for kind in BaselineKind:  # the reference's greedy baselines as extra starting points
                try:
                    cand.append(greedy_row(inst, kind).reshape(1, n))
                except InfeasibleMemoryError:
                    pass
            row, ms, _, _ = local_search(inst, np.concatenate(cand), chains=seed_chains, moves=moves, seed=1)
            if math.isfinite(ms):
                seeds = row.reshape(1, n)
        best = np.zeros(n, dtype=np.uint8)
        bms = C.c_double()
        status = C.c_int32()
        visited = C.c_int64()
        err = N.mp_error()
        code = inst._lib.mp_branch_and_bound(
            inst.handle, N.ptr(op_order), float(budget.gap),
            -1 if budget.node_limit is None else int(budget.node_limit),
            -1.0 if budget.time_limit_s is None else float(budget.time_limit_s),
            N.ptr(seeds), 0 if seeds is None else 1, N.ptr(best), C.byref(bms), C.byref(status),
            C.byref(visited), C.byref(err))
        N.check(code, err, "mp_branch_and_bound")
        st = status.value
        if st in (N.MP_SOLVE_OPTIMAL, N.MP_SOLVE_FEASIBLE):
            sched = _schedule_row(inst, best)
            if st == N.MP_SOLVE_OPTIMAL:
                return Solution(Status.OPTIMAL, sched.makespan_s, sched, budget.gap)
            return Solution(Status.FEASIBLE, sched.makespan_s, sched, None)
        return Solution(Status.BUDGET if st == N.MP_SOLVE_BUDGET else Status.INFEASIBLE, math.inf, None)


def solve_with_derived_mesh(gc: CompGraph, c: Cluster, budget: SolveBudget | None = None) -> Solution:
    return solve_exact(gc, c, effective_bandwidth(c), budget)


def local_search(gc, seeds, c: Cluster | None = None, mesh: EffectiveMesh | None = None, *,
                 chains: int = 4096, moves: int = 256, seed: int = 0, chain_base: int = 0):
    """GPU hill climbing (K5): ``chains`` independent chains, each starting from
    seed row ``chain % len(seeds)`` and trying ``moves`` single-op device
    changes, accepting a move when the makespan does not increase.  Returns
    ``(best_row uint8[n_ops], best_makespan, best_chain, chain_makespans)``.
    Every reported row is an ordinary placement: re-evaluating it with
    :func:`evaluate_batch` (or the reference ``_schedule``) gives the same
    makespan bit for bit."""
    inst, own = _as_instance(gc, c, mesh)
    try:
        rows = _rows(inst, seeds)
        best = np.empty(inst.n_ops, dtype=np.uint8)
        bms = C.c_double()
        bch = C.c_int64()
        cms = np.empty(chains, dtype=np.float64)
        err = N.mp_error()
        code = inst._lib.mp_local_search(inst.handle, N.ptr(rows), rows.shape[0], chains, chain_base,
                                         moves, seed, N.ptr(best), C.byref(bms), C.byref(bch),
                                         N.ptr(cms), None, C.byref(err))
        N.check(code, err, "mp_local_search")
        return best, float(bms.value), int(bch.value), cms
    finally:
        if own:
            inst.close()
