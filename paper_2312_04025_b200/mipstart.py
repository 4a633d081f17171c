"""GPU incumbent -> MILP start ("which can seed the MILP placement", north star).

The reference's MILP (``pkg/src/opplace/milp.py:116-294``, out of scope here) names
its variables ``x_{op}_{dev}`` (assignment), ``z_{flow}`` (flow crosses devices),
``u_{flow}_{a}_{b}`` (channel), ``S_{node}`` / ``C_{node}`` (start / completion),
``milp.py:151-160``.  :func:`mip_start_text` writes a schedule — e.g. the best
local-search or branch-and-bound placement, timed exactly by the GPU evaluator —
as a MIP start in the plain ``name value`` format Gurobi (``.mst``) and HiGHS
read next to the reference's ``export_lp`` file; the solver completes the
ordering binaries itself.
"""

from __future__ import annotations

from pathlib import Path

from .graph import CompGraph
from .placement import Schedule
from .profiles import Cluster


def mip_start_values(schedule: Schedule, gc: CompGraph, c: Cluster) -> dict[str, float]:
    """Variable name -> value for every assignment, crossing, channel and time
    variable of the reference model."""
    vals: dict[str, float] = {}
    devs = c.device_ids
    assign = schedule.assignment
    for i in gc.node_ids:
        for k in devs:
            vals[f"x_{i}_{k}"] = 1.0 if assign[i] == k else 0.0
    max_id = max(gc.node_ids)
    for f, e in enumerate(gc.edges):
        q = max_id + 1 + f
        ch = schedule.channels.get(q)
        vals[f"z_{q}"] = 0.0 if ch is None else 1.0
        for a in devs:
            for b in devs:
                if a != b:
                    vals[f"u_{q}_{a}_{b}"] = 1.0 if ch == (a, b) else 0.0
    for n in sorted(schedule.starts):
        vals[f"S_{n}"] = schedule.starts[n]
        vals[f"C_{n}"] = schedule.ends[n]
    return vals


def mip_start_text(schedule: Schedule, gc: CompGraph, c: Cluster) -> str:
    vals = mip_start_values(schedule, gc, c)
    lines = [f"# MIP start: makespan {schedule.makespan_s!r} s (GPU-evaluated placement)"]
    lines += [f"{name} {value!r}" for name, value in vals.items()]
    return "\n".join(lines) + "\n"


def write_mip_start(schedule: Schedule, gc: CompGraph, c: Cluster, path: str | Path) -> None:
    Path(path).write_text(mip_start_text(schedule, gc, c))
