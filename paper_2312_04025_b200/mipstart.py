"""GPU incumbent -> MILP start ("which can seed the MILP placement", north star).

The reference's MILP (``pkg/src/opplace/milp.py:116-294``, out of scope here) names
its variables ``x_{op}_{dev}`` (assignment), ``z_{flow}`` (flow crosses devices),
``u_{flow}_{a}_{b}`` (channel), ``S_{node}`` / ``C_{node}`` (start / completion),
``dord_{i}_{j}`` / ``dcom_{q}_{r}`` (order of unrelated op / flow pairs) and ``T``
(makespan), ``milp.py:144-165``.  :func:`mip_start_text` writes a schedule — e.g.
the best local-search or branch-and-bound placement, timed exactly by the GPU
evaluator — as a complete MIP start in the plain ``name value`` format Gurobi
(``.mst``) and HiGHS read next to the reference's ``export_lp`` file.

Ordering binaries follow ``ord1``/``ord2`` and ``con_*`` (``milp.py:196-257``):
``d = 1`` forces ``C_i <= S_j`` when both sides share the resource, ``d = 0``
forces ``C_j <= S_i``; the start writes ``d = 1`` iff ``C_i <= S_j`` (else the
reverse order holds in a feasible schedule, or the pair does not share a
resource and either value is feasible).
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
    st, en = schedule.starts, schedule.ends
    ops = sorted(gc.node_ids)
    flows = [max_id + 1 + f for f in range(len(gc.edges))]
    reach = _reachability(gc, max_id)
    for nodes, prefix in ((ops, "dord"), (flows, "dcom")):
        for a_i, i in enumerate(nodes):
            for j in nodes[a_i + 1:]:
                if (reach[i] >> j) & 1 or (reach[j] >> i) & 1:
                    continue  # related pairs have no ordering variable (milp.py:141-145)
                vals[f"{prefix}_{i}_{j}"] = 1.0 if en[i] <= st[j] else 0.0
    vals["T"] = schedule.makespan_s
    return vals


def _reachability(gc: CompGraph, max_id: int) -> dict[int, int]:
    """Descendant bitsets of every node of the augmented graph (op -> flow -> op),
    as in the reference's ``succ_closure`` (``milp.py:139``)."""
    succ: dict[int, list[int]] = {i: [] for i in gc.node_ids}
    for f, e in enumerate(gc.edges):
        q = max_id + 1 + f
        succ[e.src].append(q)
        succ[q] = [e.dst]
    indeg = {n: 0 for n in succ}
    for n, ss in succ.items():
        for s in ss:
            indeg[s] += 1
    order = [n for n in succ if indeg[n] == 0]
    for n in order:
        for s in succ[n]:
            indeg[s] -= 1
            if indeg[s] == 0:
                order.append(s)
    reach: dict[int, int] = {}
    for n in reversed(order):
        r = 0
        for s in succ[n]:
            r |= (1 << s) | reach[s]
        reach[n] = r
    return reach


def mip_start_text(schedule: Schedule, gc: CompGraph, c: Cluster) -> str:
    vals = mip_start_values(schedule, gc, c)
    lines = [f"# MIP start: makespan {schedule.makespan_s!r} s (GPU-evaluated placement)"]
    lines += [f"{name} {value!r}" for name, value in vals.items()]
    return "\n".join(lines) + "\n"


def write_mip_start(schedule: Schedule, gc: CompGraph, c: Cluster, path: str | Path) -> None:
    Path(path).write_text(mip_start_text(schedule, gc, c))
