#!/usr/bin/env python3
"""How fast is oracle/pyref.py (the CPU reference arm of bench.py) compared with
the reference package's own `_schedule` (pkg/src/opplace/solver.py:80-148)?

Run HERE (the container with /root/reference); the GPU box has no reference.
For each workload: the coarse graph, one `_Instance` / `pyref.Instance` built
outside the timer, then N placements (pre-converted to dicts for the reference,
as brute_force's loop does, solver.py:263-274) timed single-threaded, median of
3.  Also checks that both give bit-identical makespans.

    python scripts/pyref_vs_reference.py [--rows 400] > profiles/r02/pyref_vs_reference.txt
"""

from __future__ import annotations

import argparse
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import bench  # noqa: E402
from oracle import pyref  # noqa: E402
from paper_2312_04025_b200 import workloads  # noqa: E402


def main():
    import opplace
    from opplace import solver as rsolver

    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=400)
    args = ap.parse_args()
    for name in ("c1", "c2", "c2k8", "c4"):
        w = bench.build_workload(name)
        g = bench.coarse_on_cpu(w)
        arrays = bench.flat_arrays(g, w.cluster)
        n_ops, K = len(g), len(w.cluster.device_ids)
        rows = workloads.placements(w.seed, args.rows, n_ops, K)
        # reference objects
        rg = opplace.CompGraph([opplace.OpNode(n.id, n.op_type, n.mem_bytes, dict(n.compute_time), n.members,
                                               n.type_seq, opplace.Tag(n.tag.value)) for n in g.nodes],
                               [opplace.FlowEdge(e.src, e.dst, e.payload_bytes) for e in g.edges])
        rc = opplace.Cluster([opplace.Device(d.id, d.mem_bytes) for d in w.cluster.devices], dict(w.cluster.links))
        rinst = rsolver._Instance(rg, rc, opplace.effective_bandwidth(rc))
        ids, devs = g.node_ids, w.cluster.device_ids
        dicts = [{ids[i]: devs[int(r[i])] for i in range(n_ops)} for r in rows]
        pinst = pyref.Instance.from_arrays(arrays)

        def t_ref():
            t0 = time.perf_counter()
            out = [rsolver._schedule(rinst, a).makespan_s for a in dicts]
            return time.perf_counter() - t0, out

        def t_port():
            t0 = time.perf_counter()
            out = pyref.eval_rows(pinst, rows)
            return time.perf_counter() - t0, out

        tr = [t_ref() for _ in range(3)]
        tp = [t_port() for _ in range(3)]
        same = [float(a).hex() for a in tr[0][1]] == [float(b).hex() for b in tp[0][1]]
        r_s = statistics.median(x[0] for x in tr)
        p_s = statistics.median(x[0] for x in tp)
        print(f"{w.name}: {n_ops} ops, {args.rows} placements, 1 core: reference _schedule {args.rows / r_s:,.0f}/s, "
              f"pyref {args.rows / p_s:,.0f}/s, pyref/reference speed {r_s / p_s:.2f}x, makespans bit-identical {same}",
              flush=True)


if __name__ == "__main__":
    main()
