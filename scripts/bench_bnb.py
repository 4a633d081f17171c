"""Time the GPU branch and bound (solve_exact) against the reference algorithm
restated serially in C (oracle/moirai_oracle.c orc_solve_exact, the CPU
checker) on instances past the brute-force guard.  Prints one JSON line per
instance.

python scripts/bench_bnb.py [--oracle] [--cases 20x4:0,22x4:0,...] [--accept8]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2312_04025_b200 as mp  # noqa: E402
from test_gpu_bnb import _random_instance  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="20x4:0,20x4:1,24x3:1,22x4:0")
    ap.add_argument("--oracle", action="store_true", help="also time the serial C restatement")
    ap.add_argument("--accept8", action="store_true")
    ap.add_argument("--time-limit", type=float, default=None)
    args = ap.parse_args()
    mp.solve_exact(*_random_instance(1, 8, 2, False), mp.effective_bandwidth(_random_instance(1, 8, 2, False)[1]))
    for spec in filter(None, args.cases.split(",")):
        shape, seed = spec.split(":")
        n, k = (int(x) for x in shape.split("x"))
        g, c = _random_instance(1000 + int(seed), n, k, tight=False)
        mesh = mp.effective_bandwidth(c)
        t0 = time.perf_counter()
        sol = mp.solve_exact(g, c, mesh, mp.SolveBudget(time_limit_s=args.time_limit))
        dt = time.perf_counter() - t0
        rec = {"case": spec, "ops": n, "devices": k, "status": sol.status.value, "objective": sol.objective_s,
               "gpu_s": dt}
        if args.oracle:
            from oracle import oracle
            from test_oracle import _flat_instance

            orc = _flat_instance(oracle, g, c, mesh)
            ids = g.node_ids
            order = [ids.index(x) for x in mp.topo_order(g)]
            t0 = time.perf_counter()
            st, row, best, visited = orc.solve_exact(order)
            rec.update({"oracle_s": time.perf_counter() - t0, "oracle_nodes": visited, "oracle_objective": best,
                        "same": best == sol.objective_s and sol.placement ==
                        {ids[i]: c.device_ids[int(d)] for i, d in enumerate(row)}})
        print(json.dumps(rec), flush=True)
    if args.accept8:
        from conftest import cluster_from, golden, graph_from

        case = next(x for x in golden("solve_exact.json") if x["name"] == "accept8-nodes500")
        g = graph_from(case["graph"])
        c = cluster_from(case["cluster"])
        mesh = mp.effective_bandwidth(c)
        for gap, tl in ((0.05, 120.0), (0.0, 120.0)):
            t0 = time.perf_counter()
            sol = mp.solve_exact(g, c, mesh, mp.SolveBudget(gap=gap, time_limit_s=tl))
            print(json.dumps({"case": f"accept8 gap={gap} limit={tl}s", "status": sol.status.value,
                              "objective": sol.objective_s, "gpu_s": time.perf_counter() - t0}), flush=True)


if __name__ == "__main__":
    main()
