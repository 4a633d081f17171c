"""CPU baselines for every SURVEY §8(d) configuration on this host: the
reference algorithm in pure Python (oracle/pyref.py) on all cores and the C
restatement (oracle/moirai_oracle.c) on all cores, beside the GPU numbers of
profiles/r01/workloads_sweep_tpp.txt.  One JSON line per configuration.

python scripts/cpu_baselines.py [--seconds 4]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2312_04025_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=4.0)
    args = ap.parse_args()
    cfgs = [("c1", workloads.c1), ("c2", lambda: workloads.c2(4)), ("c2k8", lambda: workloads.c2(8)),
            ("c3", workloads.c3), ("c4", workloads.c4), ("c5:1000:4", lambda: workloads.c5(1000, 4)),
            ("c5:5000:8", lambda: workloads.c5(5000, 8))]
    for name, fn in cfgs:
        w = fn()
        g = bench.coarse_on_cpu(w)
        arrays = bench.flat_arrays(g, w.cluster)
        rows = workloads.placements(w.seed, 200_000 if not name.startswith("c5") else 20_000, len(g),
                                    len(w.cluster.device_ids))
        py = bench.cpu_baseline_python(arrays, rows, args.seconds)
        nat = bench.cpu_baseline_native(arrays, rows, args.seconds / 2)
        print(json.dumps({"config": name, "workload": w.name, "ops": len(g), "flows": len(g.edges),
                          "python_all_cores": py, "c_all_cores": nat}), flush=True)


if __name__ == "__main__":
    main()
