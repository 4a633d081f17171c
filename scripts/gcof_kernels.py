"""gcof calls on one graph (for an ncu launch list: per-kernel split).
usage: gcof_kernels.py [N ops of the synthetic graph | c1 | c2 | c3 | c4]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_04025_b200 as mp  # noqa: E402
from paper_2312_04025_b200 import workloads  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "100000"
if arg.isdigit():
    n = int(arg)
    g = mp.gen_synthetic(mp.GenSpec(ops=n, width=32, density=0.5, devices=(0, 1, 2, 3)), 0)
    rules = workloads.table_rules()
else:
    w = {"c1": workloads.c1, "c2": lambda: workloads.c2(4), "c3": workloads.c3, "c4": workloads.c4}[arg]()
    g, rules = w.raw, w.rules
for _ in range(2):
    t0 = time.perf_counter()
    out = mp.gcof(g, rules)
    print(f"gcof {arg}: {len(g)} -> {len(out)} nodes, {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
