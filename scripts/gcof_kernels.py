"""One gcof call on a synthetic graph (for an ncu launch list: per-kernel split)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_04025_b200 as mp  # noqa: E402
from paper_2312_04025_b200 import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
g = mp.gen_synthetic(mp.GenSpec(ops=n, width=32, density=0.5, devices=(0, 1, 2, 3)), 0)
rules = workloads.table_rules()
for _ in range(2):
    t0 = time.perf_counter()
    out = mp.gcof(g, rules)
    print(f"gcof {n}: {len(out)} nodes, {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
