"""Small runs of every kernel family, for compute-sanitizer (memcheck /
racecheck / synccheck): TPP (shared-memory and register ready sets), group
kernel (on- and off-chip), local search (TPP and group), wide C5 graph, GCOF,
branch and bound, greedy, audit."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_04025_b200 as mp  # noqa: E402
from paper_2312_04025_b200 import workloads  # noqa: E402

w = workloads.c1()
g = mp.gcof(w.raw, w.rules)
bw = mp.effective_bandwidth(w.cluster)
rows = workloads.placements(7, 512, len(g), len(w.cluster.device_ids))
ref = None
for kw in ({}, {"tpp_registers": True}, {"tpp": False}, {"tpp": False, "offchip": True}):
    inst = mp.Instance(g, w.cluster, bw)
    if kw:
        inst.tune(**kw)
    ms = np.asarray(mp.evaluate_batch(inst, rows))
    ref = ms if ref is None else ref
    assert np.array_equal(ms.view(np.int64), ref.view(np.int64)), kw
    r = mp.local_search(inst, rows[:64], chains=64, moves=4)
    print("eval + local search", kw or "default", "ok", r[1], flush=True)
    inst.close()
w5 = workloads.c5(1000, 4)
g5 = mp.gcof(w5.raw, w5.rules)
inst5 = mp.Instance(g5, w5.cluster, mp.effective_bandwidth(w5.cluster))
r5 = workloads.placements(3, 256, len(g5), 4)
print("c5 eval", float(np.min(mp.evaluate_batch(inst5, r5))), flush=True)
small = mp.gen_synthetic(mp.GenSpec(ops=9, width=3, density=0.5, devices=(0, 1)), 1)
c2 = mp.Cluster([mp.Device(0, 10**12), mp.Device(1, 10**12)], {(0, 1): 1e9, (1, 0): 1e9})
sol = mp.solve_exact(small, c2, mp.effective_bandwidth(c2))
print("bnb", sol.status, sol.objective_s, flush=True)
s = mp.greedy_place(g, w.cluster, bw)
print("greedy", s.makespan_s, flush=True)
print("audit", len(mp.check_feasibility(s, g, w.cluster, bw)), flush=True)
big = mp.gen_synthetic(mp.GenSpec(ops=15_000, width=32, density=0.5, devices=(0, 1)), 2)
print("gcof 15k (global DFS, side-stream Kahn)", len(mp.gcof(big, workloads.table_rules())), flush=True)
print("done", flush=True)
