"""GPU incumbent -> MIP start for the reference MILP (INTEGRATION.md example), C2."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_04025_b200 as mp  # noqa: E402
from paper_2312_04025_b200 import workloads  # noqa: E402

w = workloads.c2(4)
graph = mp.gcof(w.raw, w.rules)
mesh = mp.effective_bandwidth(w.cluster)
inst = mp.Instance(graph, w.cluster, mesh)
seeds = workloads.placements(1, 256, len(graph), len(w.cluster.device_ids))
row, ms, _, _ = mp.local_search(inst, seeds, chains=4096, moves=32)
sched = mp.schedule_for_assignment(graph, w.cluster, mesh, inst.decode(row))
assert sched.makespan_s == ms, (sched.makespan_s, ms)
out = Path("gpurun_out/start.mst")
out.parent.mkdir(exist_ok=True)
mp.write_mip_start(sched, graph, w.cluster, out)
lines = out.read_text().splitlines()
print(lines[0], len(lines) - 1, "values", flush=True)
