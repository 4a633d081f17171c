"""A schema-1 graph file -> load_graph -> gcof, 10^5 ops: time of each step, first
(cold) gcof call on the loaded graph (fed from the reader's arrays, no OpNode built) vs
the first call on the generator's object graph (interning from the objects)."""
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_04025_b200 as mp  # noqa: E402
from paper_2312_04025_b200 import fileio, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
rules = workloads.table_rules()
mp.gcof(mp.gen_synthetic(mp.GenSpec(ops=2000, width=32, density=0.5, devices=(0, 1, 2, 3)), 9), rules)  # warm-up
g = mp.gen_synthetic(mp.GenSpec(ops=n, width=32, density=0.5, devices=(0, 1, 2, 3)), 0)
with tempfile.TemporaryDirectory() as d:
    p = Path(d) / "g.json"
    fileio.save_graph(g, p)
    t0 = time.perf_counter()
    loaded = fileio.load_graph(p)
    t1 = time.perf_counter()
    out = mp.gcof(loaded, rules)
    t2 = time.perf_counter()
    mp.gcof(loaded, rules)
    t3 = time.perf_counter()
    objs = loaded._nodes_d is None
t4 = time.perf_counter()
mp.gcof(g, rules)
t5 = time.perf_counter()
print(f"{n} ops ({p.name}): load_graph {1e3 * (t1 - t0):.1f} ms, first gcof on the loaded graph "
      f"{1e3 * (t2 - t1):.1f} ms (input objects never built: {objs}), warm {1e3 * (t3 - t2):.1f} ms; "
      f"first gcof on the object graph {1e3 * (t5 - t4):.1f} ms; {len(out)} groups")
