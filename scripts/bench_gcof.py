"""GCOF timing on the GPU (median of repeats, input already parsed) for the
named raw graphs and the gen_synthetic sweep; parity vs the CPU oracle."""
import statistics, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_04025_b200 as mp
from paper_2312_04025_b200 import workloads
from paper_2312_04025_b200.fusion import _Flat
from oracle.oracle import gcof_partition

cases = [(w.name, w.raw, w.rules) for w in (workloads.c1(), workloads.c2(4), workloads.c3(), workloads.c4())]
for n in [int(x) for x in (sys.argv[1:] or ["5000", "20000", "50000", "100000"])]:
    t0 = time.perf_counter()
    g = mp.gen_synthetic(mp.GenSpec(ops=n, width=32, density=0.5, devices=(0, 1, 2, 3)), 0)
    cases.append((f"synth-{n} (gen {time.perf_counter() - t0:.1f}s)", g, workloads.table_rules()))
for name, g, rules in cases:
    out = mp.gcof(g, rules)  # warm
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); out = mp.gcof(g, rules); ts.append(time.perf_counter() - t0)
    k = _Flat(g, rules, None).keep
    t0 = time.perf_counter(); part = gcof_partition(k[1], k[2], k[3], k[6], k[7], k[10], k[11]); t_orc = time.perf_counter() - t0
    idx = g.csr().index
    ok = [[idx[m] for m in nd.members] for nd in out.nodes] == [p for p, _ in part]
    print(f"{name}: {len(g)} -> {len(out)} nodes, {len(out.edges)} edges; gpu gcof median {statistics.median(ts)*1e3:.2f} ms; C-oracle DFS+partition {t_orc*1e3:.2f} ms; partition equal {ok}", flush=True)
