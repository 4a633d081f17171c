"""Wall time of the native mp_coarsen call alone (input already flattened) vs the
whole gcof() call, C1-C4 graphs."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_04025_b200 as mp  # noqa: E402
from paper_2312_04025_b200 import _native as N, workloads  # noqa: E402
from paper_2312_04025_b200.fusion import _Flat  # noqa: E402

lib = N.lib()
cases = [(n, w.raw, w.rules) for n, w in (("c1", workloads.c1()), ("c2", workloads.c2(4)), ("c3", workloads.c3()))]
if len(sys.argv) > 1:
    n = int(sys.argv[1])
    cases = [(f"synth-{n}", mp.gen_synthetic(mp.GenSpec(ops=n, width=32, density=0.5, devices=(0, 1, 2, 3)), 0),
              workloads.table_rules())]
reps = 200 if len(sys.argv) == 1 else 5
for name, g, rules in cases:
    mp.gcof(g, rules)
    flat = _Flat(g, rules, None)
    ts = []
    for _ in range(reps):
        out = N.mp_coarsen_output()
        err = N.mp_error()
        t0 = time.perf_counter()
        code = lib.mp_coarsen(C.byref(flat.cin), 0, C.byref(out), C.byref(err))
        ts.append(time.perf_counter() - t0)
        lib.mp_coarsen_free(C.byref(out))
    t_flat = []
    for _ in range(reps):
        t0 = time.perf_counter(); _Flat(g, rules, None); t_flat.append(time.perf_counter() - t0)
    t_all = []
    for _ in range(reps):
        t0 = time.perf_counter(); mp.gcof(g, rules); t_all.append(time.perf_counter() - t0)
    med = lambda x: sorted(x)[len(x) // 2] * 1e3
    print(f"{name}: native mp_coarsen {med(ts):.3f} ms, _Flat {med(t_flat):.3f} ms, gcof() {med(t_all):.3f} ms", flush=True)
