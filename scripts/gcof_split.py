"""Where one gcof call spends its time: host flattening (_Flat), the native call
(upload, kernels, download), and building the result objects — median of 7
warm calls per graph.

    python scripts/gcof_split.py [c2 c3 synth:100000 ...]
"""
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_04025_b200 as mp  # noqa: E402
from paper_2312_04025_b200 import _native as N  # noqa: E402
from paper_2312_04025_b200 import fusion, workloads  # noqa: E402
from paper_2312_04025_b200.graph import _bulk_objects  # noqa: E402


def graph(name):
    if name.startswith("synth:"):
        n = int(name.split(":")[1])
        return name, mp.gen_synthetic(mp.GenSpec(ops=n, width=32, density=0.5, devices=(0, 1, 2, 3)), 0), \
            workloads.table_rules()
    w = {"c1": workloads.c1, "c2": lambda: workloads.c2(4), "c3": workloads.c3, "c4": workloads.c4}[name]()
    return w.name, w.raw, w.rules


for name in sys.argv[1:] or ["c2", "c3", "synth:20000", "synth:100000"]:
    label, g, rules = graph(name)
    mp.gcof(g, rules)
    tf, tn, tt = [], [], []
    for _ in range(7):
        t0 = time.perf_counter()
        t_all0 = t0
        with _bulk_objects():
            flat = fusion._Flat(g, rules, None)
        t1 = time.perf_counter()
        out = N.mp_coarsen_output()
        err = N.mp_error()
        N.check(N.lib().mp_coarsen(C.byref(flat.cin), 0, C.byref(out), C.byref(err)), err)
        t2 = time.perf_counter()
        N.lib().mp_coarsen_free(C.byref(out))
        mp.gcof(g, rules)
        t3 = time.perf_counter()
        tf.append(t1 - t0)
        tn.append(t2 - t1)
        tt.append(t3 - t2)
    f, n, t = (statistics.median(x) * 1e3 for x in (tf, tn, tt))
    print(f"{label}: whole gcof {t:.2f} ms = flatten {f:.2f} + native {n:.2f} + result objects {t - f - n:.2f} ms "
          f"(ordered replay: {fusion.LAST_GCOF['ordered_replay']})", flush=True)
