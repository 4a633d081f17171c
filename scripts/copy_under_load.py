"""Does a 278 MB pinned H2D copy slow down while the C2-K8 evaluation kernel runs?
Times the copy alone and concurrently with a device-pointer evaluation (events on the copy
stream), and the evaluation alone / with the copy (events on its stream)."""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2312_04025_b200 as mp  # noqa: E402
from paper_2312_04025_b200 import _native as N  # noqa: E402
from paper_2312_04025_b200 import workloads  # noqa: E402

w = workloads.c2(8)
inst = mp.Instance(mp.gcof(w.raw, w.rules), w.cluster, mp.effective_bandwidth(w.cluster))
P = 1 << 20
rows = workloads.placements(2, P, inst.n_ops, inst.K)
h = torch.from_numpy(rows).pin_memory()
d = h.cuda()
d2 = torch.empty_like(d)
dm = torch.empty(P, dtype=torch.float64, device="cuda")
lib, err, best, bms = N.lib(), N.mp_error(), C.c_int64(), C.c_double()
ks, cs = torch.cuda.Stream(), torch.cuda.Stream()


def kernel():
    with torch.cuda.stream(ks):
        N.check(lib.mp_evaluate_argmin(inst.handle, C.c_void_p(d.data_ptr()), P, C.c_void_p(dm.data_ptr()), None,
                                       C.byref(best), C.byref(bms), N.MP_DEVICE_PTRS, C.c_void_p(ks.cuda_stream),
                                       C.byref(err)), err, "argmin")


def run(with_kernel, with_copy):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(ks)
    e[2].record(cs)
    if with_copy:
        with torch.cuda.stream(cs):
            d2.copy_(h, non_blocking=True)
    e[3].record(cs)
    if with_kernel:
        kernel()
    e[1].record(ks)
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3])


for _ in range(2):
    run(True, True)
for label, k, c in (("copy alone", False, True), ("kernel alone", True, False), ("both", True, True)):
    r = [run(k, c) for _ in range(5)]
    km = sorted(x[0] for x in r)[2]
    cm = sorted(x[1] for x in r)[2]
    print(f"{label:14s} kernel-stream span {km:7.2f} ms   copy {cm:6.2f} ms ({h.numel() / cm / 1e6:5.1f} GB/s)", flush=True)
