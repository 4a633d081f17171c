"""Where the e2e time goes: H2D bandwidth from pinned memory, and wall time of
the host-pointer (streamed) vs device-pointer argmin calls on C2-K8, plus the
device-pointer call with a concurrent 278 MB H2D copy on another stream (the
copy's interference alone) and with the 8 MB makespan read-back."""
import ctypes as C
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2312_04025_b200 as mp  # noqa: E402
from paper_2312_04025_b200 import _native as N  # noqa: E402
from paper_2312_04025_b200 import workloads  # noqa: E402

w = workloads.c2(8)
coarse = mp.gcof(w.raw, w.rules)
inst = mp.Instance(coarse, w.cluster, mp.effective_bandwidth(w.cluster))
P = 1 << 20
rows = workloads.placements(2, P, inst.n_ops, inst.K)
h = torch.from_numpy(rows).pin_memory()
d = torch.empty_like(h, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print(f"H2D pinned: {h.numel() / dt / 1e9:.1f} GB/s ({dt * 1e3:.2f} ms for {h.numel() / 1e6:.0f} MB)")
hm = torch.empty(P, dtype=torch.float64).pin_memory()
dm = torch.empty(P, dtype=torch.float64, device="cuda")
lib, err, best, bms = N.lib(), N.mp_error(), C.c_int64(), C.c_double()
s = torch.cuda.current_stream()


def call(host):
    if host:
        code = lib.mp_evaluate_argmin(inst.handle, C.c_void_p(h.data_ptr()), P, C.c_void_p(hm.data_ptr()), None,
                                      C.byref(best), C.byref(bms), 0, C.c_void_p(s.cuda_stream), C.byref(err))
    else:
        code = lib.mp_evaluate_argmin(inst.handle, C.c_void_p(d.data_ptr()), P, C.c_void_p(dm.data_ptr()), None,
                                      C.byref(best), C.byref(bms), N.MP_DEVICE_PTRS, C.c_void_p(s.cuda_stream),
                                      C.byref(err))
    N.check(code, err)


side = torch.cuda.Stream()
d2 = torch.empty_like(h, device="cuda")


def timed(label, fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"{label}: {dt * 1e3:.2f} ms/call, {P / dt / 1e6:.1f} M placements/s", flush=True)


def dev_with_copy():
    with torch.cuda.stream(side):
        d2.copy_(h, non_blocking=True)
    call(False)
    side.synchronize()


def dev_with_readback():
    call(False)
    hm.copy_(dm, non_blocking=True)


def gpu_span(label, fn, n=5):
    """GPU-side span of the call (events on its stream) next to its wall time."""
    fn()
    torch.cuda.synchronize()
    spans, walls = [], []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
        spans.append(e0.elapsed_time(e1))
    print(f"{label}: GPU span {min(spans):.2f} ms, wall {min(walls):.2f} ms", flush=True)


gpu_span("device ptrs", lambda: call(False))
gpu_span("host (streamed)", lambda: call(True))


def fresh_then_call():
    d.copy_(h, non_blocking=True)  # rows just written by DMA, then the kernel reads them
    call(False)


gpu_span("device ptrs, rows freshly copied (copy + call)", fresh_then_call)
gpu_span("copy only", lambda: d.copy_(h, non_blocking=True))
for _ in range(2):
    timed("device ptrs", lambda: call(False))
    timed("device ptrs + 8 MB makespan read-back", dev_with_readback)
    timed("device ptrs + concurrent 278 MB H2D copy", dev_with_copy)
    timed("host (streamed)", lambda: call(True))
