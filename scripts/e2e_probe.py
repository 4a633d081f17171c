"""Where the e2e time goes: H2D bandwidth from pinned memory, and wall time of
the host-pointer (streamed) vs device-pointer argmin calls on C2."""
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

w = workloads.c2(4)
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


for host in (False, True, False, True):
    for _ in range(2):
        call(host)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        call(host)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"{'host (streamed)' if host else 'device ptrs'}: {dt * 1e3:.2f} ms/call, {P / dt / 1e6:.1f} M placements/s")
