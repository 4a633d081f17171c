"""Time the evaluator kernel on device-resident placements for several launch
shapes (lanes per placement G); optional single config for ncu.

python scripts/prof_eval.py [--workload c2] [--rows 262144] [--G 4,8,16,32] [--iters 3]
"""

from __future__ import annotations

import argparse
import ctypes as C
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2312_04025_b200 as mp  # noqa: E402
from paper_2312_04025_b200 import _native as N  # noqa: E402
from paper_2312_04025_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--rows", type=int, default=1 << 18)
    ap.add_argument("--G", default="0", help="G or G:U list (0 = automatic shape)")
    ap.add_argument("--rcap", type=int, default=0)
    ap.add_argument("--no-colo", action="store_true")
    ap.add_argument("--no-tpp", action="store_true")
    ap.add_argument("--tpp-reg", action="store_true")
    ap.add_argument("--offchip", action="store_true")
    ap.add_argument("--round1", action="store_true", help="the round-1 TPP evaluator (A/B)")
    ap.add_argument("--no-durtab", action="store_true", help="divide flow durations at run time (A/B)")
    ap.add_argument("--costs", default="auto", choices=("auto", "global", "smem"), help="TPP op-cost placement (A/B)")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    args = ap.parse_args()
    if args.workload.startswith("c5:"):
        _, n, k = args.workload.split(":")
        w = workloads.c5(int(n), int(k))
    else:
        w = {"c1": workloads.c1, "c2": lambda: workloads.c2(4), "c2k8": lambda: workloads.c2(8),
             "c3": workloads.c3, "c4": workloads.c4, "c4pcie": lambda: workloads.c4("pcie")}[args.workload]()
    coarse = mp.gcof(w.raw, w.rules)
    inst = mp.Instance(coarse, w.cluster, mp.effective_bandwidth(w.cluster))
    rows = workloads.placements(w.seed, args.rows, inst.n_ops, inst.K)
    dev_rows = torch.from_numpy(rows).cuda()
    ms = torch.empty(args.rows, dtype=torch.float64, device="cuda")
    st = torch.empty(args.rows, dtype=torch.int8, device="cuda")
    stream = torch.cuda.current_stream()
    lib = N.lib()
    for spec in args.G.split(","):
        G, U = (int(x) for x in (spec.split(":") + ["0"])[:2])
        inst.tune(G, args.ctas_per_sm, ready_cap=args.rcap, colo=not args.no_colo, lanes_used=U, tpp=not args.no_tpp,
                  tpp_registers=args.tpp_reg, offchip=args.offchip, tpp_round1=args.round1,
                  durtab=not args.no_durtab, costs=args.costs)
        info = inst.info()
        best = C.c_int64()
        bms = C.c_double()
        err = N.mp_error()

        def run():
            code = lib.mp_evaluate_argmin(inst.handle, C.c_void_p(dev_rows.data_ptr()), args.rows,
                                          C.c_void_p(ms.data_ptr()), C.c_void_p(st.data_ptr()), C.byref(best),
                                          C.byref(bms), N.MP_DEVICE_PTRS, C.c_void_p(stream.cuda_stream),
                                          C.byref(err))
            N.check(code, err)

        run()
        torch.cuda.synchronize()
        times = []
        for _ in range(args.iters):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        t = min(times)
        feas = int((st == 0).sum().item())
        print(f"{w.name} a={inst.n_ops} b={inst.n_flows} peak={info['peak_probe']} feasible={feas}/{args.rows} G={info['group_lanes']} U={info['lanes_used']} colo={info['colo']} gpc={info['groups_per_cta']} "
              f"ctas={info['ctas']} rcap={info['ready_cap']} smem={info['smem_bytes']} state={info['state_bytes']} "
              f"mode={info['mode']} tables={info['table_bytes']} durtab={info['dur_classes']} tpp={info['tpp_kind']}:{info['tpp_ready_cap']}x{info['tpp_threads']}: {args.rows / t:,.0f} placements/s ({t * 1e3:.2f} ms), feasible rows scheduled {feas / t:,.0f}/s best={best.value}",
              flush=True)


if __name__ == "__main__":
    main()
