#!/usr/bin/env python3
"""Headline benchmark: candidate placements evaluated per second (makespan).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2k8]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU, NCCL)

``--gpus N`` without torchrun re-launches this script under
``torch.distributed.run`` with N ranks; asking for more GPUs than the box has is
an error (exit 2), never a silent one-rank run.

Workload (BASELINE.json north star: "BERT-large 8-device config"): the BERT-large
inference graph (embed + 24 encoder layers, 481 raw ops) coarsened by GCOF on the
GPU to 265 ops / 360 flows, placed on two Table-III intra-server quads joined by
100 Gb/s InfiniBand (K=8).  A step evaluates one batch of
ROWS random placements per GPU (uint8 device indices from PCG64(2 + 1000*rank):
weak scaling, each rank a disjoint shard) and reduces the best placement across
GPUs (16-byte NCCL all-gather of (makespan bits, global row)).  Inputs are
278 MB per GPU per step (> L2).  ``--workload c2`` is the K=4 quad (configs[1]).

value  = device-resident throughput: rows already in HBM, max time over ranks.
e2e    = the same step through the C ABI with HOST (pinned) buffers: H2D of the
         rows and D2H of every makespan inside the timed region.
parity = after timing, every makespan and status of rank 0's last step is
         compared bit for bit with the CPU oracle (oracle/moirai_oracle.c), and
         the argmin with the oracle's first strict minimum.
Reference arm (--impl reference): the reference algorithm in pure Python
(oracle/pyref.py, faithful to opplace._schedule) on every host core.
"""

from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "candidate placements evaluated/sec (makespan) at 1/2/4/8 B200 vs host-CPU ref"
UNIT = "placements/s"
WORKLOADS = ("c1", "c2", "c2k8", "c3", "c4", "c4pcie")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---- workload (built identically on every rank and in both arms) ---------------------------
def build_workload(name: str):
    from paper_2312_04025_b200 import workloads

    return {"c1": workloads.c1, "c2": lambda: workloads.c2(4), "c2k8": lambda: workloads.c2(8),
            "c3": workloads.c3, "c4": workloads.c4, "c4pcie": lambda: workloads.c4("pcie")}[name]()


def workload_config(w, n_ops: int, n_flows: int, K: int) -> dict:
    """The `config` object of the JSON line — identical in both arms."""
    return {"workload": f"{w.name} (GCOF {len(w.raw)} -> {n_ops} ops / {n_flows} flows, K={K})",
            "placements": "PCG64(seed=2+1000*rank) uint8 device indices per op, one row per placement",
            "l2": "inputs larger than L2 (265 B x 2^20 rows = 278 MB per GPU per step)",
            "dtype_note": "fp64 makespans, bit-exact with the reference"}


def coarse_on_cpu(w):
    """The coarse graph via the CPU oracle (reference arm only; identical to the
    GPU gcof by tests/test_gpu_parity.py)."""
    import paper_2312_04025_b200 as mp
    from oracle.oracle import gcof_partition, materialize
    from paper_2312_04025_b200.fusion import _Flat

    k = _Flat(w.raw, w.rules, None).keep
    nodes, edges = materialize(w.raw, gcof_partition(k[1], k[2], k[3], k[6], k[7], k[10], k[11]))
    return mp.CompGraph([mp.OpNode(i, t, mem, cost, m, s, mp.Tag(tag)) for i, t, m, s, tag, mem, cost in nodes],
                        [mp.FlowEdge(*e) for e in edges])


def flat_arrays(g, cluster):
    import paper_2312_04025_b200 as mp

    mesh = mp.effective_bandwidth(cluster)
    ids = g.node_ids
    devs = cluster.device_ids
    dg = g.csr()
    K = len(devs)
    bw = np.zeros((K, K))
    for a, da in enumerate(devs):
        for b, db in enumerate(devs):
            if a != b:
                bw[a, b] = mesh.bandwidth(da, db)
    return (np.array([[g.node(i).compute_time[d] for d in devs] for i in ids], dtype=np.float64),
            np.array([g.node(i).mem_bytes for i in ids], dtype=np.int64), dg.esrc, dg.edst, dg.payload,
            np.array([cluster.device(d).mem_bytes for d in devs], dtype=np.int64), bw)


# ---- CPU baselines ---------------------------------------------------------------------
def cpu_baseline_python(arrays, rows_all, seconds: float):
    """The reference algorithm in pure Python on every host core (bounded sample)."""
    from oracle import pyref

    inst = pyref.Instance.from_arrays(arrays)
    t0 = time.perf_counter()
    pyref.eval_rows(inst, rows_all[:20])
    per_row = (time.perf_counter() - t0) / 20
    cores = os.cpu_count() or 1
    n = int(max(cores * 4, min(len(rows_all), seconds / per_row * cores)))
    dt, _, procs = pyref.time_all_cores(arrays, rows_all[:n], processes=cores)
    return {"value": n / dt, "unit": UNIT, "cores": procs, "kind": "port",
            "sample": f"first {n} placements of the workload stream, pure-Python restatement of "
                      f"opplace._schedule (oracle/pyref.py), {procs} processes, {dt:.1f} s"}


def cpu_baseline_native(orc, rows_all, seconds: float):
    """The C restatement (oracle/moirai_oracle.c) on every host core — a far
    stronger CPU baseline than the reference's own Python, reported alongside."""
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    orc.eval_batch(rows_all[:2000], threads=cores)
    per = (time.perf_counter() - t0) / 2000
    n = int(min(len(rows_all), max(10000, seconds / per)))
    t0 = time.perf_counter()
    orc.eval_batch(rows_all[:n], threads=cores)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"first {n} placements, C restatement (oracle/moirai_oracle.c), {cores} pthreads, {dt:.1f} s"}


# ---- parity self-check (outside every timed region) -----------------------------------------
def parity_check(orc, rows, ms, st, best_row, best_ms, budget_s: float = 60.0) -> dict:
    """Bitwise comparison of the GPU's makespans/statuses with the C oracle on the
    same rows, plus the keep-best row (brute_force's first strict minimum,
    solver.py:277-279).  All rows when the oracle finishes within `budget_s`,
    else a 4096-row sample that includes the argmin row."""
    cores = os.cpu_count() or 1
    P = len(rows)
    t0 = time.perf_counter()
    orc.eval_batch(rows[:256], threads=cores)
    per = max((time.perf_counter() - t0) / 256, 1e-9)
    if per * P <= budget_s:
        idx = np.arange(P)
    else:
        idx = np.unique(np.concatenate([np.linspace(0, P - 1, 4096).astype(np.int64),
                                        [best_row] if best_row >= 0 else []]).astype(np.int64))
    want_ms, want_st = orc.eval_batch(np.ascontiguousarray(rows[idx]), threads=cores)
    got_st = st[idx].astype(np.int64)
    feas = want_st == 0
    mism = int(np.count_nonzero(got_st != want_st.astype(np.int64)))
    mism += int(np.count_nonzero(ms[idx][feas].view(np.uint64) != want_ms[feas].view(np.uint64)))
    out = {"checked": int(len(idx)), "mismatches": mism, "oracle": "oracle/moirai_oracle.c",
           "feasible": int(np.count_nonzero(feas)), "seconds": round(time.perf_counter() - t0, 2)}
    if len(idx) == P:
        if np.any(feas):
            fi = np.flatnonzero(feas)
            o_best = int(fi[np.argmin(want_ms[fi])])  # argmin returns the first minimum
            out["argmin_row"] = o_best
            out["argmin_match"] = bool(o_best == best_row and want_ms[o_best] == best_ms)
        else:
            out["argmin_match"] = best_row < 0
    else:
        out["argmin_match"] = bool(best_row < 0 or ms[best_row] == best_ms)
    return out


# ---- clocks ------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait(timeout=5)
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---- roofline denominators ------------------------------------------------------------------
def measured_hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json, copy)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def onchip_peaks() -> dict | None:
    """Shared-memory and L2 load bandwidth measured on this box now
    (paper_2312_04025_b200/csrc/mp_peaks.cu), before the timed region."""
    lib_path = ROOT / "paper_2312_04025_b200" / "libmoirai_peaks.so"
    if not lib_path.exists():
        return None
    lib = C.CDLL(str(lib_path))
    out = (C.c_double * 3)()
    res = {}
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    best = None
    for width in (16, 8):
        if lib.mp_peak_smem(width, 5, out) != 0:
            return None
        if best is None or out[0] > best[0]:
            best = (out[0], out[1], width)
    res["smem_TBps"] = best[0] / 1e12
    res["smem_bytes_per_clk_per_sm"] = best[1]
    res["smem_load_width"] = best[2]
    res["sms"] = int(out[2])
    if lib.mp_peak_l2(48, 5, out) != 0:
        return None
    res["l2_TBps"] = out[0] / 1e12
    res["l2_buffer_mb"] = 48
    res["clocks"] = clocks.stop()
    res["source"] = "paper_2312_04025_b200/csrc/mp_peaks.cu (ld.shared.v4/v2 conflict-free, ld.global.cg over 48 MB)"
    return res


def source_hash() -> str:
    h = hashlib.sha256()
    for p in sorted((ROOT / "paper_2312_04025_b200" / "csrc").glob("*")):
        if p.suffix in (".cu", ".cuh", ".cpp"):
            h.update(p.name.encode())
            h.update(p.read_bytes())
    h.update((ROOT / "include" / "moirai_b200.h").read_bytes())
    return h.hexdigest()[:16]


def ncu_summary(workload: str) -> dict | None:
    """ncu metrics of the headline kernel for THIS source tree (profiles/r02/ncu_<workload>.json,
    written by scripts/ncu_summary.py); ignored when its source hash differs (stale)."""
    p = ROOT / "profiles" / "r02" / f"ncu_{workload}.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
    except Exception:
        return None
    d["current"] = d.get("source_hash") == source_hash()
    return d


# ---- our arm -----------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2312_04025_b200 as mp
    from paper_2312_04025_b200 import _native as N
    from paper_2312_04025_b200 import workloads

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() < (local + 1):
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local}, the box has {torch.cuda.device_count()} GPU(s)")
    torch.cuda.set_device(local)
    # under torchrun the NCCL group is always formed (also at N=1, so the collective
    # path is the one timed on every N)
    use_dist = world > 1 or "MASTER_ADDR" in os.environ
    if use_dist:
        # NCCL prints its version banner on stdout from C; keep stdout for the one JSON line
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    peaks = onchip_peaks() if rank == 0 else None
    w = build_workload(args.workload)
    t0 = time.perf_counter()
    coarse = mp.gcof(w.raw, w.rules, device=local)
    t_gcof = time.perf_counter() - t0  # first call: includes the coarsening context's allocations
    t_warm = []
    for _ in range(5):
        t0 = time.perf_counter()
        mp.gcof(w.raw, w.rules, device=local)
        t_warm.append(time.perf_counter() - t0)
    t_gcof_warm = sorted(t_warm)[len(t_warm) // 2]
    inst = mp.Instance(coarse, w.cluster, mp.effective_bandwidth(w.cluster), device=local)
    if args.tune:
        G, U, rc = (int(x) for x in (args.tune.split(":") + ["0", "0"])[:3])
        inst.tune(G, 0, rc, True, U)
    info = inst.info()
    P = args.rows
    n_ops, n_flows = inst.n_ops, inst.n_flows
    rows = workloads.placements(w.seed + 1000 * rank, P, n_ops, inst.K)
    h_rows = torch.from_numpy(rows).pin_memory()
    d_rows = h_rows.cuda()
    d_ms = torch.empty(P, dtype=torch.float64, device="cuda")
    d_st = torch.empty(P, dtype=torch.int8, device="cuda")
    h_ms = torch.empty(P, dtype=torch.float64).pin_memory()
    stream = torch.cuda.current_stream()
    lib = N.lib()
    err = N.mp_error()
    best = C.c_int64()
    bms = C.c_double()
    gather_in = torch.zeros(2, dtype=torch.int64, device="cuda")
    gather_out = torch.zeros(2 * world, dtype=torch.int64, device="cuda")

    from paper_2312_04025_b200.distributed import combine_records, encode_record

    def exchange():
        """Global keep-best: a 16-byte (makespan bits, global row) record per rank,
        all-gathered over NCCL, lexicographic minimum (paper_2312_04025_b200.distributed)."""
        rec = encode_record(bms.value, best.value + rank * P if best.value >= 0 else -1)
        gather_in.copy_(torch.from_numpy(rec), non_blocking=True)
        if use_dist:
            dist.all_gather_into_tensor(gather_out, gather_in)
            return combine_records(gather_out.cpu().numpy())
        return combine_records(gather_in.cpu().numpy())

    def launch_device():
        code = lib.mp_evaluate_argmin(inst.handle, C.c_void_p(d_rows.data_ptr()), P, C.c_void_p(d_ms.data_ptr()),
                                      C.c_void_p(d_st.data_ptr()), C.byref(best), C.byref(bms), N.MP_DEVICE_PTRS,
                                      C.c_void_p(stream.cuda_stream), C.byref(err))
        N.check(code, err, "mp_evaluate_argmin")

    def step_host():
        code = lib.mp_evaluate_argmin(inst.handle, C.c_void_p(h_rows.data_ptr()), P, C.c_void_p(h_ms.data_ptr()),
                                      None, C.byref(best), C.byref(bms), 0, C.c_void_p(stream.cuda_stream),
                                      C.byref(err))
        N.check(code, err, "mp_evaluate_argmin(host)")
        return exchange()

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if not use_dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        launch_device()
        exchange()
    # ---- timed region: device-resident -------------------------------------------------
    clocks = ClockSampler(local) if rank == 0 else None
    barrier()
    launches0 = lib.mp_launch_count()
    kern_ms = []
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    e_start.record(stream)
    result = None
    for _ in range(args.steps):
        k0 = torch.cuda.Event(enable_timing=True)
        k1 = torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        launch_device()
        k1.record(stream)
        result = exchange()
        kern_ms.append((k0, k1))
    e_end.record(stream)
    barrier()
    launches = lib.mp_launch_count() - launches0
    clk = clocks.stop() if clocks else None
    t_dev = max_over_ranks(e_start.elapsed_time(e_end) / 1e3)
    t_kern = statistics.mean(a.elapsed_time(b) / 1e3 for a, b in kern_ms)
    value = world * P * args.steps / t_dev
    dev_ms = d_ms.cpu().numpy()
    dev_st = d_st.cpu().numpy()
    dev_best = (best.value, bms.value)

    # ---- e2e: host buffers through the C ABI --------------------------------------------
    for _ in range(max(1, args.warmup // 2)):
        step_host()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step_host()
    barrier()
    t_e2e = max_over_ranks(time.perf_counter() - t0)
    e2e = world * P * args.steps / t_e2e
    assert np.array_equal(h_ms.numpy().view(np.uint64), dev_ms.view(np.uint64)), "host/device mismatch"

    # ---- local search throughput (secondary, untimed by the driver) ----------------------
    ls = None
    if args.local_search and rank == 0:
        # K5: one chain per lane of the whole GPU (2^17 chains), warmed up once
        seeds = rows[:64]
        chains, moves = 1 << 17, 32
        mp.local_search(inst, seeds, chains=chains, moves=2, seed=1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, ls_best, _, _ = mp.local_search(inst, seeds, chains=chains, moves=moves, seed=1)
        dt = time.perf_counter() - t0
        ls = {"chains": chains, "moves": moves, "evals_per_s": chains * (moves + 1) / dt, "best_makespan_s": ls_best,
              "note": "every evaluation is a full exact schedule of the mutated placement"}

    out = None
    if rank == 0:
        from oracle.oracle import OracleInstance

        orc = OracleInstance(*inst._arrays)
        parity = parity_check(orc, rows, dev_ms, dev_st, dev_best[0], dev_best[1])
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_dev / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(w, n_ops, n_flows, inst.K),
            "rows_per_gpu": P, "global_rows_per_step": P * world, "parallelism": f"dp{world} (row shards)",
            "shape": {k: info[k] for k in ("group_lanes", "lanes_used", "groups_per_cta", "ctas", "ready_cap", "colo",
                                           "onchip", "smem_bytes") if k in info},
            "gcof_ms": t_gcof_warm * 1e3, "gcof_first_call_ms": t_gcof * 1e3,
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": P * n_ops, "d2h_bytes_per_step": P * 8 + 16},
            "gpu_launches": int(launches),
            "roofline": roofline(P, n_ops, n_flows, t_kern, peaks, ncu_summary(args.workload), info),
            "clocks": clk,
            "parity": parity,
            "best": {"makespan_s": result[0] if result[1] >= 0 else None, "global_row": result[1]},
        }
        if ls:
            out["local_search"] = ls
        if world == 1 and not args.no_cpu:
            out["cpu_baseline"] = cpu_baseline_python(inst._arrays, rows, args.cpu_seconds)
            out["cpu_baseline_native"] = cpu_baseline_native(orc, rows, args.cpu_seconds / 3)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()
    inst.close()
    if out is not None:
        print(json.dumps(out), flush=True)


def roofline(P, n_ops, n_flows, t_kern, peaks, ncu, info) -> dict:
    """Three fractions for the evaluator; `bound` = the tightest.

    * tables: B_tab = 8α + 24β bytes per placement (op cost per op, payload or
      comm entry per flow, 4 B CSR index per augmented link in each of the rank
      and dispatch passes) against the shared-memory load bandwidth measured now
      (L2 when the tables are off-chip);
    * hbm: B_hbm = α + 8 bytes (row in, makespan out) against MEASURED_PEAKS.json;
    * issue: issued warp-instructions per cycle / 4 schedulers per SM, from the ncu
      capture of this exact source tree (null when the capture is stale);
    * alu_pipe / l1_data_pipe: busy fraction of the integer ALU pipe and of the L1 data
      pipe (shared-memory and global wavefronts) in the same capture."""
    hbm_peak, hbm_src = measured_hbm_peak()
    b_hbm = n_ops + 8
    b_tab = 8 * n_ops + 24 * n_flows
    fr = {}
    hbm_ach = P * b_hbm / t_kern / 1e9
    fr["hbm"] = {"achieved": hbm_ach, "peak": hbm_peak, "unit": "GB/s", "frac": hbm_ach / hbm_peak,
                 "algorithmic_bytes_per_placement": b_hbm, "peak_source": hbm_src}
    onchip = bool(info.get("onchip", True)) or info.get("kernel", "").startswith("tpp")
    if peaks:
        pk = peaks["smem_TBps"] if onchip else peaks["l2_TBps"]
        tab_ach = P * b_tab / t_kern / 1e12
        fr["tables"] = {"achieved": tab_ach, "peak": pk, "unit": "TB/s", "frac": tab_ach / pk,
                        "algorithmic_bytes_per_placement": b_tab, "level": "smem" if onchip else "l2",
                        "peak_source": "measured now: " + peaks["source"], "peaks": peaks}
    if ncu and ncu.get("current"):
        ib = ncu.get("issue_slots_busy")
        fr["issue"] = {"achieved": ncu.get("ipc_issued"), "peak": 4.0, "unit": "warp-inst/clk/SM", "frac": ib,
                       "inst_per_placement": ncu.get("inst_per_row"), "source": ncu.get("source")}
        # the two pipes the branch-free dispatch saturates first (ncu pct_of_peak, same capture)
        for key, name in (("alu_pipe_busy", "alu_pipe"), ("l1_data_pipe_busy", "l1_data_pipe")):
            if ncu.get(key) is not None:
                fr[name] = {"achieved": ncu[key], "peak": 1.0, "unit": "fraction of peak cycles",
                            "frac": ncu[key], "source": ncu.get("source")}
    bound = max(fr, key=lambda k: fr[k]["frac"] or 0.0)
    top = fr[bound]
    traffic = None
    if ncu and ncu.get("current") and ncu.get("dram_bytes_per_row") is not None:
        traffic = ncu["dram_bytes_per_row"] * P
    return {"bound": bound, "achieved": top["achieved"], "peak": top["peak"], "unit": top["unit"],
            "frac": top["frac"], "traffic": traffic, "kernel_ms": t_kern * 1e3, "fractions": fr,
            "ncu": ({k: ncu[k] for k in ("source_hash", "so_sha256", "current", "kernel", "dram_bytes_per_row",
                                          "ipc_issued", "issue_slots_busy", "warps_per_sm", "l2_hit_rate",
                                          "smem_wavefronts_per_row") if k in ncu} if ncu else None),
            "source_hash": source_hash()}


# ---- reference arm -------------------------------------------------------------------------
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import pyref
    from paper_2312_04025_b200 import workloads

    w = build_workload(args.workload)
    g = coarse_on_cpu(w)
    arrays = flat_arrays(g, w.cluster)
    n_ops = len(g)
    n_flows = len(arrays[2])
    K = len(w.cluster.device_ids)
    cores = os.cpu_count() or 1
    # size one step for ~args.ref_step_s seconds of all-core work
    inst = pyref.Instance.from_arrays(arrays)
    probe = workloads.placements(w.seed, 20, n_ops, K)
    t0 = time.perf_counter()
    pyref.eval_rows(inst, probe)
    per_row = (time.perf_counter() - t0) / 20
    n = int(max(cores * 2, args.ref_step_s / per_row * cores))
    rows = workloads.placements(w.seed, n * (args.steps + args.warmup), n_ops, K)
    import multiprocessing as mpc

    procs = cores
    ctx = mpc.get_context("fork")
    with ctx.Pool(procs, initializer=pyref._worker_init, initargs=(arrays,)) as pool:
        pool.map(pyref._worker_rows, [rows[i:i + 1] for i in range(procs)])
        for s in range(args.warmup):
            chunk = rows[s * n:(s + 1) * n]
            pool.map(pyref._worker_rows, [chunk[i::procs] for i in range(procs)])
        t0 = time.perf_counter()
        for s in range(args.warmup, args.warmup + args.steps):
            chunk = rows[s * n:(s + 1) * n]
            pool.map(pyref._worker_rows, [chunk[i::procs] for i in range(procs)])
        dt = time.perf_counter() - t0
    value = n * args.steps / dt
    sample = (f"{n} placements per step of the {w.name} stream (GCOF {len(w.raw)} -> {n_ops} ops), pure-Python "
              f"restatement of opplace._schedule (oracle/pyref.py), {procs} processes")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": workload_config(w, n_ops, n_flows, K),
           "rows_per_step": n, "parallelism": f"{procs} host processes",
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_distributed(args) -> int:
    """`--gpus N` outside torchrun: start N ranks ourselves (same contract as the
    driver's torchrun launch).  Refuses when the box has fewer than N GPUs."""
    import torch

    have = torch.cuda.device_count()
    if args.impl == "ours" and have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} requested but this box has {have} GPU(s)", file=sys.stderr)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default="c2k8", choices=WORKLOADS)
    ap.add_argument("--rows", type=int, default=1 << 20, help="placements per GPU per step")
    ap.add_argument("--tune", default="", help="G:U:ready_cap launch-shape override")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-step-s", type=float, default=2.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-local-search", dest="local_search", action="store_false")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "reference":
            run_reference(args)  # host CPU arm: rank 0 only, nothing to launch
            return
        sys.exit(relaunch_distributed(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
