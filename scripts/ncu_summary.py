#!/usr/bin/env python3
"""Distil an `ncu --set full` capture of the headline evaluator kernel into
profiles/r02/ncu_<workload>.json, stamped with the source hash of the tree that
was profiled (bench.py ignores the file once the sources change).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep --workload c2k8 --rows 1048576 \
        [--kernel mp_tpps_kernel] [--out profiles/r02/ncu_c2k8.json]
"""

from __future__ import annotations

import argparse
import csv
import hashlib
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

METRICS = {
    "gpu__time_duration.sum": "time_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__inst_executed.sum": "inst",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.per_cycle_active": "warps",
    "lts__t_sector_hit_rate.pct": "l2_hit",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_conflicts",
    "launch__registers_per_thread": "regs",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pct",
    "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed": "l1_wavefronts_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefronts_pct",
}


def _num(s: str):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


_SCALE = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9,
          "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def read_raw(rep: str, kernel: str) -> list[dict]:
    """Raw-page metrics of every launch of `kernel`, times in ns and sizes in bytes."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        if kernel in d.get("Kernel Name", ""):
            for h, u in zip(head, units):
                if u in _SCALE and _num(d[h]) is not None:
                    d[h] = str(_num(d[h]) * _SCALE[u])
            out.append(d)
    return out


def main():
    from bench import source_hash

    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--rows", type=int, required=True, help="placements per launch")
    ap.add_argument("--kernel", default="mp_tpps_kernel")
    ap.add_argument("--out")
    a = ap.parse_args()
    launches = read_raw(a.report, a.kernel)
    if not launches:
        raise SystemExit(f"no {a.kernel} launch in {a.report}")
    d = launches[-1]
    m = {v: _num(d.get(k, "")) for k, v in METRICS.items()}
    so = ROOT / "paper_2312_04025_b200" / "libmoirai_b200.so"
    res = {
        "kernel": d.get("Kernel Name"),
        "workload": a.workload,
        "rows_per_launch": a.rows,
        "kernel_ms": m["time_ns"] / 1e6 if m["time_ns"] else None,
        "dram_bytes_per_row": ((m["dram_read"] or 0) + (m["dram_write"] or 0)) / a.rows,
        "inst_per_row": m["inst"] / a.rows if m["inst"] else None,
        "ipc_issued": m["ipc"],
        "issue_slots_busy": m["issue_pct"] / 100 if m["issue_pct"] is not None else None,
        "warps_per_sm": m["warps"],
        "l2_hit_rate": m["l2_hit"] / 100 if m["l2_hit"] is not None else None,
        "smem_wavefronts_per_row": m["smem_wavefronts"] / a.rows if m["smem_wavefronts"] else None,
        "smem_conflict_share": (m["smem_conflicts"] / m["smem_wavefronts"]) if m["smem_wavefronts"] else None,
        "registers": m["regs"],
        "threads_per_inst": m["threads_per_inst"],
        # pipe utilisation: the integer ALU pipe (selects, logic, compares: half the issue
        # rate of the FMA pipe) and the L1 data pipe (shared-memory + global wavefronts)
        "alu_pipe_busy": m["alu_pct"] / 100 if m["alu_pct"] is not None else None,
        "fma_pipe_busy": m["fma_pct"] / 100 if m["fma_pct"] is not None else None,
        "fp64_pipe_busy": m["fp64_pct"] / 100 if m["fp64_pct"] is not None else None,
        "l1_data_pipe_busy": m["l1_wavefronts_pct"] / 100 if m["l1_wavefronts_pct"] is not None else None,
        "smem_data_pipe_busy": m["smem_wavefronts_pct"] / 100 if m["smem_wavefronts_pct"] is not None else None,
        "source": f"ncu --set full --clock-control none ({Path(a.report).name}), last {a.kernel} launch",
        "source_hash": source_hash(),
        "so_sha256": hashlib.sha256(so.read_bytes()).hexdigest()[:16] if so.exists() else None,
    }
    out = Path(a.out) if a.out else ROOT / "profiles" / "r02" / f"ncu_{a.workload}.json"
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
