"""Developer sanity run on a GPU box: parity spot checks + rough timings.

Usage: python scripts/gpu_sanity.py   (writes a summary to stdout)
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_2312_04025_b200 as mp  # noqa: E402
from oracle.oracle import OracleInstance, gcof_partition  # noqa: E402
from paper_2312_04025_b200 import workloads  # noqa: E402


def check_workload(w, P=2048):
    t0 = time.perf_counter()
    coarse = mp.gcof(w.raw, w.rules)
    t_gcof = time.perf_counter() - t0
    fl = mp.fusion._Flat(w.raw, w.rules, None)
    k = fl.keep
    part = gcof_partition(k[1], k[2], k[3], k[6], k[7], k[10], k[11])
    idx = w.raw.csr().index
    got = [[idx[m] for m in n.members] for n in coarse.nodes]
    gcof_ok = got == [p for p, _ in part]
    mesh = mp.effective_bandwidth(w.cluster)
    inst = mp.Instance(coarse, w.cluster, mesh)
    info = inst.info()
    rows = workloads.placements(w.seed, P, inst.n_ops, inst.K)
    ms, st, dev, ov = mp.evaluate_batch(inst, rows, with_detail=True)
    orc = OracleInstance.from_instance(inst)
    t0 = time.perf_counter()
    want, wst = orc.eval_batch(rows, threads=8)
    t_orc = time.perf_counter() - t0
    eq = np.array_equal(st, wst) and np.array_equal(ms.view(np.uint64), want.view(np.uint64))
    nbad = int(np.sum(ms.view(np.uint64) != want.view(np.uint64)))
    # schedule_one on row 0
    s, oms, ost, oen, _, _ = orc.schedule(rows[0])
    try:
        sched = mp.solver._schedule_row(inst, rows[0])
        starts = [sched.starts[i] for i in inst.op_ids] + [sched.starts[inst.flow_id(f)] for f in range(inst.n_flows)]
        one_ok = np.array_equal(np.array(starts), ost) and sched.makespan_s == oms
    except mp.MemoryExceededError:
        one_ok = s == 1
    # throughput (device-resident would be in bench; this is host-pointer e2e)
    big = workloads.placements(w.seed, 1 << 16, inst.n_ops, inst.K)
    mp.evaluate_batch(inst, big[:4096])
    t0 = time.perf_counter()
    mp.evaluate_batch(inst, big)
    dt = time.perf_counter() - t0
    print(f"{w.name}: raw {len(w.raw)} -> {inst.n_ops}/{inst.n_flows} gcof {t_gcof*1e3:.1f} ms ok={gcof_ok}; "
          f"eval parity {eq} (bad {nbad}/{P}) feasible {int((st==0).sum())}/{P}; schedule_one ok={one_ok}; "
          f"info G={info['group_lanes']} rcap={info['ready_cap']} onchip={info['onchip']} gpc={info['groups_per_cta']} "
          f"ctas={info['ctas']} smem={info['smem_bytes']}; gpu {len(big)/dt:,.0f} pl/s (host e2e) ; "
          f"oracle 8 thr {P/t_orc:,.0f} pl/s", flush=True)
    return inst, rows


def main():
    print("devices", mp._native.lib().mp_device_count())
    for w in (workloads.c1(), workloads.c2(4), workloads.c2(8), workloads.c4()):
        inst, rows = check_workload(w)
    # enumeration vs oracle on small instance
    import random
    rng = random.Random(5)
    for trial in range(5):
        n = 10
        nodes = [mp.OpNode(i, "conv", rng.randint(1, 30), {d: round(rng.uniform(0.5, 8), 3) for d in range(3)})
                 for i in range(1, n + 1)]
        edges = [mp.FlowEdge(i, j, rng.randint(10 ** 6, 3 * 10 ** 7)) for j in range(2, n + 1) for i in range(1, j)
                 if rng.random() < 0.4]
        g = mp.CompGraph(nodes, edges)
        c = mp.Cluster([mp.Device(d, 80) for d in range(3)],
                       {(a, b): rng.uniform(4e6, 4e7) for a in range(3) for b in range(3) if a != b})
        sol = mp.brute_force(g, c, mp.effective_bandwidth(c))
        inst = mp.Instance(g, c, mp.effective_bandwidth(c))
        order = mp.topo_order(g)
        pos = {x: i for i, x in enumerate(inst.op_ids)}
        idx, bms = OracleInstance.from_instance(inst).enumerate([pos[x] for x in order])
        ok = (sol.objective_s == bms) if idx >= 0 else sol.status == mp.Status.INFEASIBLE
        print(f"brute_force trial {trial}: gpu {sol.objective_s!r} oracle {bms!r} ok={ok}")
    w = workloads.c2(4)
    coarse = mp.gcof(w.raw, w.rules)
    inst = mp.Instance(coarse, w.cluster, mp.effective_bandwidth(w.cluster))
    seeds = workloads.placements(2, 8, inst.n_ops, inst.K)
    t0 = time.perf_counter()
    row, bms, bc, cms = mp.local_search(inst, seeds, chains=2048, moves=64, seed=1)
    dt = time.perf_counter() - t0
    orc = OracleInstance.from_instance(inst)
    s, oms, *_ = orc.schedule(row)
    print(f"local search: best {bms!r} chain {bc} reverify {oms == bms}; {2048*65/dt:,.0f} evals/s")


if __name__ == "__main__":
    main()
