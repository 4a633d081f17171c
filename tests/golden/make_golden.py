"""Generate the golden fixtures from the REFERENCE package itself.

Run here (the container that has /root/reference):
    PYTHONPATH=/root/repo python tests/golden/make_golden.py

Writes tests/golden/*.json.  Every float is stored with float.hex() so the
fixtures pin bit-exact values.  The GPU box never reads /root/reference; it
only reads these committed files.

Populations (reference test file:line they come from):
* schedules   random_instance seeds 2000-2039 (test_simulator.py:74-89),
              9001-9050 (test_acceptance.py:61-66), fixtures two_op_chain,
              split_chain, skewed_pair, residual_block (conftest.py:41-99)
* brute force the 50-instance acceptance population (test_acceptance.py:61-84)
              and seeds 40-54 (test_solver.py:90-102)
* gcof        random_dag seeds 0-199 (test_fusion.py:238-276 uses 0-99 at
              max_ops=14), the frozen residual block (test_fusion.py:158-179),
              SURVEY App. B contested pairs, test_fusion.py single cases,
              GenSpec(56,4,0.6) seed 2 (test_acceptance.py:245-248), the C1-C4
              raw graphs, overrides (test_fusion.py:313-321)
* workloads   C1-C4 coarse graphs + 16 seeded placements each: reference makespans
* synth       sha256 of gen_synthetic outputs for the C1/C5 specs
* simulate    reference ``simulate`` event lists: random_instance seeds 2000-2039
              (test_simulator.py:74-89) and 0-19 (test_simulator.py:60-71), the
              frozen fixtures (test_simulator.py:25-57), graphs whose costs are
              missing on devices no op is placed on (simulator.py:85-96), and the
              validation errors (unknown device, missing placed cost, memory)
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, str(HERE.parents[1]))

import conftest as rc  # noqa: E402  (reference fixtures)
import opplace as ref  # noqa: E402
from opplace import solver as rsolver  # noqa: E402

import paper_2312_04025_b200 as mp  # noqa: E402
from paper_2312_04025_b200 import workloads  # noqa: E402


def H(x: float) -> str:
    return float(x).hex()


def ser_graph(g) -> dict:
    return {
        "nodes": [[n.id, n.op_type, n.mem_bytes, {str(k): H(v) for k, v in n.compute_time.items()},
                   list(n.members), list(n.type_seq), n.tag.value] for n in g.nodes],
        "edges": [[e.src, e.dst, e.payload_bytes] for e in g.edges],
    }


def ser_cluster(c) -> dict:
    return {"devices": [[d.id, d.mem_bytes] for d in c.devices],
            "links": [[a, b, H(bw)] for (a, b), bw in c.links.items()]}


def ser_mesh(m) -> list:
    return [[a, b, H(bw)] for (a, b), bw in sorted(m.bw.items())]


def to_ref_graph(g):
    return ref.CompGraph([ref.OpNode(n.id, n.op_type, n.mem_bytes, dict(n.compute_time), n.members, n.type_seq,
                                     ref.Tag(n.tag.value)) for n in g.nodes],
                         [ref.FlowEdge(e.src, e.dst, e.payload_bytes) for e in g.edges])


def to_ref_cluster(c):
    return ref.Cluster([ref.Device(d.id, d.mem_bytes) for d in c.devices], dict(c.links))


def to_ref_rules(rules):
    return ref.FusionRuleSet([ref.FusionRule(r.id, r.pattern) for r in rules])


def schedule_record(inst, g, assign):
    try:
        s = rsolver._schedule(inst, assign)
    except ref.MemoryExceededError as e:
        return {"status": "memory", "device": e.device, "overflow": e.overflow}
    return {"status": "ok", "makespan": H(s.makespan_s),
            "starts": {str(k): H(v) for k, v in s.starts.items()},
            "ends": {str(k): H(v) for k, v in s.ends.items()},
            "channels": {str(k): (list(v) if v else None) for k, v in s.channels.items()}}


def make_schedules():
    cases = []

    def add(tag, g, c, assigns):
        mesh = ref.effective_bandwidth(c)
        inst = rsolver._Instance(g, c, mesh)
        cases.append({"name": tag, "graph": ser_graph(g), "cluster": ser_cluster(c), "mesh": ser_mesh(mesh),
                      "assignments": [{str(k): v for k, v in a.items()} for a in assigns],
                      "results": [schedule_record(inst, g, a) for a in assigns]})

    for trial in range(40):
        rng = random.Random(2000 + trial)
        g, c = rc.random_instance(rng, tight_ok=False)
        add(f"sim-{2000 + trial}", g, c, [{i: rng.choice(c.device_ids) for i in g.node_ids} for _ in range(5)])
    for trial in range(50):
        rng = random.Random(9001 + trial)
        g, c = rc.random_instance(rng, max_ops=8, tight_ok=True, min_ops=3)
        r2 = random.Random(77 + trial)
        add(f"acc-{9001 + trial}", g, c, [{i: r2.choice(c.device_ids) for i in g.node_ids} for _ in range(6)])
    g, c = rc.two_op_chain()
    add("two_op_chain", g, c, [{1: 0, 2: 1}, {1: 1, 2: 1}, {1: 0, 2: 0}, {1: 1, 2: 0}])
    g, c = rc.split_chain()
    add("split_chain", g, c, [{1: 0, 2: 1}, {1: 1, 2: 0}])
    g, c = rc.skewed_pair()
    add("skewed_pair", g, c, [{1: 2, 2: 2}, {1: 1, 2: 2}, {1: 1, 2: 1}])
    g = rc.residual_block()
    c = rc.two_device_cluster(mem=10 ** 6)
    r3 = random.Random(5)
    add("residual_block", g, c, [{i: r3.choice([0, 1]) for i in g.node_ids} for _ in range(8)])
    c = rc.two_device_cluster(mem=10)
    g = ref.CompGraph([ref.OpNode(1, "conv", 5, {0: 2.0, 1: 50.0}), ref.OpNode(2, "bn", 5, {0: 3.0, 1: 50.0})], [])
    add("serialization", g, c, [{1: 0, 2: 0}])
    return cases


def make_brute():
    cases = []

    def add(tag, g, c):
        mesh = ref.effective_bandwidth(c)
        sol = ref.brute_force(g, c, mesh)
        rec = {"name": tag, "graph": ser_graph(g), "cluster": ser_cluster(c), "status": sol.status.value,
               "objective": H(sol.objective_s)}
        if sol.schedule is not None:
            rec["placement"] = {str(k): v for k, v in sol.placement.items()}
        cases.append(rec)

    for trial in range(50):
        g, c = rc.random_instance(random.Random(9001 + trial), max_ops=8, tight_ok=True, min_ops=3)
        add(f"acc-{9001 + trial}", g, c)
    for trial in range(15):
        g, c = rc.random_instance(random.Random(40 + trial), max_ops=5)
        add(f"solver-{40 + trial}", g, c)
    for name, fn in (("two_op_chain", rc.two_op_chain), ("split_chain", rc.split_chain),
                     ("skewed_pair", rc.skewed_pair)):
        g, c = fn()
        add(name, g, c)
    return cases


def gcof_record(name, g, rules, overrides=None):
    out = ref.gcof(g, rules, overrides)
    rec = {"name": name, "graph": ser_graph(g), "rules": [[r.id, list(r.pattern)] for r in rules],
           "out": ser_graph(out)}
    if overrides is not None:
        rec["overrides"] = [[list(s), k, H(t)] for (s, k), t in overrides.entries.items()]
    return rec


def make_gcof():
    cases = []
    rules = rc.table_rules()
    for seed in range(200):
        cases.append(gcof_record(f"random_dag14-{seed}", rc.random_dag(random.Random(seed), max_ops=14), rules))
    for seed in range(100):
        cases.append(gcof_record(f"random_dag10-{seed}", rc.random_dag(random.Random(seed)), rules))
    cases.append(gcof_record("residual_block", rc.residual_block(), rules))

    def node(i, t, **kw):
        return ref.OpNode(i, t, kw.pop("mem", 1), kw.pop("times", {0: 1.0}), **kw)

    E = ref.FlowEdge
    cases.append(gcof_record("appB-conv-conv-bn",
                             ref.CompGraph([node(1, "conv"), node(2, "conv"), node(3, "bn")], [E(1, 3, 1), E(2, 3, 1)]),
                             rules))
    cases.append(gcof_record("appB-pool-conv-bn",
                             ref.CompGraph([node(1, "pool"), node(2, "conv"), node(3, "bn")], [E(1, 3, 1), E(2, 3, 1)]),
                             rules))
    cases.append(gcof_record("bound-prefix", ref.CompGraph(
        [node(1, "conv"), node(2, "bn"), node(3, "add"), node(4, "pool")], [E(1, 2, 1), E(2, 3, 2), E(3, 4, 3)]), rules))
    cases.append(gcof_record("dissolve", ref.CompGraph([node(1, "conv"), node(2, "bn"), node(3, "pool")],
                                                       [E(1, 2, 1), E(2, 3, 2)]),
                             ref.FusionRuleSet([ref.FusionRule(5, ("conv", "bn", "relu"))])))
    fj = ref.CompGraph([node(1, "conv"), node(2, "bn"), node(3, "relu"), node(4, "add")],
                       [E(1, 2, 1), E(1, 3, 1), E(2, 4, 1), E(3, 4, 1)])
    cases.append(gcof_record("fork", fj, rules))
    cases.append(gcof_record("multi-input-join", ref.CompGraph(
        [node(1, "conv"), node(2, "bn"), node(3, "add"), node(4, "relu"), node(5, "pool")],
        [E(1, 2, 1), E(2, 3, 2), E(5, 3, 9), E(3, 4, 3)]), rules))
    ov = ref.CostOverrides({(("conv", "bn", "relu"), 0): 4.25})
    cases.append(gcof_record("override", ref.CompGraph(
        [node(1, "conv", times={0: 2.0}), node(2, "bn", times={0: 3.0}), node(3, "relu", times={0: 1.0})],
        [E(1, 2, 1), E(2, 3, 1)]), rules, ov))
    ov2 = ref.CostOverrides({(("conv", "bn"), 0): 3.5, (("conv", "bn"), 7): 1.25})
    cases.append(gcof_record("override-extra-device", ref.CompGraph(
        [node(1, "conv", times={0: 2.0, 1: 4.0}), node(2, "bn", times={0: 3.0, 1: 1.0}), node(3, "pool")],
        [E(1, 2, 100), E(2, 3, 5)]), rules, ov2))
    # pre-fused input nodes and input BOUND tags
    pre = ref.CompGraph([
        ref.OpNode(1, "conv∘bn", 3, {0: 1.5, 1: 2.5}, members=(1, 11), type_seq=("conv", "bn"), tag=ref.Tag.FUSED),
        node(2, "relu", times={0: 0.25, 1: 0.5}),
        ref.OpNode(3, "conv", 1, {0: 1.0, 1: 1.0}, tag=ref.Tag.BOUND), node(4, "pool", times={0: 1.0, 1: 1.0})],
        [E(1, 2, 7), E(3, 4, 8), E(2, 3, 9)])
    cases.append(gcof_record("prefused-input", pre, rules))
    # order-sensitive rules: (a,b) and (b,c) compete on a -> b -> c
    abc = ref.FusionRuleSet([ref.FusionRule(1, ("a", "b")), ref.FusionRule(2, ("b", "c"))])
    cases.append(gcof_record("abc-chain", ref.CompGraph([node(1, "a"), node(2, "b"), node(3, "c")],
                                                        [E(1, 2, 1), E(2, 3, 1)]), abc))
    cases.append(gcof_record("abc-visited-first", ref.CompGraph(
        [node(1, "x"), node(2, "b"), node(3, "c"), node(4, "a")], [E(1, 2, 1), E(2, 3, 1), E(4, 2, 1)]), abc))
    for seed in range(60):
        rng = random.Random(10_000 + seed)
        n = rng.randint(3, 16)
        types = ("a", "b", "c", "d")
        nodes = [ref.OpNode(i, rng.choice(types), rng.randint(1, 9),
                            {0: rng.uniform(0.1, 3.0), 1: rng.uniform(0.1, 3.0) * 10 ** rng.randint(-8, 8)})
                 for i in range(1, n + 1)]
        edges = [E(i, j, rng.randint(1, 100)) for j in range(2, n + 1) for i in range(1, j) if rng.random() < 0.3]
        g = ref.CompGraph(nodes, edges)
        rr = ref.FusionRuleSet([ref.FusionRule(1, ("a", "b")), ref.FusionRule(2, ("b", "c")),
                                ref.FusionRule(3, ("a", "b", "c", "d")), ref.FusionRule(4, ("c", "d"))])
        cases.append(gcof_record(f"abcd-{seed}", g, rr))
    g = ref.gen_synthetic(ref.GenSpec(ops=56, width=4, density=0.6, devices=(0, 1, 2, 3)), seed=2)
    cases.append(gcof_record("acceptance-56", g, rules))
    g = ref.gen_synthetic(ref.GenSpec(ops=18, width=1, density=1.0, devices=(0, 1),
                                      patterns=(("conv", "bn", "relu"),)), 42)
    cases.append(gcof_record("synth-18-chain", g, rules))
    for w in (workloads.c1(), workloads.c2(4), workloads.c3(), workloads.c4()):
        cases.append(gcof_record(w.name, to_ref_graph(w.raw), to_ref_rules(w.rules)))
    for spec, seed in ((ref.GenSpec(ops=2000, width=16, density=0.5, devices=(0, 1)), 3),):
        cases.append(gcof_record(f"synth-{spec.ops}", ref.gen_synthetic(spec, seed), rules))
    return cases


def make_workload_evals():
    out = []
    for w in (workloads.c1(), workloads.c2(4), workloads.c2(8), workloads.c3(), workloads.c4("nvlink"),
              workloads.c4("pcie")):
        g = ref.gcof(to_ref_graph(w.raw), to_ref_rules(w.rules))
        c = to_ref_cluster(w.cluster)
        mesh = ref.effective_bandwidth(c)
        inst = rsolver._Instance(g, c, mesh)
        rows = workloads.placements(w.seed, 16, len(g), len(c))
        devs = c.device_ids
        ops = g.node_ids
        res = []
        for row in rows:
            a = {op: devs[int(k)] for op, k in zip(ops, row)}
            r = schedule_record(inst, g, a)
            r.pop("starts", None)
            r.pop("ends", None)
            r.pop("channels", None)
            res.append(r)
        out.append({"name": w.name, "n_ops": len(g), "n_flows": len(g.edges),
                    "coarse_sha256": hashlib.sha256(json.dumps(ser_graph(g), sort_keys=True).encode()).hexdigest(),
                    "rows_seed": w.seed, "results": res})
    return out


def make_solve_exact():
    """Reference solve_exact (solver.py:172-254) under gap / node-limit budgets."""
    cases = []

    def add(tag, g, c, gap, node_limit):
        mesh = ref.effective_bandwidth(c)
        sol = ref.solve_exact(g, c, mesh, ref.SolveBudget(gap=gap, node_limit=node_limit))
        rec = {"name": tag, "graph": ser_graph(g), "cluster": ser_cluster(c), "status": sol.status.value,
               "objective": H(sol.objective_s), "gap": H(gap), "node_limit": node_limit}
        if sol.schedule is not None:
            rec["placement"] = {str(k): v for k, v in sol.placement.items()}
        cases.append(rec)

    for trial in range(50):
        g, c = rc.random_instance(random.Random(9001 + trial), max_ops=8, tight_ok=True, min_ops=3)
        add(f"acc-{9001 + trial}-gap0.3", g, c, 0.3, None)
        add(f"acc-{9001 + trial}-nodes{7 + 13 * trial}", g, c, 0.0, 7 + 13 * trial)
    for trial in range(20):
        g, c = rc.random_instance(random.Random(500 + trial), max_ops=10, tight_ok=True, min_ops=6)
        add(f"rnd-{500 + trial}", g, c, 0.0, None)
        add(f"rnd-{500 + trial}-gap0.1", g, c, 0.1, None)
    g, c = rc.skewed_pair()
    add("skewed_pair-gap0.5", g, c, 0.5, None)
    g, c = rc.random_instance(random.Random(3), max_ops=6, tight_ok=False)
    add("node_limit_1", g, c, 0.0, 1)
    # the acceptance-8 coarse graph (test_acceptance.py:244-263) under node limits
    g = ref.gen_synthetic(ref.GenSpec(ops=56, width=4, density=0.6, devices=(0, 1, 2, 3)), seed=2)
    coarse = ref.gcof(g, rc.table_rules())
    bw = [2e7, 5e7, 1e8, 2e8]
    c = ref.Cluster([ref.Device(k, 6_000_000_000) for k in range(4)],
                    {(a, b): bw[(a + b) % 4] for a in range(4) for b in range(4) if a != b})
    for nl in (500, 5000):
        add(f"accept8-nodes{nl}", coarse, c, 0.05, nl)
    return cases


def _ser_sched(s):
    return {"assignment": {str(k): v for k, v in s.assignment.items()},
            "starts": {str(k): H(v) for k, v in s.starts.items()}, "ends": {str(k): H(v) for k, v in s.ends.items()},
            "channels": {str(k): (list(v) if v else None) for k, v in s.channels.items()}, "makespan": H(s.makespan_s)}


def make_aux():
    """greedy_place (baselines.py:27-86), check_feasibility (simulator.py:179-264)
    and fuse (fusion.py:251-268) outputs of the reference."""
    import copy

    from opplace import baselines as rb
    from opplace import simulator as rs

    greedy, audit, fuse = [], [], []

    def add_greedy(tag, g, c):
        mesh = ref.effective_bandwidth(c)
        for kind in (rb.BaselineKind.EARLIEST_FINISH, rb.BaselineKind.EARLIEST_START):
            rec = {"name": tag, "kind": kind.value, "graph": ser_graph(g), "cluster": ser_cluster(c)}
            try:
                rec["schedule"] = _ser_sched(rb.greedy_place(g, c, mesh, kind))
            except ref.InfeasibleMemoryError as e:
                rec["error"] = [e.needed, e.available]
            greedy.append(rec)

    for trial in range(50):
        g, c = rc.random_instance(random.Random(9001 + trial), max_ops=8, tight_ok=True, min_ops=3)
        add_greedy(f"acc-{9001 + trial}", g, c)
    for trial in range(20):
        g, c = rc.random_instance(random.Random(700 + trial), max_ops=12, tight_ok=True, min_ops=6)
        add_greedy(f"rnd-{700 + trial}", g, c)
    for name in ("two_op_chain", "split_chain", "skewed_pair"):
        g, c = getattr(rc, name)()
        add_greedy(name, g, c)
    for w in (workloads.c1(), workloads.c2(4)):
        add_greedy(w.name, ref.gcof(to_ref_graph(w.raw), to_ref_rules(w.rules)), to_ref_cluster(w.cluster))

    def add_audit(tag, g, c, sched, tol=0.0):
        mesh = ref.effective_bandwidth(c)
        out = rs.check_feasibility(sched, g, c, mesh, tol)
        audit.append({"name": tag, "graph": ser_graph(g), "cluster": ser_cluster(c), "schedule": _ser_sched(sched),
                      "tol": H(tol), "violations": [[v.kind.value, v.details, list(v.nodes)] for v in out]})

    for trial in range(30):
        rng = random.Random(3000 + trial)
        g, c = rc.random_instance(rng, tight_ok=trial % 3 == 0)
        mesh = ref.effective_bandwidth(c)
        assign = {i: rng.choice(c.device_ids) for i in g.node_ids}
        try:
            sched = ref.schedule_for_assignment(g, c, mesh, assign)
        except ref.MemoryExceededError:
            continue
        add_audit(f"clean-{trial}", g, c, sched)
        # deterministic corruptions of the canonical schedule
        nodes = sorted(sched.starts)
        for m in range(4):
            bad = copy.deepcopy(sched)
            pick = nodes[(trial * 7 + m * 3) % len(nodes)]
            if m == 0:      # shift a node earlier: precedence / overlap breaks
                bad.starts[pick] -= 0.75
                bad.ends[pick] -= 0.75
            elif m == 1:    # stretch a node: duration mismatch
                bad.ends[pick] += 0.5
            elif m == 2:    # pull everything to time zero: overlaps everywhere
                for n in nodes:
                    d = bad.ends[n] - bad.starts[n]
                    bad.starts[n] = 0.0
                    bad.ends[n] = d
            else:           # negative start
                bad.starts[pick] = -1.0
            add_audit(f"bad-{trial}-{m}", g, c, bad)
            if m == 1:
                add_audit(f"bad-{trial}-{m}-tol", g, c, bad, tol=0.6)
    # memory over: the same schedule audited against a smaller cluster
    g, c = rc.random_instance(random.Random(3100), tight_ok=False)
    mesh = ref.effective_bandwidth(c)
    sched = ref.schedule_for_assignment(g, c, mesh, {i: c.device_ids[0] for i in g.node_ids})
    small = ref.Cluster([ref.Device(d.id, 1) for d in c.devices], dict(c.links))
    add_audit("memory-over", g, small, sched)

    def add_fuse(tag, g, a, b, ov=None):
        rec = {"name": tag, "graph": ser_graph(g), "pred": a, "succ": b,
               "overrides": None if ov is None else [[list(s), k, H(t)] for (s, k), t in ov.entries.items()]}
        try:
            out, merged = ref.fuse(g, a, b, ov)
            rec["out"] = ser_graph(out)
            rec["merged"] = merged.id
        except ref.OpPlaceError as e:
            rec["error"] = type(e).__name__
        fuse.append(rec)

    rb_g = rc.residual_block()
    for e in rb_g.edges:
        add_fuse(f"residual-{e.src}-{e.dst}", rb_g, e.src, e.dst)
    add_fuse("residual-missing", rb_g, 9, 1)
    for seed in range(20):
        g = rc.random_dag(random.Random(seed), max_ops=10)
        for e in g.edges[:4]:
            add_fuse(f"dag-{seed}-{e.src}-{e.dst}", g, e.src, e.dst)
    tri = ref.CompGraph([ref.OpNode(1, "conv", 1, {0: 1.0}), ref.OpNode(2, "bn", 1, {0: 1.0}),
                         ref.OpNode(3, "relu", 1, {0: 1.0})],
                        [ref.FlowEdge(1, 2, 1), ref.FlowEdge(2, 3, 1), ref.FlowEdge(1, 3, 1)])
    add_fuse("triangle", tri, 1, 3)
    two = ref.CompGraph([ref.OpNode(1, "conv", 10, {0: 2.0, 1: 4.0}), ref.OpNode(2, "bn", 5, {0: 3.0, 1: 1.0})],
                        [ref.FlowEdge(1, 2, 100)])
    add_fuse("override", two, 1, 2, ref.CostOverrides({(("conv", "bn"), 0): 3.5}))
    return {"greedy": greedy, "audit": audit, "fuse": fuse}


def make_synth():
    out = []
    for ops, width, dens, devs, seed in ((490, 4, 0.5, (0, 1), 2312), (490, 4, 0.5, (0, 1), 1),
                                         (1000, 32, 0.5, (0, 1, 2, 3), 0), (5000, 32, 0.5, tuple(range(8)), 0)):
        spec = ref.GenSpec(ops=ops, width=width, density=dens, devices=devs,
                           mem_range=(1_000_000, 64_000_000) if seed == 2312 else (1_000_000, 256_000_000))
        g = ref.gen_synthetic(spec, seed)
        out.append({"ops": ops, "width": width, "density": dens, "devices": list(devs), "seed": seed,
                    "mem_range": list(spec.mem_range),
                    "sha256": hashlib.sha256(json.dumps(ser_graph(g), sort_keys=True).encode()).hexdigest()})
    return out


def _ser_events(events) -> list:
    return [[H(e.time_s), e.kind.value, e.node, e.device, list(e.channel) if e.channel else None] for e in events]


def make_simulate():
    cases = []

    def add(tag, g, c, assigns):
        mesh = ref.effective_bandwidth(c)
        res = []
        for a in assigns:
            try:
                ms, ev = ref.simulate(g, c, mesh, a)
                res.append({"status": "ok", "makespan": H(ms), "events": _ser_events(ev)})
            except ref.MemoryExceededError as e:
                res.append({"status": "memory", "device": e.device, "overflow": e.overflow})
            except ref.MissingCostError as e:
                res.append({"status": "missing", "op": e.op, "device": e.device})
            except KeyError as e:
                res.append({"status": "keyerror", "message": str(e)})
        cases.append({"name": tag, "graph": ser_graph(g), "cluster": ser_cluster(c),
                      "assignments": [{str(k): v for k, v in a.items()} for a in assigns], "results": res})

    for trial in range(40):
        rng = random.Random(2000 + trial)
        g, c = rc.random_instance(rng, tight_ok=False)
        add(f"sweep-{2000 + trial}", g, c, [{i: rng.choice(c.device_ids) for i in g.node_ids}])
    for trial in range(20):
        rng = random.Random(trial)
        g, c = rc.random_instance(rng, tight_ok=False)
        add(f"sorted-{trial}", g, c, [{i: rng.choice(c.device_ids) for i in g.node_ids}])
    c = rc.two_device_cluster()
    add("single_op", ref.CompGraph([ref.OpNode(1, "conv", 1, {0: 2.0, 1: 5.0})], []), c, [{1: 0}, {1: 1}])
    g, c = rc.split_chain()
    add("split_chain", g, c, [{1: 0, 2: 1}, {1: 1, 2: 0}, {1: 0, 2: 0}])
    g, c = rc.two_op_chain()
    add("two_op_chain", g, c, [{1: 0, 2: 0}, {1: 0, 2: 1}])
    # costs present only on the devices the placement uses (simulator.py:85-96
    # checks the placed device alone); sparse-cost copies of random instances
    for trial in range(30):
        rng = random.Random(5000 + trial)
        g, c = rc.random_instance(rng, tight_ok=False)
        assign = {i: rng.choice(c.device_ids) for i in g.node_ids}
        nodes = []
        for n in g.nodes:
            keep = {assign[n.id]: n.compute_time[assign[n.id]]}
            for d in c.device_ids:
                if d != assign[n.id] and rng.random() < 0.4:
                    keep[d] = n.compute_time[d]
            nodes.append(ref.OpNode(n.id, n.op_type, n.mem_bytes, keep, n.members, n.type_seq, n.tag))
        gs = ref.CompGraph(nodes, list(g.edges))
        add(f"sparse-{5000 + trial}", gs, c, [assign])
    # validation errors, in the reference's order
    c = rc.two_device_cluster(mem=10)
    add("memory", ref.CompGraph([ref.OpNode(1, "conv", 11, {0: 1.0, 1: 1.0})], []), c, [{1: 0}])
    g2 = ref.CompGraph([ref.OpNode(1, "conv", 1, {0: 1.0}), ref.OpNode(2, "bn", 1, {0: 1.0, 1: 2.0})],
                       [ref.FlowEdge(1, 2, 1000)])
    add("missing_on_placed", g2, rc.two_device_cluster(), [{1: 1, 2: 0}, {1: 0, 2: 1}])
    add("unknown_device", g2, rc.two_device_cluster(), [{1: 0, 2: 7}])
    return cases


def main():
    jobs = {"schedules.json": make_schedules, "brute_force.json": make_brute, "gcof.json": make_gcof,
            "workload_evals.json": make_workload_evals, "synth.json": make_synth,
            "solve_exact.json": make_solve_exact, "aux.json": make_aux,
            "simulate.json": make_simulate}
    only = set(sys.argv[1:])
    for fname, fn in jobs.items():
        if only and fname not in only:
            continue
        data = fn()
        (HERE / fname).write_text(json.dumps(data, separators=(",", ":"), sort_keys=True))
        print(fname, len(data), "records", (HERE / fname).stat().st_size, "bytes")


if __name__ == "__main__":
    main()
