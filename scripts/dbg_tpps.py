import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import paper_2312_04025_b200 as mp
from conftest import golden, graph_from, cluster_from
for case in golden("brute_force.json")[:10]:
    g = graph_from(case["graph"]); c = cluster_from(case["cluster"])
    with mp.Instance(g, c, mp.effective_bandwidth(c)) as inst:
        print(case["name"], inst.info(), flush=True)
        rows = np.random.default_rng(0).integers(0, inst.K, (64, inst.n_ops), dtype=np.uint8)
        print(" eval", mp.evaluate_batch(inst, rows)[:4], flush=True)
        print(" ls", mp.local_search(inst, rows[:4], chains=64, moves=4, seed=1)[1], flush=True)
