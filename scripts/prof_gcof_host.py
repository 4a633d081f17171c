"""cProfile of one gcof call on a 100k-op synthetic graph (host vs kernel split)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_04025_b200 as mp  # noqa: E402
from paper_2312_04025_b200 import workloads  # noqa: E402

g = mp.gen_synthetic(mp.GenSpec(ops=100_000, width=32, density=0.5, devices=(0, 1, 2, 3)), 0)
rules = workloads.table_rules()
mp.gcof(g, rules)
cProfile.run("mp.gcof(g, rules)", "/tmp/gcof.prof")
pstats.Stats("/tmp/gcof.prof").sort_stats("tottime").print_stats(15)
