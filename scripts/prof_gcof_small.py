"""cProfile of repeated gcof calls on C2 (host vs native split for small graphs)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_04025_b200 as mp  # noqa: E402
from paper_2312_04025_b200 import workloads  # noqa: E402

w = workloads.c2(4)
mp.gcof(w.raw, w.rules)
cProfile.run("for _ in range(200): mp.gcof(w.raw, w.rules)", "/tmp/gcof_small.prof")
pstats.Stats("/tmp/gcof_small.prof").sort_stats("tottime").print_stats(14)
