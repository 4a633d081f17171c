"""Aggregate an ncu source page (cuda,sass CSV) per CUDA line and per region of
tpp_eval; usage: python scripts/ncu_regions.py export.csv [function-marker]"""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
cur = None; agg = defaultdict(lambda: [0, 0]); src = {}; hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        k = (cur, int(r[0]))
        if r[1]: src[k] = r[1]
        agg[k][0] += int(r[hdr.index('Instructions Executed')] or 0)
        agg[k][1] += int(r[hdr.index('Warp Stall Sampling (All Samples)')] or 0)
tot = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
print('instructions', tot, 'stall samples', ts)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{k[0][:12]:12s}:{k[1]:5d} {v[0]/tot*100:5.1f}% inst {v[1]/ts*100:5.1f}% stall | {src.get(k,'')[:100]}")
