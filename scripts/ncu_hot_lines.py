"""Summarise an ncu source page export: top CUDA source lines by warp-stall samples.

    ncu -i rep.ncu-rep --page source --csv --print-source=cuda,sass > src.csv
    python scripts/ncu_hot_lines.py src.csv [N]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr_i]
si = h.index("Warp Stall Sampling (All Samples)")
agg = defaultdict(float)
src = {}
cur = None
for r in rows[hdr_i + 1:]:
    if not r:
        continue
    if r[0]:
        cur = r[0]
        src[cur] = r[1]
    try:
        agg[cur] += float(r[si] or 0)
    except (ValueError, IndexError):
        pass
tot = sum(agg.values()) or 1
for line, s in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{100 * s / tot:5.1f}%  L{line}: {src.get(line, '')[:110]}")
