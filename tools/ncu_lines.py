"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line:
prints the top lines by warp-stall samples and executed instructions."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
agg = defaultdict(lambda: [0.0, 0.0, ""])
cur = None
files = {}
for r in rows[hdr + 1:]:
    if len(r) <= si:
        continue
    if r[0] not in ("", "-") and r[0].isdigit() and r[2] == "-":  # a CUDA source line header
        cur = int(r[0])
        agg[cur][2] = r[1]
        continue
    try:
        s, n = float(r[si]), float(r[ie])
    except ValueError:
        continue
    if cur is not None:
        agg[cur][0] += s
        agg[cur][1] += n
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot_s:.0f}, instructions {tot_i:.3e}")
for ln, (s, n, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / tot_s:5.1f}% stall {100 * n / tot_i:5.1f}% inst  L{ln}: {src.strip()[:100]}")
