"""Per-CUDA-source-line totals (instructions executed, stall samples) from
`ncu -i rep --page source --csv --print-source cuda,sass`: which source lines
issue the instructions and which ones the warps wait on."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
f = None
acc = defaultdict(lambda: [0.0, 0.0, ""])
hdr = None
cur = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if not hdr or len(r) < 8:
        continue
    if r[0]:
        cur = (f, r[0])
        acc[cur][2] = r[1].strip()[:70]
        continue
    try:
        ins = float(r[hdr["Instructions Executed"]] or 0)
        st = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, KeyError):
        continue
    if cur:
        acc[cur][0] += ins
        acc[cur][1] += st
ti = sum(v[0] for v in acc.values()) or 1
ts = sum(v[1] for v in acc.values()) or 1
print(f"total instructions {ti:.3g}, stall samples {ts:.0f}")
for k, v in sorted(acc.items(), key=lambda x: -(x[1][0] / ti + x[1][1] / ts))[:top]:
    print(f"{k[0]:>12s}:{k[1]:<5s} inst {100 * v[0] / ti:5.1f}%  stall {100 * v[1] / ts:5.1f}%  {v[2]}")
