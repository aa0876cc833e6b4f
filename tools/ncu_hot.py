"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
data = []
for r in rows[2:]:
    if len(r) != len(h):
        continue
    try:
        s = float(r[ix["Warp Stall Sampling (All Samples)"]])
    except ValueError:
        continue
    stalls = {k: float(r[ix[k]]) for k in h if k.startswith("stall_") and "Not Issued" not in k
              and r[ix[k]] not in ("", "0")}
    top = sorted(stalls.items(), key=lambda x: -x[1])[:2]
    data.append((s, r[ix["Address"]][-5:], r[ix["Source"]].strip()[:60], top))
tot = sum(d[0] for d in data) or 1
for s, a, src, top in sorted(data, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100*s/tot:5.1f}% {a} {src:60s} {top}")
