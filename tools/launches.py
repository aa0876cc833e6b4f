"""Summarise an ncu --csv launch list: per kernel name, count and total us."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((int(d["ID"]), d["Kernel Name"].split("(")[0][:70], float(d["Metric Value"])))
last = int(sys.argv[2]) if len(sys.argv) > 2 else len(out)
sel = out[-last:]
agg = collections.OrderedDict()
for _, k, t in sel:
    c, s = agg.get(k, (0, 0.0))
    agg[k] = (c + 1, s + t)
tot = sum(s for _, s in agg.values())
for k, (c, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{s/1e3:10.1f} us {100*s/tot:5.1f}%  x{c:4d}  {k}")
print(f"total {tot/1e3:.1f} us over {len(sel)} launches")
