"""Per-launch table (time, dram read/write, instructions) from an ncu --metrics
--csv log: `python tools/ncu_launches.py log.csv [first_n]`."""
import csv
import sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
by, order = {}, []
for r in rows:
    key = (r["ID"], r["Kernel Name"][:44])
    if key not in by:
        by[key] = {}
        order.append(key)
    by[key][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
for key in order[:n or len(order)]:
    d = by[key]
    print(f"{key[1]:46s} t={d.get('gpu__time_duration.sum', 0) / 1e3:8.1f}us "
          f"rd={d.get('dram__bytes_read.sum', 0) / 1e6:8.1f}MB wr={d.get('dram__bytes_write.sum', 0) / 1e6:7.1f}MB "
          f"inst={d.get('smsp__inst_executed.sum', 0):.3g}")
