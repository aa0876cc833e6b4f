"""Run the bench's DOBFS workload (exact-cost, the 8 bench sources) once, for an
ncu metrics pass over the pull kernels:

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k regex:dobfs_pull --csv --log-file gpurun_out/pull_traffic.csv \
      python tools/pull_traffic.py
  python tools/pull_traffic.py --summarise gpurun_out/pull_traffic.csv

The summary gives dram bytes per pull STEP (thread + group kernel of one
superstep), the unit the bench's roofline `achieved` is averaged over.
"""
import csv
import json
import sys

sys.path.insert(0, ".")

if len(sys.argv) > 2 and sys.argv[1] == "--summarise":
    rows = list(csv.reader(open(sys.argv[2])))
    hdr, recs = None, {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = int(d["ID"])
            recs.setdefault(k, {"name": d["Kernel Name"].split("(")[0]})
            v = float(d["Metric Value"].replace(",", ""))
            unit = d.get("Metric Unit", "")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1,
                     "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
            recs[k][d["Metric Name"]] = v * scale
    steps, cur = [], None
    for k in sorted(recs):
        r = recs[k]
        b = r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)
        if "thread" in r["name"]:
            cur = {"bytes": b, "ns": r.get("gpu__time_duration.sum", 0),
                   "thread_bytes": b, "thread_ns": r.get("gpu__time_duration.sum", 0)}
            steps.append(cur)
        elif cur is not None:
            cur["bytes"] += b
            cur["ns"] += r.get("gpu__time_duration.sum", 0)
    tot = sum(s["bytes"] for s in steps)
    print(json.dumps({"pull_steps": len(steps), "dram_bytes_total": tot,
                      "dram_bytes_per_step": tot / max(len(steps), 1),
                      "largest_step_bytes": max(s["bytes"] for s in steps),
                      "ncu_ns_total": sum(s["ns"] for s in steps),
                      "steps": [[int(s["bytes"]), int(s["ns"]), int(s["thread_bytes"]),
                                 int(s["thread_ns"])] for s in steps]}))
    sys.exit(0)

import bench  # noqa: E402
import paper_1504_04804_b200 as mg  # noqa: E402

plan = mg.PartitionPlan.rmat_device(26, 16, 1)
off, _, _ = plan.download_graph().arrays()
cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                      dobfs_exact_cost=True)
for s in bench.pick_sources(off, 8):
    mg.dobfs(plan, mg.DobfsOptions(source=s), cfg, download=False)
