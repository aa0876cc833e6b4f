"""Device time of the bench workload (exact-cost DOBFS, RMAT-26, the 8 bench
sources) with the device-driven graph loop and, with MG_NO_GRAPH=1, the
host-driven loop.  No profiler attached.

    python tools/graph_probe.py [scale] [graph|host|ref]

ref: the reference schedule (dobfs_exact_cost off: every forward superstep
pushes, host-driven loop)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1504_04804_b200 as mg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
plan = mg.PartitionPlan.rmat_device(scale, 16, 1)
off, _, _ = plan.download_graph().arrays()
srcs = bench.pick_sources(off, 8)
cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                      dobfs_exact_cost=True)
modes = [sys.argv[2]] if len(sys.argv) > 2 else ["graph", "host"]
for mode in modes:
    if mode == "host":
        os.environ["MG_NO_GRAPH"] = "1"
    if mode == "ref":
        cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                              dobfs_exact_cost=False)
    for s in srcs:
        mg.dobfs(plan, mg.DobfsOptions(source=s), cfg, download=False)
    per = []
    for s in srcs:
        ts = [mg.dobfs(plan, mg.DobfsOptions(source=s), cfg, download=False).stats.device_ms
              for _ in range(5)]
        per.append(min(ts))
    print(mode, "total ms", round(sum(per), 3), [round(x, 3) for x in per])
