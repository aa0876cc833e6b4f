"""Per-source DOBFS breakdown on the bench graph (direction log, W per superstep, time)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1504_04804_b200 as mg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
plan = mg.PartitionPlan.rmat_device(scale, 16, 1)
off, _, _ = plan.download_graph().arrays()
srcs = bench.pick_sources(off, 8)
cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On)
cfg2 = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On, dobfs_exact_cost=True)
for do_a, exact in ((0.01, False), (0.001, False), (0.01, True)):
    for s in srcs:
        mg.dobfs(plan, mg.DobfsOptions(source=s, do_a=do_a), cfg2 if exact else cfg, download=False)
        r = mg.dobfs(plan, mg.DobfsOptions(source=s, do_a=do_a), cfg2 if exact else cfg, download=False)
        st = r.stats
        print(f"do_a={do_a} exact={exact} src={s} deg={off[s+1]-off[s]} {st.device_ms:.3f} ms "
              f"dir={list(map(int, r.direction_log))} out={list(map(int, st.out_per_iter))} "
              f"W={list(map(int, st.edges_per_iter))}", flush=True)
