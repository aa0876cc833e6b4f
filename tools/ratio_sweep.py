"""Total device time of exact-cost DOBFS over source 0 + 64 random sources on
RMAT-26 (one process per MG_PULL_RATIO value; the ratio is read once)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1504_04804_b200 as mg  # noqa: E402

plan = mg.PartitionPlan.rmat_device(26, 16, 1)
off, _, _ = plan.download_graph().arrays()
srcs = bench.pick_sources(off, 65)
cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                      dobfs_exact_cost=True)
per = []
for s in srcs:
    mg.dobfs(plan, mg.DobfsOptions(source=s), cfg, download=False)
    per.append(min(mg.dobfs(plan, mg.DobfsOptions(source=s), cfg, download=False).stats.device_ms
                   for _ in range(3)))
print("total ms", round(sum(per), 3), "first8", round(sum(per[:8]), 3), "max", round(max(per), 3))
