import sys, os
sys.path.insert(0, ".")
import paper_1504_04804_b200 as mg
plan = mg.PartitionPlan.rmat_device(26, 16, 1)
cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On, dobfs_exact_cost=True)
for i in range(3):
    r = mg.dobfs(plan, mg.DobfsOptions(source=0), cfg, download=False)

print("device_ms", r.stats.device_ms, file=sys.stderr)
