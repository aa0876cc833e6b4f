"""C1 device time (BFS RMAT-18/16 seed 1, exact-cost graph loop and push schedule), min/mean of 30 runs."""
import sys

sys.path.insert(0, ".")
import paper_1504_04804_b200 as mg  # noqa: E402

plan = mg.PartitionPlan(mg.Csr.rmat(18, 16, 1), None, 1)
for name, cfg in [("exact", mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                                             dobfs_exact_cost=True)),
                  ("push", mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On))]:
    for _ in range(5):
        mg.bfs(plan, mg.BfsOptions(source=0), cfg, download=False)
    ts = [mg.bfs(plan, mg.BfsOptions(source=0), cfg, download=False).stats.device_ms for _ in range(30)]
    print(name, "min %.4f mean %.4f" % (min(ts), sum(ts) / len(ts)))
