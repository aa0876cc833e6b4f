"""W per superstep of one DOBFS case under several configs vs the reference engine."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1504_04804_b200 as mg  # noqa: E402
from oracle import ref  # noqa: E402

g = mg.Csr.rmat(12, 32, 6)
off, col, _ = g.arrays()
src, do_a = 301, 0.001
rr = ref.RefPlan(ref.RefGraph.from_csr(off, col), np.zeros(len(off) - 1, np.uint32), 1).dobfs(
    src, do_a, 0.1)
print("ref", list(rr.direction_log), list(rr.edges_per_iter), list(rr.out_per_iter))
plan = mg.PartitionPlan(g, None, 1)
for name, cfg in [("default", mg.EngineConfig()),
                  ("max-fused", mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum,
                                                fused=mg.FusedMode.On)),
                  ("just-fused", mg.EngineConfig(fused=mg.FusedMode.On)),
                  ("max-unfused", mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum,
                                                  fused=mg.FusedMode.Off))]:
    r = mg.dobfs(plan, mg.DobfsOptions(source=src, do_a=do_a), cfg)
    print(name, list(r.direction_log), list(r.stats.edges_per_iter), list(r.stats.out_per_iter))
