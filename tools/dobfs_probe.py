"""Per-superstep probe of one DOBFS run (direction log, frontier sizes, W)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1504_04804_b200 as mg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
plan = mg.PartitionPlan.rmat_device(scale, 16, 1)
DO_A = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
EXACT = len(sys.argv) > 3 and sys.argv[3] == "exact"
SRC = int(sys.argv[4]) if len(sys.argv) > 4 else 0
cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                      dobfs_exact_cost=EXACT)
for rep in range(3):
    t0 = time.perf_counter()
    r = mg.dobfs(plan, mg.DobfsOptions(source=SRC, do_a=DO_A), cfg, download=False)
    t1 = time.perf_counter()
    st = r.stats
    print(f"rep {rep}: device {st.device_ms:.3f} ms wall {(t1-t0)*1e3:.3f} ms S={st.supersteps} "
          f"launches={st.gpu_launches}")
print("dir", list(r.direction_log))
print("out/iter", list(st.out_per_iter))
print("edges/iter", list(st.edges_per_iter))
