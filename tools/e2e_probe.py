"""Time the end-to-end C-ABI DOBFS call (labels into pinned host memory) for
the label-download split fraction given by MG_D2H_SPLIT."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1504_04804_b200 as mg  # noqa: E402

plan = mg.PartitionPlan.rmat_device(26, 16, 1)
cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                      dobfs_exact_cost=True)
host = torch.empty(plan.num_global_vertices, dtype=torch.int32, pin_memory=True)
labels = host.numpy().view(np.uint32)
for _ in range(3):
    bench.e2e_call(mg, plan, 0, cfg, labels)
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    st = bench.e2e_call(mg, plan, 0, cfg, labels)
    ts.append((time.perf_counter() - t0) * 1e3)
print(f"call ms: median {np.median(ts):.3f} min {min(ts):.3f}  device {st.device_ms:.3f}")
