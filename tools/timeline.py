"""Kernel timeline of one primitive run (CUPTI via torch.profiler, real concurrent
timings, not ncu-serialised): start offset, duration and the idle gap before
every kernel the library launches.

    python tools/timeline.py dobfs 26 [source] [exact]
    python tools/timeline.py bfs 18
    python tools/timeline.py sssp|bc 24
    python tools/timeline.py pr|cc 24        (RGG 2^24)
"""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_1504_04804_b200 as mg  # noqa: E402

prim = sys.argv[1]
scale = int(sys.argv[2])
src = int(sys.argv[3]) if len(sys.argv) > 3 else 0
exact = "exact" in sys.argv
cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                      dobfs_exact_cost=exact)
if prim in ("pr", "cc"):
    plan = mg.PartitionPlan.rgg_device(1 << scale, 1)
elif prim == "bfs" and scale <= 20:
    plan = mg.PartitionPlan(mg.Csr.rmat(scale, 16, 1), None, 1)
else:
    plan = mg.PartitionPlan.rmat_device(scale, 16, 1,
                                        weights=(1, 64, 102) if prim == "sssp" else None)


def run():
    if prim == "dobfs":
        return mg.dobfs(plan, mg.DobfsOptions(source=src), cfg, download=False)
    if prim == "bfs":
        return mg.bfs(plan, mg.BfsOptions(source=src), cfg, download=False)
    if prim == "sssp":
        return mg.sssp(plan, src, False, cfg, download=False)
    if prim == "bc":
        return mg.bc(plan, src, cfg, download=False)
    if prim == "cc":
        return mg.cc(plan, cfg, download=False)
    return mg.pagerank(plan, mg.PrOptions(damping=0.85, epsilon=1e-6, max_iter=1000), cfg,
                       download=False)


for _ in range(3):
    r = run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    r = run()
    torch.cuda.synchronize()
print(f"device_ms {r.stats.device_ms:.3f} S={r.stats.supersteps}")
ev = sorted([e for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
if not ev:
    sys.exit(0)
t0 = ev[0].time_range.start
prev_end = t0
busy = 0.0
agg = {}
for e in ev:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    gap = s - prev_end
    name = e.name.replace("(anonymous namespace)::", "").split("(")[0][-48:]
    print(f"{(s - t0):9.1f} us  {d:8.1f} us  gap {gap:7.1f}  {name}")
    prev_end = max(prev_end, e.time_range.end)
    busy += d
    c, t = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, t + d)
span = prev_end - t0
print(f"span {span:.1f} us, kernel busy {busy:.1f} us ({100 * busy / span:.1f}%)")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:9.1f} us x{c:4d} {k}")
