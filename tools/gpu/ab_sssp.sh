# same-box A/B of C3 SSSP (RMAT-24 w 1..64) and C5 BC: default vs variants
cat > /tmp/sp.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, paper_1504_04804_b200 as mg
plan = mg.PartitionPlan.rmat_device(24, 16, 1, weights=(1, 64, 102))
cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On)
r = mg.sssp(plan, 0, False, cfg)
ts = [mg.sssp(plan, 0, False, cfg, download=False).stats.device_ms for _ in range(5)]
bc = [mg.bc(plan, 0, cfg, download=False).stats.device_ms for _ in range(4)]
print(f"sssp {min(ts):.3f} ms  bc {min(bc[1:]):.3f} ms  S={r.stats.supersteps} W={r.stats.edges_examined} sum={int(r.dists[r.dists < 2**63].sum())}")
PY
for i in 1 2; do
echo default; python /tmp/sp.py
for v in "$@"; do echo $v; MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_$v.so python /tmp/sp.py; done
done
