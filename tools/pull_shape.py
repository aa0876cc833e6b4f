"""Work shape of the first pull of an exact-cost DOBFS (RMAT-26): for every
vertex still unvisited when the pull runs, where in its row the first
frontier neighbour sits.  Tells how much of the pull is record hits, short
scans and full-row scans (the long-row stage's load).  Diagnostic only."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1504_04804_b200 as mg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
src = int(sys.argv[2]) if len(sys.argv) > 2 else 8582448
plan = mg.PartitionPlan.rmat_device(scale, 16, 1)
cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                      dobfs_exact_cost=True)
r = mg.dobfs(plan, mg.DobfsOptions(source=src), cfg)
first_pull = int(sys.argv[3]) if len(sys.argv) > 3 else 2  # superstep of the first pull
print("S", r.stats.supersteps, "direction log", list(r.direction_log))
off, col, _ = plan.download_graph().arrays()
lab = r.labels
deg = np.diff(off.astype(np.int64))
front = first_pull  # frontier of superstep t = label t
unv = np.nonzero((lab > front) & (deg > 0))[0]
print(f"first pull at superstep {first_pull}: frontier {(lab == front).sum()}, unvisited {len(unv)}, "
      f"frontier degree sum {int(deg[lab == front].sum())}, unvisited degree sum {int(deg[unv].sum())}")
isf = (lab == front)
fh = np.empty(len(unv), np.int64)
CH = 1 << 22
for a in range(0, len(unv), CH):
    vs = unv[a:a + CH]
    o, d = off[vs].astype(np.int64), deg[vs]
    idx = np.repeat(o - np.cumsum(np.r_[0, d[:-1]]), d) + np.arange(d.sum())
    h = isf[col[idx]]
    pos = np.arange(len(idx)) - np.repeat(np.cumsum(np.r_[0, d[:-1]]), d)
    big = np.where(h, pos, np.iinfo(np.int64).max)
    starts = np.cumsum(np.r_[0, d[:-1]])
    fh[a:a + CH] = np.minimum.reduceat(big, starts)
d = deg[unv]
hit = fh < d
print("hit in arc 0/1:", int((fh < 2).sum()), " rows deg<=2 no hit:", int(((d <= 2) & ~hit).sum()))
lng = (d > 2) & (fh >= 2)
print("long rows:", int(lng.sum()), " of which hit:", int((lng & hit).sum()))
sc = np.where(hit, fh + 1, d)[lng] - 2
print("long-stage arcs scanned:", int(sc.sum()), " arcs of long rows:", int(d[lng].sum()))
for lo, hi in ((3, 8), (9, 32), (33, 128), (129, 1024), (1025, 1 << 40)):
    m = lng & (d >= lo) & (d <= hi)
    print(f"  deg {lo}-{hi}: rows {int(m.sum())} hit {int((m & hit).sum())} "
          f"scanned {int((np.where(hit, fh + 1, d) - 2)[m].sum())}")
m = lng & hit
print("hit position (long rows) percentiles 50/90/99:", np.percentile(fh[m], [50, 90, 99]))
