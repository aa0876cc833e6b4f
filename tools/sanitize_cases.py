"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck --target-processes all python tools/sanitize_cases.py
    compute-sanitizer --tool memcheck --target-processes all python tools/sanitize_cases.py --mp

Every primitive at n = 1, 2, 3 partitions on one GPU (rmat 12/16 and a grid),
the DOBFS pull kernels and the device-driven superstep loop (scale 16,
exact-cost), the dense exchange (bitmap / value arrays, scale 14 at n = 2),
each result checked against the oracle so a silent corruption also fails.
--mp runs the two-process CUDA-IPC fabric (every rank on GPU 0), including
the device-driven DOBFS superstep loop (one CUDA graph per rank)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1504_04804_b200 as mg  # noqa: E402
from oracle import seq  # noqa: E402


def check(cond, what):
    if not cond:
        raise SystemExit(f"FAIL: {what}")


def single_process():
    exact = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                            dobfs_exact_cost=True)
    for g in (mg.Csr.rmat(12, 16, 1), mg.Csr.grid(24, 24)):
        off, col, _ = g.arrays()
        want = seq.bfs_levels(off, col, 0)
        gw = g.with_weights(1, 64, 3)
        offw, colw, w = gw.arrays()
        for n in (1, 2, 3):
            owner = mg.partition_random(g.num_vertices, n, 7)
            plan = mg.PartitionPlan(g, owner, n)
            check(np.array_equal(mg.bfs(plan, mg.BfsOptions(source=0)).labels, want), "bfs")
            check(np.array_equal(mg.dobfs(plan, mg.DobfsOptions(source=0)).labels, want), "dobfs")
            check(np.array_equal(mg.dobfs(plan, mg.DobfsOptions(source=0, mark_preds=True),
                                          exact).labels, want), "dobfs exact")
            check(np.array_equal(mg.cc(plan).components, seq.connected_components(off, col)),
                  "cc")
            bc, sigma, _ = seq.brandes_bc(off, col, 0)
            r = mg.bc(plan, 0)
            check(np.array_equal(r.sigma, sigma), "bc sigma")
            r = mg.pagerank(plan, mg.PrOptions(epsilon=1e-6))
            ranks, it, _ = seq.pagerank_power(off, col, 0.85, 1e-6, 1000)
            check(r.iterations == it and np.max(np.abs(r.ranks - ranks)) <= 1e-6, "pagerank")
            pw = mg.PartitionPlan(gw, mg.partition_biased_random(gw, n, 7, 1.0), n)
            check(np.array_equal(mg.sssp(pw, 0).dists, seq.dijkstra(offw, colw, w, 0)), "sssp")
    # pull kernels + device-driven loop (one partition, exact cost)
    g = mg.Csr.rmat(16, 16, 1)
    off, col, _ = g.arrays()
    plan = mg.PartitionPlan(g, None, 1)
    for s in (0, 7):
        check(np.array_equal(mg.dobfs(plan, mg.DobfsOptions(source=s), exact).labels,
                             seq.bfs_levels(off, col, s)), "dobfs pull")
    # dense exchange: discoveries >= |V|/32 per worker (bitmap), CC deltas > |V|/2 (values)
    g = mg.Csr.rmat(14, 16, 2)
    off, col, _ = g.arrays()
    plan = mg.PartitionPlan(g, mg.partition_random(g.num_vertices, 2, 7), 2)
    check(np.array_equal(mg.dobfs(plan, mg.DobfsOptions(source=0)).labels,
                         seq.bfs_levels(off, col, 0)), "dobfs dense")
    check(np.array_equal(mg.cc(plan).components, seq.connected_components(off, col)), "cc dense")
    # DOBFS runs back to back (incremental label reset), an interleaved BC
    g = mg.Csr.rmat(13, 8, 4)
    off, col, _ = g.arrays()
    plan = mg.PartitionPlan(g, None, 1)
    for s in (0, 9, 0):
        check(np.array_equal(mg.dobfs(plan, mg.DobfsOptions(source=s), exact).labels,
                             seq.bfs_levels(off, col, s)), "dobfs reuse")
        mg.bc(plan, 1)
    print("sanitize cases ok")


def multi_process():
    import subprocess
    import tempfile
    import uuid
    key = uuid.uuid4().hex
    prog = f"""
import sys, numpy as np
sys.path.insert(0, {ROOT!r})
import paper_1504_04804_b200 as mg
from oracle import seq
rank = int(sys.argv[1])
g = mg.Csr.rmat(13, 16, 1)
off, col, _ = g.arrays()
owner = mg.partition_random(g.num_vertices, 2, 7)
plan = mg.PartitionPlan.multiprocess(g, owner, 2, rank, 0, {key!r})
hosted = owner == rank
want = seq.bfs_levels(off, col, 0)
mx = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                    dobfs_exact_cost=True)
cases = [lambda: mg.bfs(plan, mg.BfsOptions(source=0)).labels,
         lambda: mg.dobfs(plan, mg.DobfsOptions(source=0)).labels,
         lambda: mg.dobfs(plan, mg.DobfsOptions(source=0), mx).labels]  # device loop
import os
if os.environ.get("MG_SAN_ONLY_LOOP"):
    cases = cases[2:]
for f in cases:
    lab = f()
    assert np.array_equal(lab[hosted], want[hosted])
if not os.environ.get("MG_SAN_ONLY_LOOP"):
    comp = mg.cc(plan).components
    assert np.array_equal(comp[hosted], seq.connected_components(off, col)[hosted])
print("rank", rank, "ok")
"""
    with tempfile.NamedTemporaryFile("w", suffix=".py", delete=False) as f:
        f.write(prog)
    ps = [subprocess.Popen([sys.executable, f.name, str(r)]) for r in range(2)]
    rc = [p.wait(timeout=1800) for p in ps]
    os.unlink(f.name)
    check(rc == [0, 0], f"multi-process ranks exited {rc}")
    print("sanitize multi-process ok")


if __name__ == "__main__":
    if "--mp-loop" in sys.argv:  # only the device-driven DOBFS loop, two processes
        os.environ["MG_SAN_ONLY_LOOP"] = "1"
        multi_process()
    elif "--mp" in sys.argv:
        multi_process()
    else:
        single_process()
