"""Measure every BASELINE.json config on one B200 (device-timed, CUDA events on
the library stream) beside the reference CPU engine on the same graph.

    python tools/bench_configs.py [--configs 1,2,3,4,5] [--cpu-seconds 30]

GTEPS conventions: BFS/DOBFS/SSSP/BC: A_r / t; PR: |A| x
iterations / t; CC: |A| / t.  Prints one JSON line per (config, primitive).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1504_04804_b200 as mg  # noqa: E402

MAXCFG = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On)


def reached(labels_or_dists, deg, inf):
    return int(deg[labels_or_dists != inf].sum())


def timeit(fn, reps):
    fn()  # warm
    ms = []
    for _ in range(reps):
        ms.append(fn())
    return float(np.mean(ms)), float(np.min(ms))


def cpu(fn, budget):
    """run fn (returns wall_ms of the reference engine) until the budget is spent"""
    t0, out = time.time(), []
    while not out or (time.time() - t0 < budget and len(out) < 3):
        out.append(fn())
    return float(np.min(out)), len(out)


def emit(**kw):
    print(json.dumps(kw), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=30.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--scale24", type=int, default=24)
    ap.add_argument("--rgg-log2", type=int, default=24)
    a = ap.parse_args()
    cfgs = {int(x) for x in a.configs.split(",")}
    from oracle import ref

    if 1 in cfgs:  # BFS, RMAT-18/16 seed 1 (the reference's own generator), source 0
        g = mg.Csr.rmat(18, 16, 1)
        off, col, _ = g.arrays()
        deg = np.diff(off.astype(np.int64))
        plan = mg.PartitionPlan(g, None, 1)
        exact = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                                dobfs_exact_cost=True)
        # the exact-cost BFS (same labels) runs as one device-driven graph here
        r = mg.bfs(plan, mg.BfsOptions(source=0), exact)
        ar = reached(r.labels, deg, mg.kInfLabel)
        mean, best = timeit(lambda: mg.bfs(plan, mg.BfsOptions(source=0), exact,
                                          download=False).stats.device_ms, a.reps)
        emit(config=1, primitive="bfs_exact_cost", graph="rmat18_ef16_seed1", reached_arcs=ar,
             device_ms_mean=mean, device_ms_min=best, gteps=ar / (mean * 1e-3) / 1e9,
             supersteps=int(r.stats.supersteps))
        r = mg.bfs(plan, mg.BfsOptions(source=0), MAXCFG)
        ar = reached(r.labels, deg, mg.kInfLabel)
        mean, best = timeit(lambda: mg.bfs(plan, mg.BfsOptions(source=0), MAXCFG,
                                          download=False).stats.device_ms, a.reps)
        out = dict(config=1, primitive="bfs", graph="rmat18_ef16_seed1", reached_arcs=ar,
                   device_ms_mean=mean, device_ms_min=best, gteps=ar / (mean * 1e-3) / 1e9,
                   supersteps=int(r.stats.supersteps))
        if not a.no_cpu:
            rp = ref.RefPlan(ref.RefGraph.from_csr(off, col), np.zeros(len(off) - 1, np.uint32), 1)
            ms, k = cpu(lambda: rp.bfs(0).stats.wall_ms, a.cpu_seconds)
            out.update(cpu_ms=ms, cpu_gteps=ar / (ms * 1e-3) / 1e9, cpu_cores=1, cpu_runs=k)
        emit(**out)

    if 2 in cfgs:  # BFS on the C2 graph (RMAT-26/16): the reference's push schedule, and
        # the exact-cost extension (heavy supersteps as pulls, same labels/S/W)
        plan = mg.PartitionPlan.rmat_device(26, 16, 1)
        off, _, _ = plan.download_graph().arrays()
        deg = np.diff(off.astype(np.int64))
        exact = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                                dobfs_exact_cost=True)
        for name, cfg in (("bfs", MAXCFG), ("bfs_exact_cost", exact)):
            r = mg.bfs(plan, mg.BfsOptions(source=0), cfg)
            ar = reached(r.labels, deg, mg.kInfLabel)
            mean, best = timeit(lambda: mg.bfs(plan, mg.BfsOptions(source=0), cfg,
                                              download=False).stats.device_ms, a.reps)
            emit(config=2, primitive=name, graph="rmat26_ef16", reached_arcs=ar,
                 device_ms_mean=mean, device_ms_min=best, gteps=ar / (mean * 1e-3) / 1e9,
                 supersteps=int(r.stats.supersteps), edges_examined=int(r.stats.edges_examined))
        # DOBFS over source 0 + 64 random non-isolated sources:
        # per-source GTEPS and their harmonic mean, exact-cost and reference schedule
        import bench
        srcs = bench.pick_sources(off, 65)
        for name, cfg in (("dobfs_exact_cost", exact), ("dobfs", MAXCFG)):
            per = []
            for s in srcs:
                r = mg.dobfs(plan, mg.DobfsOptions(source=s), cfg)
                ar = reached(r.labels, deg, mg.kInfLabel)
                mean, _ = timeit(lambda: mg.dobfs(plan, mg.DobfsOptions(source=s), cfg,
                                                 download=False).stats.device_ms, 3)
                per.append((s, ar, mean))
            g = [ar / (ms * 1e-3) / 1e9 for _, ar, ms in per]
            emit(config=2, primitive=name + "_65_sources", graph="rmat26_ef16",
                 sources="0 + 64 random non-isolated (bench.pick_sources seed 7)",
                 hmean_gteps=len(g) / sum(1.0 / x for x in g), min_gteps=min(g), max_gteps=max(g),
                 per_source=[[s, ar, round(ms, 4), round(x, 1)] for (s, ar, ms), x in zip(per, g)])
        del plan, off, deg

    if cfgs & {3, 5}:  # RMAT-24/16 (device hashed generator), weights U[1,64] seed+101
        plan = mg.PartitionPlan.rmat_device(a.scale24, 16, 1, weights=(1, 64, 102))
        g = plan.download_graph()
        off, col, w = g.arrays()
        deg = np.diff(off.astype(np.int64))
        if 3 in cfgs:
            r = mg.sssp(plan, 0, cfg=MAXCFG)
            ar = reached(r.dists, deg, mg.kInfDist)
            mean, best = timeit(lambda: mg.sssp(plan, 0, cfg=MAXCFG,
                                               download=False).stats.device_ms, a.reps)
            out = dict(config=3, primitive="sssp", graph=f"rmat{a.scale24}_ef16_w1-64",
                       reached_arcs=ar, device_ms_mean=mean, device_ms_min=best,
                       gteps=ar / (mean * 1e-3) / 1e9, supersteps=int(r.stats.supersteps),
                       edges_examined=int(r.stats.edges_examined))
            if not a.no_cpu:
                rp = ref.RefPlan(ref.RefGraph.from_csr(off, col, w),
                                 np.zeros(len(off) - 1, np.uint32), 1)
                ms, k = cpu(lambda: rp.sssp(0).stats.wall_ms, a.cpu_seconds)
                out.update(cpu_ms=ms, cpu_gteps=ar / (ms * 1e-3) / 1e9, cpu_cores=1, cpu_runs=k)
                del rp
            emit(**out)
        if 5 in cfgs:
            r = mg.bc(plan, 0, cfg=MAXCFG)
            ar = reached(r.labels, deg, mg.kInfLabel)
            mean, best = timeit(lambda: mg.bc(plan, 0, cfg=MAXCFG,
                                             download=False).stats.device_ms, a.reps)
            out = dict(config=5, primitive="bc", graph=f"rmat{a.scale24}_ef16", reached_arcs=ar,
                       device_ms_mean=mean, device_ms_min=best, gteps=ar / (mean * 1e-3) / 1e9,
                       supersteps=int(r.stats.supersteps))
            if not a.no_cpu:
                rp = ref.RefPlan(ref.RefGraph.from_csr(off, col),
                                 np.zeros(len(off) - 1, np.uint32), 1)
                ms, k = cpu(lambda: rp.bc(0).stats.wall_ms, a.cpu_seconds)
                out.update(cpu_ms=ms, cpu_gteps=ar / (ms * 1e-3) / 1e9, cpu_cores=1, cpu_runs=k)
                del rp
            emit(**out)
        del plan

    if 4 in cfgs:  # PR (0.85, 1e-6) and CC on RGG n = 2^24
        n = 1 << a.rgg_log2
        t0 = time.time()
        plan = mg.PartitionPlan.rgg_device(n, 1)
        prep = time.time() - t0
        g = plan.download_graph()
        off, col, _ = g.arrays()
        ne = int(len(col))
        r = mg.pagerank(plan, mg.PrOptions(epsilon=1e-6), MAXCFG)
        iters = int(r.iterations)
        mean, best = timeit(lambda: mg.pagerank(plan, mg.PrOptions(epsilon=1e-6), MAXCFG,
                                               download=False).stats.device_ms, a.reps)
        out = dict(config=4, primitive="pagerank", graph=f"rgg_2^{a.rgg_log2}", arcs=ne,
                   iterations=iters, device_ms_mean=mean, device_ms_min=best,
                   gteps=ne * iters / (mean * 1e-3) / 1e9, graph_prep_s=prep,
                   avg_degree=ne / n)
        if not a.no_cpu:
            rp = ref.RefPlan(ref.RefGraph.from_csr(off, col), np.zeros(n, np.uint32), 1)
            # bounded sample: 3 PageRank iterations of the reference engine
            rr = rp.pagerank(0.85, 1e-6, 3)
            ms = rr.stats.wall_ms
            out.update(cpu_ms_per_iter=ms / 3, cpu_gteps=ne * 3 / (ms * 1e-3) / 1e9, cpu_cores=1,
                       cpu_sample="3 reference PR iterations (max_iter=3)")
        emit(**out)
        r = mg.cc(plan, MAXCFG)
        mean, best = timeit(lambda: mg.cc(plan, MAXCFG, download=False).stats.device_ms, a.reps)
        out = dict(config=4, primitive="cc", graph=f"rgg_2^{a.rgg_log2}", arcs=ne,
                   device_ms_mean=mean, device_ms_min=best, gteps=ne / (mean * 1e-3) / 1e9,
                   supersteps=int(r.stats.supersteps),
                   components=int(len(np.unique(r.components))))
        if not a.no_cpu:
            ms, k = cpu(lambda: rp.cc().stats.wall_ms, a.cpu_seconds)
            out.update(cpu_ms=ms, cpu_gteps=ne / (ms * 1e-3) / 1e9, cpu_cores=1, cpu_runs=k)
        emit(**out)


if __name__ == "__main__":
    main()
