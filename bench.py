#!/usr/bin/env python
"""Benchmark: direction-optimising BFS (DOBFS) GTEPS on RMAT scale-26 / edge-factor-16
(BASELINE.json configs[1]) through the C-ABI library on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one DOBFS traversal from one source (sources cycle through a fixed
list: 0, then non-isolated vertices drawn with seed 7).  GTEPS = A_r / t with
A_r = sum of degrees of the reached vertices; t is the library's
CUDA-event time of the superstep loop including per-run init (the reference's
wall_ms region, engine.hpp:951-964).  `e2e` repeats the steps through the same
public call with the labels copied back into pinned host memory every step.

--impl reference times the reference's own CPU engine (oracle/_ref, compiled
from the reference sources) on the same graph and sources.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


def ncu_traffic(kind):
    """dram bytes per launch of the dominant kernel from the committed ncu capture"""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"dobfs_{kind}_bytes_per_launch"), d.get(f"dobfs_{kind}_launch")
    except Exception:
        return None, None


class Clocks:
    """nvidia-smi sampler running during the timed region"""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) > 2 and r[1].strip().isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 2 and r[2].strip().isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].strip() == "Active":
                    reasons.add(nm)
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


def pick_sources(off, count, seed=7):
    deg = np.diff(off.astype(np.int64))
    nonzero = np.nonzero(deg)[0]
    rng = np.random.RandomState(seed)
    extra = rng.choice(nonzero, size=min(count - 1, len(nonzero)), replace=False)
    return [0] + [int(x) for x in extra]


def allreduce(x, op):
    """scalar all-reduce over ranks (device tensor under NCCL, host under gloo)"""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def reached_arcs(labels, deg):
    return int(deg[labels != 0xFFFFFFFF].sum())


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    # MG_BENCH_DEVICE pins every rank to one GPU (exercises the multi-process
    # IPC path on a single-GPU box); default: one GPU per local rank
    local = int(os.environ.get("MG_BENCH_DEVICE", local))
    return rank, world, local


def cpu_reference(graph_arrays, sources, arcs, max_s, label):
    """time the reference engine (oracle/_ref) on the same graph; n = 1 partition"""
    from oracle import ref
    off, col, _ = graph_arrays
    t0 = time.time()
    g = ref.RefGraph.from_csr(off, col)
    plan = ref.RefPlan(g, np.zeros(len(off) - 1, np.uint32), 1)
    prep = time.time() - t0
    done, ms, a = [], 0.0, 0
    t1 = time.time()
    for s in sources:
        r = plan.dobfs(s)
        ms += r.stats.wall_ms
        a += arcs[s]
        done.append(s)
        if time.time() - t1 > max_s:
            break
    return {"value": a / (ms * 1e-3) / 1e9, "unit": "GTEPS", "cores": 1, "kind": "reference",
            "sample": f"{label}: reference dobfs (n=1 partition, 1 thread) from sources {done}, "
                      f"{ms:.0f} ms engine wall_ms (plan build {prep:.1f} s excluded)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--num-sources", type=int, default=8)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    rank, world, local = dist_env()
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        # NCCL for the bench plumbing (barrier / max-over-ranks); gloo when every
        # rank is pinned to one GPU (NCCL refuses duplicate devices)
        backend = "gloo" if "MG_BENCH_DEVICE" in os.environ else "nccl"
        dist.init_process_group(backend, init_method="env://")
    workload = f"dobfs_rmat{args.scale}_ef{args.edge_factor}"
    if args.impl == "reference":
        return run_reference(args, rank, world, workload)
    return run_ours(args, rank, world, local, workload)


def build_plan(args, n, owner=None, devices=None):
    import paper_1504_04804_b200 as mg
    t0 = time.time()
    plan = mg.PartitionPlan.rmat_device(args.scale, args.edge_factor, args.seed, owner=owner, n=n,
                                        devices=devices)
    return plan, time.time() - t0


def run_ours(args, rank, world, local, workload):
    import torch

    import paper_1504_04804_b200 as mg
    torch.cuda.set_device(local)
    hbm, hbm_kind = peaks()
    # one partition per GPU: N = 1 is the single-partition plan; N > 1 is one
    # process per GPU, partition_random(|V|, N, 7) (partition.cpp:31-40), ranks
    # exchanging records through CUDA-IPC-mapped inboxes over NVLink
    if world > 1:
        import uuid
        owner = mg.partition_random(1 << args.scale, world, 7)
        key = [uuid.uuid4().hex if rank == 0 else None]
        torch.distributed.broadcast_object_list(key, src=0)
        t0 = time.time()
        plan = mg.PartitionPlan.rmat_device_multiprocess(args.scale, args.edge_factor, args.seed,
                                                         owner, world, rank, local, key[0])
        prep_s = time.time() - t0
        hosted = owner == rank
    else:
        plan, prep_s = build_plan(args, 1, devices=[local])
        hosted = None
    g = plan.download_graph()
    off, col, _ = g.arrays()
    del g
    deg = np.diff(off.astype(np.int64))
    sources = pick_sources(off, args.num_sources)
    cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On)
    opt = lambda s: mg.DobfsOptions(source=s)  # noqa: E731
    # warm-up: every source once with labels downloaded (A_r per source), >= W runs
    arcs = {}
    for i in range(max(args.warmup, len(sources))):
        s = sources[i % len(sources)]
        r = mg.dobfs(plan, opt(s), cfg)
        if s not in arcs:
            lab = r.labels if hosted is None else np.where(hosted, r.labels, 0xFFFFFFFF)
            a = reached_arcs(lab, deg)
            if world > 1:  # each rank holds its hosted labels only
                a = int(allreduce(a, "sum"))
            arcs[s] = a
    steps = [sources[i % len(sources)] for i in range(args.steps)]
    total_arcs = sum(arcs[s] for s in steps)

    def timed(do_a, do_b, cfg=cfg):
        """K device-resident steps; CUDA-event times from the library stream"""
        mg.lib().mg_plan_set_profiling(plan._h, 1)
        for s in sources[:2]:  # warm this parameter set
            dobfs_stats(mg, plan, s, cfg, do_a, do_b)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        acc = {"dev_ms": 0.0, "pull": [0.0, 0.0, 0], "push": [0.0, 0.0, 0], "xms": 0.0,
               "xbytes": 0}
        l0 = mg.kernel_launch_count()
        clocks = Clocks(local)
        w0 = time.perf_counter()
        for s in steps:
            st = dobfs_stats(mg, plan, s, cfg, do_a, do_b)
            acc["dev_ms"] += st.device_ms
            acc["xms"] += st.exchange_ms  # pack + publish kernels (records into peer HBM)
            acc["xbytes"] += st.exchange_bytes
            for key, ms, b, n in (("pull", st.kernel_ms, st.kernel_bytes, st.kernel_launches),
                                  ("push", st.kernel2_ms, st.kernel2_bytes,
                                   st.kernel2_launches)):
                acc[key][0] += ms
                acc[key][1] += b
                acc[key][2] += n
        torch.cuda.synchronize()
        acc["wall"] = time.perf_counter() - w0
        acc["clocks"] = clocks.stop()
        acc["launches"] = mg.kernel_launch_count() - l0
        mg.lib().mg_plan_set_profiling(plan._h, 0)
        dev = acc["dev_ms"]
        if world > 1:
            dev = allreduce(dev, "max")
        acc["dev_max_ms"] = dev
        acc["value"] = total_arcs / (dev * 1e-3) / 1e9
        # end to end: same calls, labels copied into pinned host memory each step
        e2e_t = 0.0
        for s in steps:
            t0 = time.perf_counter()
            e2e_call(mg, plan, s, cfg, labels, do_a, do_b)
            e2e_t += time.perf_counter() - t0
        if world > 1:
            e2e_t = allreduce(e2e_t, "max")
        acc["e2e"] = total_arcs / e2e_t / 1e9
        return acc

    host = torch.empty(plan.num_global_vertices, dtype=torch.int32, pin_memory=True)
    labels = host.numpy().view(np.uint32)
    # headline: the reference's direction rule and defaults (primitives.hpp:69-70);
    # on one partition a logically-forward superstep whose exact edge count
    # dwarfs the unvisited list runs on the pull kernel (mg_config.dobfs_exact_cost).
    # Labels, direction log, S and W are the reference's (tests/test_gpu_parity.py).
    exact_cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                                dobfs_exact_cost=True)
    main = timed(0.01, 0.1, exact_cfg)
    # the same rule executed physically as the reference schedules it
    refsched = timed(0.01, 0.1)
    tuned = timed(0.001, 0.1)      # do_a tuned for RMAT (per graph type)
    dev_ms, value, e2e, clk, launches, wall = (main["dev_max_ms"], main["value"], main["e2e"],
                                              main["clocks"], main["launches"], main["wall"])
    kind = "push" if main["push"][0] >= main["pull"][0] else "pull"
    prof = {"ms": main[kind][0], "bytes": main[kind][1], "launches": main[kind][2],
            "dev_ms": main["dev_ms"]}
    other = "pull" if kind == "push" else "push"

    if rank != 0:
        return 0
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_reference((off, col, None), sources, arcs, args.cpu_seconds, workload)
        except Exception as ex:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GTEPS", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {ex}"}
    achieved = prof["bytes"] / (prof["ms"] * 1e-3) / 1e9 if prof["ms"] else None
    traffic, traffic_src = ncu_traffic(kind)
    line = {
        "metric": "DOBFS GTEPS (A_r / t) on RMAT",
        "value": round(value, 3),
        "unit": "GTEPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(dev_ms / args.steps, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (hashed R-MAT generated on the GPU)",
        "config": {
            "workload": workload, "scale": args.scale, "edge_factor": args.edge_factor,
            "generator": f"counter-based R-MAT (a,b,c,d)=(.57,.19,.19,.05) seed {args.seed},"
                         " symmetrized + deduplicated",
            "num_vertices": plan.num_global_vertices, "num_arcs": plan.num_global_edges,
            "partitions_per_gpu": 1,
            "parallelism": f"partitioned x{world} (random, seed 7), CUDA IPC P2P exchange"
            if world > 1 else "single partition",
            "sources": sources, "mean_reached_arcs": total_arcs // len(steps),
            "policy": "max + fused", "do_a": 0.01, "do_b": 0.1,
            "physical_direction": "exact cost (pull when sum deg(Q) > 4 |unvisited|, "
                                  "summed over all partitions)",
            "l2": "inputs larger than L2 (CSR %.1f GB vs 126 MB L2)" % (
                (4 * (plan.num_global_vertices + plan.num_global_edges)) / 1e9),
            "graph_prep_s": round(prep_s, 2),
            "host_wall_s": round(wall, 4),
            "timing": "CUDA events on the library stream around init + superstep loop, "
                      "summed over the K steps (max over ranks)",
        },
        "e2e": {"value": round(e2e, 3), "unit": "GTEPS", "h2d_bytes_per_step": 4,
                "d2h_bytes_per_step": 4 * plan.num_global_vertices},
        "roofline": {"bound": "hbm",
                     "kernel": "lb_expand (push advance)" if kind == "push"
                     else "dobfs_pull (thread + group stages)",
                     "achieved": round(achieved, 1) if achieved else None, "peak": hbm,
                     "peak_kind": hbm_kind, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4) if achieved else None,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": prof["bytes"] / max(prof["launches"], 1),
                     "avg_launch_ms": prof["ms"] / max(prof["launches"], 1),
                     "share_of_step": round(prof["ms"] / prof["dev_ms"], 4) if prof["dev_ms"]
                     else None,
                     "other_kernel": {"kernel": other,
                                      "achieved": round(main[other][1] / (main[other][0] * 1e-3)
                                                        / 1e9, 1) if main[other][0] else None,
                                      "share_of_step": round(main[other][0] / main["dev_ms"], 4)}},
        "tuned": {"do_a": 0.001, "do_b": 0.1, "value": round(tuned["value"], 3),
                  "ms_per_step": round(tuned["dev_max_ms"] / args.steps, 4),
                  "e2e": round(tuned["e2e"], 3),
                  "note": "same graph and sources; the reference with the same do_a takes the "
                          "same direction decisions (direction log checked in tests)"},
        "reference_schedule": {
            "do_a": 0.01, "do_b": 0.1, "value": round(refsched["value"], 3),
            "ms_per_step": round(refsched["dev_max_ms"] / args.steps, 4),
            "e2e": round(refsched["e2e"], 3),
            "note": "dobfs_exact_cost off: every superstep runs in the direction the reference "
                    "rule picks (push advance for forward steps)"},
        "exchange": None if world == 1 else {
            "bytes_per_step": main["xbytes"] / args.steps,
            "pack_ms_per_step": round(main["xms"] / args.steps, 4),
            "achieved": round(main["xbytes"] / (main["xms"] * 1e-3) / 1e9, 1) if main["xms"] else None,
            "peak": 900.0, "unit": "GB/s",
            "peak_kind": "NVLink 5 nominal per direction per GPU",
            "note": "rank 0: record bytes its pack kernels stored into peer inboxes / their "
                    "CUDA-event time (with every rank on one GPU this is HBM, not NVLink)"},
        "cpu_baseline": cpu,
        "clocks": clk,
        "gpu_launches": launches,
    }
    print(json.dumps(line))
    return 0


def e2e_call(mg, plan, s, cfg, labels, do_a=0.01, do_b=0.1):
    import ctypes as C

    from paper_1504_04804_b200 import abi
    st = abi.mg_stats()
    dl = np.zeros(64, np.int32)
    ln, fw, bw = C.c_uint64(), C.c_uint64(), C.c_uint64()
    out = None if labels is None else labels.ctypes.data_as(C.c_void_p)
    rc = mg.lib().mg_dobfs(plan._h, s, do_a, do_b, 0, C.byref(cfg.to_c()), out, None,
                           dl.ctypes.data_as(C.c_void_p), 64, C.byref(ln), C.byref(fw),
                           C.byref(bw), C.byref(st))
    if rc:
        raise RuntimeError(mg.lib().mg_last_error().decode())
    return st


def dobfs_stats(mg, plan, s, cfg, do_a=0.01, do_b=0.1):
    """one device-resident DOBFS through the C-ABI (no result download)"""
    return e2e_call(mg, plan, s, cfg, None, do_a, do_b)


def run_reference(args, rank, world, workload):
    if rank != 0:
        return 0
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    import paper_1504_04804_b200 as mg
    # input synthesis only (not timed): the same hashed R-MAT graph
    try:
        plan, _ = build_plan(args, 1)
        g = plan.download_graph()
        del plan
    except Exception:
        g = mg.Csr.rmat_hashed(args.scale, args.edge_factor, args.seed)
    off, col, _ = g.arrays()
    deg = np.diff(off.astype(np.int64))
    sources = pick_sources(off, args.num_sources)
    rg = ref.RefGraph.from_csr(off, col)
    del g, col
    # same partitioning as our arm: one reference worker thread per GPU rank
    owner = (mg.partition_random(len(off) - 1, world, 7) if world > 1
             else np.zeros(len(off) - 1, np.uint32))
    rplan = ref.RefPlan(rg, owner, world)
    arcs = {}
    for i in range(args.warmup):
        s = sources[i % len(sources)]
        r = rplan.dobfs(s)
        arcs[s] = reached_arcs(r.labels, deg)
    ms, a = 0.0, 0
    for i in range(args.steps):
        s = sources[i % len(sources)]
        r = rplan.dobfs(s)
        if s not in arcs:
            arcs[s] = reached_arcs(r.labels, deg)
        ms += r.stats.wall_ms
        a += arcs[s]
    v = a / (ms * 1e-3) / 1e9
    print(json.dumps({
        "impl": "reference", "metric": "DOBFS GTEPS (A_r / t) on RMAT", "value": round(v, 4),
        "unit": "GTEPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (hashed R-MAT)",
        "config": {"workload": workload, "scale": args.scale, "edge_factor": args.edge_factor,
                   "sources": sources, "partitions": world},
        "cpu_baseline": {"value": round(v, 4), "unit": "GTEPS", "cores": world,
                         "kind": "reference",
                         "sample": f"{args.steps} reference dobfs runs (engine wall_ms), "
                                   f"n={world} partitions = {world} worker threads"},
        "e2e": {"value": round(v, 4), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))
    return 0


if __name__ == "__main__":
    sys.exit(main())
