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

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
with N ranks (one process per GPU, partition_random(|V|, N, 7)); with
MG_BENCH_DEVICE=0 every rank shares GPU 0 (the path, not its speed).

--impl reference times the reference's own CPU engine (oracle/_ref, compiled
from the reference sources) on the same graph and sources.  That process never
loads the product library: its graph comes from the oracle's own generator
(oracle/gen_oracle.cpp), bit-identical to the device generator
(tests/test_oracle.py, tests/test_gpu_parity.py).
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
NVLINK_GBS = 900.0  # NVLink 5, per direction per GPU (nominal)
METRIC = "DOBFS GTEPS (A_r / t) on RMAT"


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


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


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


def reached_arcs(labels, deg):
    return int(deg[labels != 0xFFFFFFFF].sum())


def workload_config(args, n, sources, nv, ne):
    """the config dict both arms print (identical for the same arguments)"""
    return {
        "workload": f"dobfs_rmat{args.scale}_ef{args.edge_factor}",
        "scale": args.scale, "edge_factor": args.edge_factor, "seed": args.seed,
        "generator": f"counter-based R-MAT (a,b,c,d)=(.57,.19,.19,.05) seed {args.seed},"
                     " symmetrized + deduplicated",
        "num_vertices": int(nv), "num_arcs": int(ne),
        "partitions": n,
        "partitioner": "partition_random(|V|, N, 7)" if n > 1 else "single partition",
        "sources": sources, "do_a": 0.01, "do_b": 0.1,
        "l2": "inputs larger than L2 (CSR %.1f GB vs 126 MB L2)" % (4 * (nv + ne) / 1e9),
    }


def allreduce(x, op):
    """scalar all-reduce over ranks (device tensor under NCCL, host under gloo)"""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    # MG_BENCH_DEVICE pins every rank to one GPU (exercises the multi-process
    # IPC path on a single-GPU box); default: one GPU per local rank
    local = int(os.environ.get("MG_BENCH_DEVICE", local))
    return rank, world, local


def spawn(argv, n):
    """--gpus N without a launcher: run this script under torch.distributed.run"""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)]
    return subprocess.call(cmd + argv)


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

    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(sys.argv[1:], args.gpus)
    rank, world, local = dist_env()
    if args.impl == "reference":
        # CPU reference: rank 0 alone runs and prints; other ranks exit at once
        return run_reference(args, rank, max(world, args.gpus)) if rank == 0 else 0
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        # NCCL for the bench plumbing (barrier / max-over-ranks); gloo when every
        # rank is pinned to one GPU (NCCL refuses duplicate devices)
        backend = "gloo" if "MG_BENCH_DEVICE" in os.environ else "nccl"
        dist.init_process_group(backend, init_method="env://")
    return run_ours(args, rank, world, local)


# ------------------------------------------------------------------------------ our arm
def e2e_call(mg, plan, s, cfg, labels, do_a=0.01, do_b=0.1):
    """one DOBFS through the C-ABI (mg_dobfs); labels=None keeps them on the device"""
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


def d2h_bytes(mg, plan):
    import ctypes as C
    b = C.c_uint64()
    mg.lib().mg_plan_last_d2h_bytes(plan._h, C.byref(b))
    return b.value


def run_ours(args, rank, world, local):
    import torch

    import paper_1504_04804_b200 as mg
    torch.cuda.set_device(local)
    hbm, hbm_kind = peaks()
    # one partition per GPU: N = 1 is the single-partition plan; N > 1 is one
    # process per GPU, partition_random(|V|, N, 7) (partition.cpp:31-40), ranks
    # exchanging through CUDA-IPC-mapped inboxes over NVLink
    t0 = time.time()
    if world > 1:
        import uuid
        owner = mg.partition_random(1 << args.scale, world, 7)
        key = [uuid.uuid4().hex if rank == 0 else None]
        torch.distributed.broadcast_object_list(key, src=0)
        plan = mg.PartitionPlan.rmat_device_multiprocess(args.scale, args.edge_factor, args.seed,
                                                         owner, world, rank, local, key[0])
        hosted = owner == rank
    else:
        plan = mg.PartitionPlan.rmat_device(args.scale, args.edge_factor, args.seed,
                                            devices=[local])
        hosted = None
    torch.cuda.synchronize()
    prep_s = time.time() - t0
    g = plan.download_graph()
    off, col, _ = g.arrays()
    del g
    deg = np.diff(off.astype(np.int64))
    sources = pick_sources(off, args.num_sources)
    base = dict(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On)
    exact_cfg = mg.EngineConfig(dobfs_exact_cost=True, **base)
    ref_cfg = mg.EngineConfig(**base)
    # plan-lifetime precomputation (non-isolated list + its host sort, pull
    # records, CUDA-graph capture): paid by the first call on a plan, outside
    # `value`; measured here as first call minus a warm call of the same source
    t1 = time.perf_counter()
    e2e_call(mg, plan, sources[0], exact_cfg, None)
    first = time.perf_counter() - t1
    t1 = time.perf_counter()
    e2e_call(mg, plan, sources[0], exact_cfg, None)
    precompute_s = max(first - (time.perf_counter() - t1), 0.0)
    # warm-up: every source once with labels downloaded (A_r per source), >= W runs
    arcs = {}
    for i in range(max(args.warmup, len(sources))):
        s = sources[i % len(sources)]
        r = mg.dobfs(plan, mg.DobfsOptions(source=s), exact_cfg)
        if s not in arcs:
            lab = r.labels if hosted is None else np.where(hosted, r.labels, 0xFFFFFFFF)
            a = reached_arcs(lab, deg)
            if world > 1:  # each rank holds its hosted labels only
                a = int(allreduce(a, "sum"))
            arcs[s] = a
    steps = [sources[i % len(sources)] for i in range(args.steps)]
    total_arcs = sum(arcs[s] for s in steps)
    host = torch.empty(plan.num_global_vertices, dtype=torch.int32, pin_memory=True)
    labels = host.numpy().view(np.uint32)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def timed(do_a, do_b, cfg):
        """K device-resident steps, profiling off: the library's CUDA-event time of
        every run (init + superstep loop), summed; then the same K steps through the
        public call with the labels downloaded (e2e)"""
        for s in sources[:2]:  # warm this parameter set
            e2e_call(mg, plan, s, cfg, None, do_a, do_b)
        barrier()
        acc = {"dev_ms": 0.0, "xms": 0.0, "xbytes": 0, "device_loop": 0}
        l0 = mg.kernel_launch_count()
        clocks = Clocks(local)
        w0 = time.perf_counter()
        for s in steps:
            st = e2e_call(mg, plan, s, cfg, None, do_a, do_b)
            acc["dev_ms"] += st.device_ms
            acc["xms"] += st.exchange_ms  # pack + publish kernels (records into peer HBM)
            acc["xbytes"] += st.exchange_bytes
            acc["device_loop"] += st.device_loop
        barrier()
        acc["wall"] = time.perf_counter() - w0
        acc["clocks"] = clocks.stop()
        acc["launches"] = mg.kernel_launch_count() - l0
        acc["dev_max_ms"] = allreduce(acc["dev_ms"], "max") if world > 1 else acc["dev_ms"]
        acc["value"] = total_arcs / (acc["dev_max_ms"] * 1e-3) / 1e9
        # end to end: same calls, labels copied into pinned host memory each step
        barrier()
        e2e_t, d2h = 0.0, 0
        for s in steps:
            t = time.perf_counter()
            e2e_call(mg, plan, s, cfg, labels, do_a, do_b)
            e2e_t += time.perf_counter() - t
            d2h += d2h_bytes(mg, plan)
        if world > 1:
            e2e_t = allreduce(e2e_t, "max")
        acc["e2e"] = total_arcs / e2e_t / 1e9
        acc["d2h_per_step"] = d2h // len(steps)
        return acc

    def profiled(do_a, do_b, cfg):
        """the same K steps with per-kernel CUDA events on the library stream
        (host-driven loop): the roofline of the dominant kernel classes"""
        mg.lib().mg_plan_set_profiling(plan._h, 1)
        for s in sources:  # the host loop's scratch at its size before the timed steps
            e2e_call(mg, plan, s, cfg, None, do_a, do_b)
        barrier()
        acc = {"pull": [0.0, 0.0, 0], "push": [0.0, 0.0, 0], "dev_ms": 0.0, "xms": 0.0,
               "xbytes": 0}
        for s in steps:
            st = e2e_call(mg, plan, s, cfg, None, do_a, do_b)
            acc["dev_ms"] += st.device_ms
            acc["xms"] += st.exchange_ms
            acc["xbytes"] += st.exchange_bytes
            for key, ms, b, n in (("pull", st.kernel_ms, st.kernel_bytes, st.kernel_launches),
                                  ("push", st.kernel2_ms, st.kernel2_bytes,
                                   st.kernel2_launches)):
                acc[key][0] += ms
                acc[key][1] += b
                acc[key][2] += n
        barrier()
        mg.lib().mg_plan_set_profiling(plan._h, 0)
        return acc

    # headline: the reference's direction rule and defaults (primitives.hpp:69-70);
    # a logically-forward superstep whose exact edge count dwarfs the unvisited
    # list runs on the pull kernels (mg_config.dobfs_exact_cost).  Labels,
    # direction log, S and W are the reference's (tests/test_gpu_parity.py).
    main = timed(0.01, 0.1, exact_cfg)
    prof = profiled(0.01, 0.1, exact_cfg)
    # the same rule executed physically as the reference schedules it
    refsched = timed(0.01, 0.1, ref_cfg)
    tuned = timed(0.001, 0.1, exact_cfg)  # do_a tuned for RMAT
    kind = "push" if prof["push"][0] >= prof["pull"][0] else "pull"
    other = "pull" if kind == "push" else "push"
    k_ms, k_bytes, k_n = prof[kind]

    if rank != 0:
        return 0
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_reference((off, col), sources, arcs, args.cpu_seconds)
        except Exception as ex:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GTEPS", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {ex}"}
    achieved = k_bytes / (k_ms * 1e-3) / 1e9 if k_ms else None
    traffic, traffic_src = ncu_traffic(kind)
    hbm_roof = {
        "bound": "hbm",
        "kernel": "lb_expand (push advance)" if kind == "push"
        else "dobfs_pull (thread + group stages)",
        "achieved": round(achieved, 1) if achieved else None, "peak": hbm,
        "peak_kind": hbm_kind, "unit": "GB/s",
        "frac": round(achieved / hbm, 4) if achieved else None,
        "traffic": traffic, "traffic_source": traffic_src,
        "algorithmic_bytes_per_launch": k_bytes / max(k_n, 1),
        "avg_launch_ms": k_ms / max(k_n, 1),
        "share_of_step": round(k_ms / prof["dev_ms"], 4) if prof["dev_ms"] else None,
        "timing": "CUDA events around each launch pair on the library stream (profiled pass, "
                  "host-driven loop)",
        "other_kernel": {"kernel": other,
                         "achieved": round(prof[other][1] / (prof[other][0] * 1e-3) / 1e9, 1)
                         if prof[other][0] else None,
                         "share_of_step": round(prof[other][0] / prof["dev_ms"], 4)
                         if prof["dev_ms"] else None}}
    xchg = None
    if world > 1:
        # the device-driven loop runs the exchange inside one graph launch, so
        # its kernels are timed in the profiled (host-driven) pass
        xsrc = main if main["xms"] else prof
        xa = xsrc["xbytes"] / (xsrc["xms"] * 1e-3) / 1e9 if xsrc["xms"] else None
        xchg = {"bound": "nvlink", "kernel": "dobfs exchange pack + publish (P2P stores into "
                                             "peer inboxes)",
                "achieved": round(xa, 1) if xa else None, "peak": NVLINK_GBS,
                "peak_kind": "NVLink 5 nominal per direction per GPU", "unit": "GB/s",
                "frac": round(xa / NVLINK_GBS, 4) if xa else None, "traffic": None,
                "bytes_per_step": xsrc["xbytes"] / args.steps,
                "ms_per_step": round(xsrc["xms"] / args.steps, 4),
                "share_of_step": round(xsrc["xms"] / xsrc["dev_ms"], 4) if xsrc["dev_ms"] else None,
                "note": "rank 0: bytes its pack kernels stored into peer inboxes / their "
                        "CUDA-event time" + (" (every rank on one GPU: HBM, not NVLink)"
                                             if "MG_BENCH_DEVICE" in os.environ else "") +
                        ("" if xsrc is main else "; timed in the profiled host-driven pass")}
    roofline = dict(xchg, hbm_kernel=hbm_roof) if xchg else hbm_roof
    dev_ms = main["dev_max_ms"]
    loop = "device (CUDA-graph loop)" if main["device_loop"] == len(steps) else \
        "host-driven enactor loop" if main["device_loop"] == 0 else "mixed"
    line = {
        "metric": METRIC,
        "value": round(main["value"], 3),
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
        "config": workload_config(args, world, sources, plan.num_global_vertices,
                                  plan.num_global_edges),
        "run": {
            "policy": "max + fused",
            "physical_direction": "exact cost (pull when sum deg(Q) > 4 |unvisited|, "
                                  "summed over all partitions)",
            "loop": loop,
            "mean_reached_arcs": total_arcs // len(steps),
            "graph_prep_s": round(prep_s, 2),
            "plan_precompute_s": round(precompute_s, 3),
            "precompute_note": "first call on a plan builds the non-isolated vertex list "
                               "(device select + host sort), the 16-byte pull records and, "
                               "under 2^30 arcs, the CUDA-graph loop; excluded from value",
            "host_wall_s": round(main["wall"], 4),
            "timing": "CUDA events on the library stream around init + superstep loop, "
                      "summed over the K steps (max over ranks), profiling off",
        },
        "e2e": {"value": round(main["e2e"], 3), "unit": "GTEPS", "h2d_bytes_per_step": 4,
                "d2h_bytes_per_step": int(main["d2h_per_step"]),
                "note": "mg_dobfs with the labels into pinned host memory every step; h2d = the "
                        "4-byte source (a kernel argument); d2h = bytes the library copied "
                        "(u32 head + 4/8-bit tail of the level array, widened on the host)"},
        "roofline": roofline,
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
        "cpu_baseline": cpu,
        "clocks": main["clocks"],
        "gpu_launches": main["launches"],
    }
    print(json.dumps(line))
    return 0


def cpu_reference(graph_arrays, sources, arcs, max_s):
    """time the reference engine (oracle/_ref) on the same graph; n = 1 partition"""
    from oracle import ref
    off, col = graph_arrays
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
    return dict({"value": a / (ms * 1e-3) / 1e9, "unit": "GTEPS", "cores": 1,
                 "kind": "reference",
                 "sample": f"reference dobfs (n=1 partition, 1 thread) from sources {done}, "
                           f"{ms:.0f} ms engine wall_ms (plan build {prep:.1f} s excluded)"},
                **host_info())


# ------------------------------------------------------------------------------ reference arm
def reference_sweep(args, budget_s=60.0):
    """best partition count of the reference engine (one std::thread per partition,
    engine.hpp:951-959), chosen on a bounded sample: the same generator at scale - 4,
    two sources per n, n in {1, 2, 4, 8, 16} up to the host's cores"""
    from oracle import ref
    sc = max(args.scale - 4, 10)
    g = ref.RefGraph.rmat_hashed(sc, args.edge_factor, args.seed)
    off = g.offsets()
    deg = np.diff(off.astype(np.int64))
    nv = len(off) - 1
    srcs = pick_sources(off, 2)
    out, t0 = {}, time.time()
    for n in (1, 2, 4, 8, 16):
        if n > (os.cpu_count() or 1) or time.time() - t0 > budget_s:
            break
        own = ref.partition_random(nv, n, 7) if n > 1 else np.zeros(nv, np.uint32)
        p = ref.RefPlan(g, own, n)
        ms, a = 0.0, 0
        for s in srcs:
            r = p.dobfs(s)
            ms += r.stats.wall_ms
            a += reached_arcs(r.labels, deg)
        out[n] = a / (ms * 1e-3) / 1e9
        del p
    return sc, out


def run_reference(args, rank, n_gpus):
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    sweep_scale, sweep = reference_sweep(args)
    best_n = max(sweep, key=sweep.get) if sweep else 1
    # input synthesis (not timed): the oracle's own counter-based R-MAT builder,
    # bit-identical to the product's device generator, so this process never
    # maps libmgraph_b200.so
    t0 = time.time()
    rg = ref.RefGraph.rmat_hashed(args.scale, args.edge_factor, args.seed)
    gen_s = time.time() - t0
    nv, ne, _ = rg.info()
    off = rg.offsets()
    deg = np.diff(off.astype(np.int64))
    sources = pick_sources(off, args.num_sources)
    del off
    owner = ref.partition_random(nv, best_n, 7) if best_n > 1 else np.zeros(nv, np.uint32)
    t0 = time.time()
    rplan = ref.RefPlan(rg, owner, best_n)
    plan_s = time.time() - t0
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
    info = host_info()
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 4),
        "unit": "GTEPS", "n_gpus": n_gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (the same hashed R-MAT, built by the oracle's host generator)",
        "config": workload_config(args, n_gpus, sources, nv, ne),
        "cpu_baseline": dict({"value": round(v, 4), "unit": "GTEPS", "cores": best_n,
                              "kind": "reference",
                              "sample": f"{args.steps} reference dobfs runs (engine wall_ms, "
                                        f"engine.hpp:951-964) with n={best_n} partitions = "
                                        f"{best_n} worker threads (the engine runs one thread "
                                        f"per partition)"}, **info),
        "reference_engine": {
            "partitions": best_n,
            "sweep": {"scale": sweep_scale, "gteps_by_partitions": {str(k): round(x, 4)
                                                                   for k, x in sweep.items()},
                      "note": "best partition count picked on the scale-4 sample (2 sources "
                              "each), then used at full size"},
            "graph_gen_s": round(gen_s, 1), "plan_build_s": round(plan_s, 1),
            "graph_source": "oracle/gen_oracle.cpp (no product library in this process)"},
        "e2e": {"value": round(v, 4), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))
    return 0


if __name__ == "__main__":
    sys.exit(main())
