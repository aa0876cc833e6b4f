"""Multi-process path (one process per GPU).

CPU (world size 2, no GPU): the shared-memory rendezvous that carries the
barrier, the WorkerReport all-gather and the IPC-handle exchange, driven from
two processes that also agree on the job key through torch.distributed/gloo
(as bench.py does under torchrun).

GPU: two processes on ONE B200, each owning one partition of the same plan:
records cross between the processes through CUDA IPC mappings of each other's
inbox arenas, i.e. the exact multi-GPU code path minus the NVLink hop.  Each
rank's hosted results and the engine statistics must equal the single-process
two-partition run and the oracle.
"""
import os
import socket
import sys
import uuid

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _selftest_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_1504_04804_b200 as mg
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    obj = [uuid.uuid4().hex if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)  # job-unique fabric key, as in bench.py
    rc = mg.lib().mg_fabric_selftest(obj[0].encode(), rank, world, 200)
    msg = mg.lib().mg_last_error().decode() if rc else ""
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, rc, msg))


def _spawn(target, world, *args):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return sorted(out, key=lambda x: x[0])


@pytest.mark.parametrize("world", [2, 3])
def test_shm_rendezvous_gloo_world(world):
    res = _spawn(_selftest_worker, world)
    assert all(rc == 0 for _, rc, _ in res), res


def test_fabric_rejects_bad_arguments():
    import paper_1504_04804_b200 as mg
    assert mg.lib().mg_fabric_selftest(b"x", 3, 2, 1) != 0
    g = mg.Csr.path(4)
    with pytest.raises(ValueError):
        mg.PartitionPlan.multiprocess(g, np.array([0, 0, 1, 1], np.uint32), 2, 5, 0, "k")


def _gpu_worker(rank, world, port, q, case, fabric="device"):
    sys.path.insert(0, ROOT)
    if fabric == "host":  # shared-memory barrier + all-gather instead of device mailboxes
        os.environ["MG_HOST_FABRIC"] = "1"
    try:
        import torch.distributed as dist

        import paper_1504_04804_b200 as mg
        from oracle import seq
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        obj = [uuid.uuid4().hex if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        g = mg.Csr.rmat(12, 16, 1).with_weights(1, 64, 7)
        off, col, w = g.arrays()
        owner = mg.partition_random(g.num_vertices, world, 11)
        mine = owner == rank
        plan = mg.PartitionPlan.multiprocess(g, owner, world, rank, 0, obj[0])
        out = {}
        r = mg.bfs(plan, mg.BfsOptions(source=0))
        out["bfs"] = bool(np.array_equal(r.labels[mine], seq.bfs_levels(off, col, 0)[mine]))
        out["bfs_S"] = int(r.stats.supersteps)
        out["bfs_H"] = r.stats.h_matrix.tolist()
        r = mg.dobfs(plan, mg.DobfsOptions(source=0))
        out["dobfs"] = bool(np.array_equal(r.labels[mine], seq.bfs_levels(off, col, 0)[mine]))
        out["dobfs_dir"] = [int(x) for x in r.direction_log]
        r = mg.sssp(plan, 0)
        out["sssp"] = bool(np.array_equal(r.dists[mine], seq.dijkstra(off, col, w, 0)[mine]))
        r = mg.cc(plan)
        out["cc"] = bool(np.array_equal(r.components[mine],
                                        seq.connected_components(off, col)[mine]))
        r = mg.bc(plan, 1)
        bc, _, _ = seq.brandes_bc(off, col, 1)
        scale = np.maximum(np.maximum(np.abs(r.bc[mine]), np.abs(bc[mine])), 1e-12)
        out["bc"] = bool(np.all(np.abs(r.bc[mine] - bc[mine]) / scale <= 1e-5))
        r = mg.pagerank(plan, mg.PrOptions(epsilon=1e-6))
        ranks, it, _ = seq.pagerank_power(off, col, 0.85, 1e-6, 1000)
        out["pr"] = bool(np.max(np.abs(r.ranks[mine] - ranks[mine])) <= 1e-6)
        out["pr_iters"] = (int(r.iterations), int(it))
        del plan
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, 0, out))
    except Exception as ex:  # pragma: no cover - reported to the parent
        q.put((rank, 1, repr(ex)))


@pytest.mark.gpu
@pytest.mark.parametrize("fabric", ["device", "host"])
def test_two_processes_one_gpu_cuda_ipc_exchange(fabric):
    """device: publish flags and WorkerReports through IPC-mapped mailboxes,
    the barrier and the all-gather on the GPUs; host: the shm rendezvous"""
    import paper_1504_04804_b200 as mg
    res = _spawn(_gpu_worker, 2, "rmat12", fabric)
    assert all(rc == 0 for _, rc, _ in res), res
    outs = [o for _, _, o in res]
    for o in outs:
        for k in ("bfs", "dobfs", "sssp", "cc", "bc", "pr"):
            assert o[k], (k, o)
        assert o["pr_iters"][0] == o["pr_iters"][1]
    # both ranks saw the same global view, equal to the single-process run
    assert outs[0]["bfs_H"] == outs[1]["bfs_H"] and outs[0]["bfs_S"] == outs[1]["bfs_S"]
    g = mg.Csr.rmat(12, 16, 1).with_weights(1, 64, 7)
    owner = mg.partition_random(g.num_vertices, 2, 11)
    single = mg.bfs(mg.PartitionPlan(g, owner, 2), mg.BfsOptions(source=0))
    assert outs[0]["bfs_S"] == single.stats.supersteps
    assert outs[0]["bfs_H"] == single.stats.h_matrix.tolist()
    dob = mg.dobfs(mg.PartitionPlan(g, owner, 2), mg.DobfsOptions(source=0))
    assert outs[0]["dobfs_dir"] == [int(x) for x in dob.direction_log]


def _gpu_worker_dobfs(rank, world, port, q, fabric):
    sys.path.insert(0, ROOT)
    if fabric == "host":
        os.environ["MG_HOST_FABRIC"] = "1"
    try:
        import torch.distributed as dist

        import paper_1504_04804_b200 as mg
        from oracle import seq
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        obj = [uuid.uuid4().hex if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        g = mg.Csr.rmat(11, 16, 4)
        off, col, _ = g.arrays()
        owner = mg.partition_random(g.num_vertices, world, 5)
        mine = owner == rank
        plan = mg.PartitionPlan.multiprocess(g, owner, world, rank, 0, obj[0])
        want = seq.bfs_levels(off, col, 0)
        out = {}
        for name, cfg in (("ref", None), ("exact", mg.EngineConfig(dobfs_exact_cost=True))):
            r = mg.dobfs(plan, mg.DobfsOptions(source=0), cfg)
            out[name] = bool(np.array_equal(r.labels[mine], want[mine]))
            out[name + "_dir"] = [int(x) for x in r.direction_log]
            out[name + "_S"] = int(r.stats.supersteps)
        del plan
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, 0, out))
    except Exception as ex:  # pragma: no cover
        q.put((rank, 1, repr(ex)))


@pytest.mark.gpu
def test_three_processes_dobfs_device_fabric_and_exact_cost():
    """three ranks (one GPU): reference schedule and the exact-cost extension
    through the device-side protocol agree with the oracle and with each other"""
    res = _spawn(_gpu_worker_dobfs, 3, "device")
    assert all(rc == 0 for _, rc, _ in res), res
    outs = [o for _, _, o in res]
    for o in outs:
        assert o["ref"] and o["exact"], o
        assert o["ref_dir"] == o["exact_dir"] and o["ref_S"] == o["exact_S"]
    assert all(o["ref_dir"] == outs[0]["ref_dir"] for o in outs)


def _gpu_worker_dobfs_loop(rank, world, port, q, scale):
    """DOBFS through the device-driven superstep loop (one CUDA graph per
    rank) and through the host loop on the same plan: everything the run
    reports must be identical"""
    sys.path.insert(0, ROOT)
    try:
        import torch.distributed as dist

        import paper_1504_04804_b200 as mg
        from oracle import seq
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        obj = [uuid.uuid4().hex if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        g = mg.Csr.rmat(scale, 16, 2)
        off, col, _ = g.arrays()
        owner = mg.partition_random(g.num_vertices, world, 7)
        mine = owner == rank
        plan = mg.PartitionPlan.multiprocess(g, owner, world, rank, 0, obj[0])
        out = {}
        for exact in (False, True):
            cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                                  dobfs_exact_cost=exact)
            for src in (0, 5):
                want = seq.bfs_levels(off, col, src)
                res = {}
                for mode in ("0", "1", "1"):  # host loop, device loop (twice: graph reuse)
                    os.environ["MG_MP_GRAPH_LOOP"] = mode
                    r = mg.dobfs(plan, mg.DobfsOptions(source=src), cfg)
                    st = r.stats
                    res.setdefault(mode, []).append(dict(
                        ok=bool(np.array_equal(r.labels[mine], want[mine])),
                        dir=[int(x) for x in r.direction_log], S=int(st.supersteps),
                        W=int(st.edges_examined), C=int(st.combine_ops),
                        H=st.h_matrix.astype(int).tolist(),
                        Hi=st.h_per_iter_by_src.astype(int).tolist(),
                        out=st.out_per_iter.astype(int).tolist(),
                        loop=bool(st.device_loop), stop=st.stop_reason,
                        fe=int(r.forward_edges), be=int(r.backward_edges)))
                out[f"{int(exact)}_{src}"] = res
        del plan
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, 0, out))
    except Exception as ex:  # pragma: no cover
        q.put((rank, 1, repr(ex)))


@pytest.mark.gpu
@pytest.mark.parametrize("world,scale", [(2, 12), (3, 11), (4, 10)])
def test_dobfs_device_loop_equals_host_loop(world, scale):
    """the whole superstep loop on the device (decide, pull / push, pack,
    publish, merge, report all-gather, convergence) gives the host loop's
    labels, direction log, S, W, C, H matrix, per-iteration H and frontier
    sizes, on every rank, for the reference schedule and the exact-cost
    extension"""
    res = _spawn(_gpu_worker_dobfs_loop, world, scale)
    assert all(rc == 0 for _, rc, _ in res), res
    for _, _, o in res:
        for key, r in o.items():
            host, dev = r["0"][0], r["1"]
            assert host["ok"] and not host["loop"], (key, host)
            for d in dev:
                assert d["loop"], (key, d)
                for k in ("ok", "dir", "S", "W", "C", "H", "Hi", "out", "stop", "fe", "be"):
                    assert d[k] == host[k], (key, k, d[k], host[k])
