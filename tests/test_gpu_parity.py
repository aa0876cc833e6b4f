"""Parity of the CUDA path against the oracle (GPU).

Inputs are built by the kept host preparation (bit-identical to the reference,
tests/test_host.py); results come from the sm_100a kernels through the C-ABI
and are compared with
  * oracle.seq — the C restatement of the reference's sequential oracles, and
  * oracle.ref — the unmodified reference engine (same plan, same config) for
    the engine-level statistics S / W / C / H that the reference's own tests pin.
Bars (BASELINE.json north_star): labels / components / integer distances
bit-exact; BFS preds a legal tree; PageRank <= 1e-6 per vertex and the same
iteration count; BC <= 1e-5 relative (CLI validate rule, tools/mgraph.cpp:478-489).
"""
import numpy as np
import pytest

import paper_1504_04804_b200 as mg
from oracle import ref, seq

pytestmark = pytest.mark.gpu

PARTS = [1, 2, 3, 4, 8]


def graphs():
    return {
        "p4": mg.Csr.path(4),
        "star5": mg.Csr.from_edges(5, [[0, 1], [0, 2], [0, 3], [0, 4]]).symmetrize_dedup(),
        "tri_iso": mg.Csr.from_edges(4, [[0, 1], [1, 2], [0, 2]]).symmetrize_dedup(),
        "rmat12": mg.Csr.rmat(12, 16, 1),
        "grid32": mg.Csr.grid(32, 32),
    }


@pytest.fixture(scope="module")
def G():
    return graphs()


def plan_for(g, n, seed=7, dup=mg.Duplication.All, biased=False):
    owner = (mg.partition_biased_random(g, n, seed, 1.0) if biased
             else mg.partition_random(g.num_vertices, n, seed))
    return mg.PartitionPlan(g, owner, n, dup), owner


def rel_close(a, b, tol):
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-12)
    return np.all(np.abs(a - b) / scale <= tol)


# --------------------------------------------------------------------------- BFS
@pytest.mark.parametrize("n", PARTS)
@pytest.mark.parametrize("name", ["p4", "star5", "tri_iso", "rmat12", "grid32"])
def test_bfs_labels_and_stats_match_reference(G, name, n):
    g = G[name]
    off, col, _ = g.arrays()
    plan, owner = plan_for(g, n, seed=3 * n + 1)
    for src in (0, g.num_vertices - 1):
        r = mg.bfs(plan, mg.BfsOptions(source=src))
        assert np.array_equal(r.labels, seq.bfs_levels(off, col, src))
        finite = r.labels[r.labels != mg.kInfLabel]
        assert r.stats.supersteps == int(finite.max()) + 1  # CLI:339-346
        if ref.available():
            rp = ref.RefPlan(ref.RefGraph.from_csr(off, col), owner, n)
            rr = rp.bfs(src)
            assert r.stats.supersteps == rr.stats.supersteps
            assert r.stats.edges_examined == rr.stats.edges_examined
            assert r.stats.combine_ops == rr.stats.combine_ops
            assert np.array_equal(r.stats.h_matrix, rr.h_matrix)
            assert np.array_equal(r.stats.h_per_iter_by_src, rr.h_per_iter)


def test_bfs_p4_engine_trace(golden):
    pins, _ = golden
    pin = pins["bfs_p4_two_way"]
    plan = mg.PartitionPlan(mg.Csr.path(4), np.array(pin["owner"], np.uint32), 2)
    r = mg.bfs(plan, mg.BfsOptions(source=0))
    assert list(r.labels) == pin["labels"]
    assert r.stats.supersteps == pin["supersteps"]
    assert r.stats.h_total() == pin["h_total"]
    assert r.stats.h_matrix.tolist() == pin["h_matrix"]
    assert r.stats.combine_ops == pin["combine_ops"]


@pytest.mark.parametrize("n", [1, 3, 4])
def test_bfs_preds_form_a_legal_tree(n):
    g = mg.Csr.rmat(9, 8, 4)
    off, col, _ = g.arrays()
    plan, _ = plan_for(g, n, seed=2)
    r = mg.bfs(plan, mg.BfsOptions(source=0, mark_preds=True))
    depth = seq.bfs_levels(off, col, 0)
    for v in range(g.num_vertices):
        if v == 0 or r.labels[v] == mg.kInfLabel:
            continue
        p = int(r.preds[v])
        assert p != mg.kInvalidVertex
        assert depth[p] + 1 == depth[v]
        assert v in col[off[p]:off[p + 1]]


def test_bfs_golden_rmat12_n4(golden):
    _, vec = golden
    g = mg.Csr.from_csr(vec["rmat12_off"], vec["rmat12_col"])
    plan = mg.PartitionPlan(g, vec["rmat12_n4_owner"], 4)
    r = mg.bfs(plan, mg.BfsOptions(source=0))
    assert np.array_equal(r.labels, vec["rmat12_n4_bfs_labels"])
    assert r.stats.supersteps == int(vec["rmat12_n4_bfs_S"])
    assert r.stats.edges_examined == int(vec["rmat12_n4_bfs_W"])
    assert r.stats.combine_ops == int(vec["rmat12_n4_bfs_C"])
    assert np.array_equal(r.stats.h_matrix, vec["rmat12_n4_bfs_H"])


def test_bfs_config1_rmat18(golden):
    """configs[0]: RMAT-18/16 seed 1, single partition, source 0"""
    _, vec = golden
    g = mg.Csr.rmat(18, 16, 1)
    plan = mg.PartitionPlan(g, None, 1)
    for cfg in (None, mg.EngineConfig(policy=mg.AllocPolicyKind.PreallocFused)):
        r = mg.bfs(plan, mg.BfsOptions(source=0), cfg)
        assert np.array_equal(r.labels, vec["rmat18_bfs0"])
        assert r.stats.supersteps == 5


def test_bfs_isolated_source_and_errors():
    g = mg.Csr.from_edges(4, [[0, 1], [1, 2], [0, 2]]).symmetrize_dedup()
    plan, _ = plan_for(g, 2, 5)
    r = mg.bfs(plan, mg.BfsOptions(source=3))
    assert r.labels[3] == 0 and all(r.labels[:3] == mg.kInfLabel)
    with pytest.raises(ValueError):
        mg.bfs(plan, mg.BfsOptions(source=99))  # primitives.cpp:27-30
    onehop = mg.PartitionPlan(mg.Csr.path(4), np.array([0, 0, 1, 1], np.uint32), 2,
                              mg.Duplication.OneHop)
    with pytest.raises(ValueError):
        mg.bfs(onehop, mg.BfsOptions(source=0))  # engine.hpp:716-719


# --------------------------------------------------------------------------- DOBFS
@pytest.mark.parametrize("n", [1, 2, 3, 4])
@pytest.mark.parametrize("name", ["p4", "star5", "tri_iso", "rmat12"])
@pytest.mark.parametrize("do_a,do_b", [(0.01, 0.1), (0.001, 0.1), (0.5, 0.9)])
def test_dobfs_labels_direction_log_and_work(G, name, n, do_a, do_b):
    g = G[name]
    off, col, _ = g.arrays()
    plan, owner = plan_for(g, n, seed=n + 3)
    r = mg.dobfs(plan, mg.DobfsOptions(source=0, do_a=do_a, do_b=do_b))
    assert np.array_equal(r.labels, seq.bfs_levels(off, col, 0))
    if ref.available():
        rr = ref.RefPlan(ref.RefGraph.from_csr(off, col), owner, n).dobfs(0, do_a, do_b)
        assert list(r.direction_log) == list(rr.direction_log)
        assert r.stats.supersteps == rr.stats.supersteps
        assert r.stats.edges_examined == rr.stats.edges_examined  # first-hit scan count
        assert r.forward_edges == rr.forward_edges and r.backward_edges == rr.backward_edges
        assert np.array_equal(r.stats.h_matrix, rr.h_matrix)


@pytest.mark.parametrize("scale,ef,seed", [(12, 16, 1), (12, 32, 6), (14, 16, 3)])
def test_dobfs_exact_cost_extension_keeps_reference_semantics(scale, ef, seed):
    """dobfs_exact_cost runs heavy forward supersteps with the pull kernel; the
    labels, direction log, S and W reported must still be the reference's"""
    g = mg.Csr.rmat(scale, ef, seed)
    off, col, _ = g.arrays()
    plan = mg.PartitionPlan(g, None, 1)
    for src in (0, 7):
        for do_a in (0.01, 0.001):
            a = mg.dobfs(plan, mg.DobfsOptions(source=src, do_a=do_a))
            b = mg.dobfs(plan, mg.DobfsOptions(source=src, do_a=do_a, mark_preds=True),
                         mg.EngineConfig(dobfs_exact_cost=True))
            assert np.array_equal(a.labels, b.labels)
            assert np.array_equal(b.labels, seq.bfs_levels(off, col, src))
            assert list(a.direction_log) == list(b.direction_log)
            assert a.stats.supersteps == b.stats.supersteps
            assert a.stats.edges_examined == b.stats.edges_examined
            depth = seq.bfs_levels(off, col, src)
            for v in np.nonzero(b.labels != mg.kInfLabel)[0][:500]:
                if v == src:
                    continue
                p = int(b.preds[v])
                assert depth[p] + 1 == depth[v] and v in col[off[p]:off[p + 1]]


def test_dobfs_work_reduction_and_broadcast_bound():
    g = mg.Csr.rmat(12, 32, 6)
    plan, _ = plan_for(g, 2, 4)
    plain = mg.bfs(plan, mg.BfsOptions(source=0))
    dob = mg.dobfs(plan, mg.DobfsOptions(source=0))
    assert np.array_equal(dob.labels, plain.labels)
    assert (dob.direction_log == 1).sum() > 0
    assert dob.stats.edges_examined < plain.stats.edges_examined
    for n in (2, 4):
        plan, _ = plan_for(mg.Csr.rmat(10, 16, 2), n, n)
        r = mg.dobfs(plan, mg.DobfsOptions(source=0))
        for i in range(n):
            assert r.stats.h_from(i) <= (n - 1) * 1024


def test_dobfs_preds_legal():
    g = mg.Csr.rmat(11, 16, 9)
    off, col, _ = g.arrays()
    depth = seq.bfs_levels(off, col, 0)
    for n in (1, 3):
        plan, _ = plan_for(g, n, 1)
        r = mg.dobfs(plan, mg.DobfsOptions(source=0, mark_preds=True))
        reach = np.nonzero(r.labels != mg.kInfLabel)[0]
        for v in reach:
            if v == 0:
                continue
            p = int(r.preds[v])
            assert depth[p] + 1 == depth[v] and v in col[off[p]:off[p + 1]]


# --------------------------------------------------------------------------- SSSP
@pytest.mark.parametrize("n", PARTS)
def test_sssp_equals_dijkstra(n):
    g = mg.Csr.rmat(12, 16, 1).with_weights(0, 64, 2)
    off, col, w = g.arrays()
    for biased in (False, True):
        plan, owner = plan_for(g, n, 13 * n, biased=biased)
        r = mg.sssp(plan, 0)
        assert np.array_equal(r.dists, seq.dijkstra(off, col, w, 0))
        if ref.available():
            rr = ref.RefPlan(ref.RefGraph.from_csr(off, col, w), owner, n).sssp(0)
            assert r.stats.supersteps == rr.stats.supersteps
            assert np.array_equal(r.stats.h_matrix, rr.h_matrix)


FUSED_CFGS = [mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On),
              mg.EngineConfig(policy=mg.AllocPolicyKind.JustEnough, fused=mg.FusedMode.On),
              mg.EngineConfig(policy=mg.AllocPolicyKind.PreallocFused)]


@pytest.mark.parametrize("name", ["rmat12", "grid32", "star5", "tri_iso", "rmat14"])
def test_sssp_dense_supersteps_match_reference(name):
    """One partition under a fused policy: supersteps whose frontier holds at least
    |V|/32 vertices relax with fire-and-forget atomics and list their output by
    comparing the distances with the superstep's snapshot (prims.cu SsspDev::red).
    Distances, S, W, per-superstep frontier sizes and edge counts equal the
    reference engine's (primitives.cpp:334-356)."""
    g = (mg.Csr.rmat(14, 16, 5) if name == "rmat14" else graphs()[name]).with_weights(0, 64, 9)
    off, col, w = g.arrays()
    plan, owner = plan_for(g, 1)
    rr = ref.RefPlan(ref.RefGraph.from_csr(off, col, w), owner, 1).sssp(0) \
        if ref.available() else None
    for cfg in FUSED_CFGS:
        r = mg.sssp(plan, 0, cfg=cfg)
        assert np.array_equal(r.dists, seq.dijkstra(off, col, w, 0))
        if rr is not None:
            assert r.stats.supersteps == rr.stats.supersteps
            assert r.stats.edges_examined == rr.stats.edges_examined
            assert np.array_equal(r.stats.out_per_iter, rr.out_per_iter)
            assert np.array_equal(r.stats.edges_per_iter, rr.edges_per_iter)


@pytest.mark.parametrize("name", ["rmat12", "grid32", "star5", "rmat14"])
def test_bc_dense_forward_matches_reference(name):
    """One partition under a fused policy: large forward supersteps label with
    plain stores and list their output by level (prims.cu BcDev::red); sigma is
    bit-exact, bc within 1e-5, S and per-superstep frontier sizes equal the
    reference engine's."""
    g = mg.Csr.rmat(14, 16, 5) if name == "rmat14" else graphs()[name]
    off, col, _ = g.arrays()
    plan, owner = plan_for(g, 1)
    bc, sigma, dist = seq.brandes_bc(off, col, 1)
    rr = ref.RefPlan(ref.RefGraph.from_csr(off, col), owner, 1).bc(1) if ref.available() else None
    for cfg in FUSED_CFGS:
        r = mg.bc(plan, 1, cfg=cfg)
        assert np.array_equal(r.labels, dist)
        assert np.array_equal(r.sigma, sigma)
        assert rel_close(r.bc, bc, 1e-5)
        if rr is not None:
            assert r.stats.supersteps == rr.stats.supersteps
            assert np.array_equal(r.stats.out_per_iter, rr.out_per_iter)


def test_sssp_pins_and_errors(golden):
    pins, _ = golden
    pin = pins["sssp_p4_weighted"]
    g = mg.Csr.from_edges(4, pin["edges"], weighted=True).symmetrize_dedup()
    plan = mg.PartitionPlan(g, np.array(pin["owner"], np.uint32), 2)
    assert list(mg.sssp(plan, 0).dists) == pin["dists"]
    with pytest.raises(ValueError):
        mg.sssp(mg.PartitionPlan(mg.Csr.path(4), np.array([0, 0, 1, 1], np.uint32), 2), 0)


# --------------------------------------------------------------------------- CC
@pytest.mark.parametrize("n", PARTS)
@pytest.mark.parametrize("name", ["tri_iso", "rmat12", "grid32", "star5"])
def test_cc_equals_union_find(G, name, n):
    g = G[name]
    off, col, _ = g.arrays()
    plan, owner = plan_for(g, n, 5 * n + 2)
    r = mg.cc(plan)
    assert np.array_equal(r.components, seq.connected_components(off, col))
    # W in the reference's unit (primitives.cpp:441-457): |E_i| per hook sweep, at
    # least one sweep per worker per superstep (the sweep count of a parallel
    # hook is its own, so W is not compared with the sequential loop's)
    E = len(col)
    assert all(int(e) >= E for e in r.stats.edges_per_iter)
    if n == 1:
        assert r.stats.edges_examined % max(E, 1) == 0
        assert r.stats.edges_examined >= r.stats.supersteps * E
    if ref.available():
        rr = ref.RefPlan(ref.RefGraph.from_csr(off, col), owner, n).cc()
        assert r.stats.supersteps == rr.stats.supersteps
        assert np.array_equal(r.stats.h_matrix, rr.h_matrix)


def test_cc_edgeless_and_fixed_comm():
    g = mg.Csr.from_edges(5, [])
    plan, _ = plan_for(g, 2, 3)
    assert list(mg.cc(plan).components) == [0, 1, 2, 3, 4]
    p4 = mg.PartitionPlan(mg.Csr.path(4), np.array([0, 0, 1, 1], np.uint32), 2)
    with pytest.raises(ValueError):
        mg.cc(p4, mg.EngineConfig(comm_override=mg.CommMode.Selective))


# --------------------------------------------------------------------------- BC
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_bc_matches_brandes(n):
    g = mg.Csr.rmat(10, 8, 12)
    off, col, _ = g.arrays()
    plan, owner = plan_for(g, n, 17 * n + 3)
    r = mg.bc(plan, 1)
    bc, sigma, dist = seq.brandes_bc(off, col, 1)
    assert rel_close(r.bc, bc, 1e-5)
    assert np.array_equal(r.sigma, sigma)
    assert np.array_equal(r.labels, dist)
    if ref.available():
        rr = ref.RefPlan(ref.RefGraph.from_csr(off, col), owner, n).bc(1)
        assert r.stats.supersteps == rr.stats.supersteps
        assert np.array_equal(r.stats.h_matrix, rr.h_matrix)


def test_bc_pins(golden):
    pins, _ = golden
    plan = mg.PartitionPlan(mg.Csr.path(4), np.array([0, 0, 1, 1], np.uint32), 2)
    assert list(mg.bc(plan, 0).bc) == pins["bc_p4"]["bc"]
    g = mg.Csr.from_edges(5, [[0, 1], [0, 2], [0, 3], [0, 4]]).symmetrize_dedup()
    plan, _ = plan_for(g, 2, 3)
    assert mg.bc(plan, 1).bc[0] == pytest.approx(3.0)


# --------------------------------------------------------------------------- PR
@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("dup", [mg.Duplication.All, mg.Duplication.OneHop])
def test_pagerank_matches_power_iteration(n, dup):
    g = mg.Csr.rmat(10, 8, 21)
    off, col, _ = g.arrays()
    plan, owner = plan_for(g, n, 3 * n + 7, dup=dup)
    for eps in (1e-4, 1e-6):
        r = mg.pagerank(plan, mg.PrOptions(epsilon=eps))
        ranks, it, _ = seq.pagerank_power(off, col, 0.85, eps, 1000)
        assert r.iterations == it
        assert np.max(np.abs(r.ranks - ranks)) <= 1e-6
        assert np.all(np.abs(np.array(r.rank_sums) - 1.0) <= 1e-9)
    r = mg.pagerank(plan, mg.PrOptions(max_iter=5))
    pair = plan.pair_border()
    for per_src in r.stats.h_per_iter_by_src:  # TP:359-370: H per iteration == |B_i|
        assert list(per_src) == [int(pair[i].sum()) for i in range(n)]


def test_pagerank_small_cases_and_validation():
    g = mg.Csr.from_edges(1, [])
    r = mg.pagerank(mg.PartitionPlan(g, None, 1), mg.PrOptions())
    assert abs(r.ranks[0] - 1.0) <= 1e-12
    g = mg.Csr.rmat(8, 4, 5)
    off, col, _ = g.arrays()
    plan, _ = plan_for(g, 2, 6)
    r = mg.pagerank(plan, mg.PrOptions(max_iter=1))
    assert r.stats.supersteps == 1 and r.iterations == 1
    ranks, _, _ = seq.pagerank_power(off, col, 0.85, 0.01, 1)
    assert np.max(np.abs(r.ranks - ranks)) <= 1e-12
    p4 = mg.PartitionPlan(mg.Csr.path(4), np.array([0, 0, 1, 1], np.uint32), 2)
    for bad in (mg.PrOptions(damping=1.5), mg.PrOptions(epsilon=0.0), mg.PrOptions(max_iter=0)):
        with pytest.raises(ValueError):
            mg.pagerank(p4, bad)


# --------------------------------------------------------------------------- engine config
def test_allocation_policies_do_not_change_results():
    g = mg.Csr.rmat(9, 8, 14).with_weights(0, 64, 15)
    plan, _ = plan_for(g, 3, 6)
    base = mg.bfs(plan, mg.BfsOptions(source=0))
    base_pr = mg.pagerank(plan, mg.PrOptions(max_iter=10))
    for kind in (mg.AllocPolicyKind.JustEnough, mg.AllocPolicyKind.FixedPrealloc,
                 mg.AllocPolicyKind.Maximum, mg.AllocPolicyKind.PreallocFused):
        cfg = mg.EngineConfig(policy=kind)
        assert np.array_equal(mg.bfs(plan, mg.BfsOptions(source=0), cfg).labels, base.labels)
        pr = mg.pagerank(plan, mg.PrOptions(max_iter=10), cfg)
        assert np.max(np.abs(pr.ranks - base_pr.ranks)) <= 1e-12


def test_fused_policy_has_no_intermediate_frontier_and_cap_aborts():
    g = mg.Csr.rmat(10, 8, 18)
    plan, _ = plan_for(g, 2, 3)
    rf = mg.bfs(plan, mg.BfsOptions(source=0), mg.EngineConfig(policy=mg.AllocPolicyKind.PreallocFused))
    ru = mg.bfs(plan, mg.BfsOptions(source=0))
    assert np.array_equal(rf.labels, ru.labels)
    for p in range(2):
        assert rf.stats.worker_buffers[p]["advance_output"].peak_items == 0
    assert ru.stats.reallocs > 0
    with pytest.raises(mg.CapacityError):
        mg.bfs(plan, mg.BfsOptions(source=0), mg.EngineConfig(hard_cap_bytes=256))
    with pytest.raises(ValueError):
        mg.bfs(plan, mg.BfsOptions(source=0),
               mg.EngineConfig(policy=mg.AllocPolicyKind.FixedPrealloc, factors={"outbox": -0.5}))


def test_broadcast_override_agrees_with_selective():
    g = mg.Csr.rmat(9, 8, 6).with_weights(0, 64, 7)
    plan, _ = plan_for(g, 3, 2)
    cfg = mg.EngineConfig(comm_override=mg.CommMode.Broadcast)
    a, b = mg.bfs(plan, mg.BfsOptions(source=0)), mg.bfs(plan, mg.BfsOptions(source=0), cfg)
    assert np.array_equal(a.labels, b.labels) and b.stats.communication == "broadcast"
    assert np.array_equal(mg.sssp(plan, 0).dists, mg.sssp(plan, 0, cfg=cfg).dists)


def test_drop_package_fault_injection_changes_h():
    plan = mg.PartitionPlan(mg.Csr.path(4), np.array([0, 0, 1, 1], np.uint32), 2)
    r = mg.bfs(plan, mg.BfsOptions(source=0),
               mg.EngineConfig(drop_package=mg.DropPackage(0, 1, 1)))
    assert r.stats.h_matrix[0][1] == 0  # the only 0->1 package was dropped
    assert r.labels[2] == mg.kInfLabel


def test_run_stats_json_has_the_reference_schema():
    """RunStats.to_json mirrors stats_json.hpp:28-61 key for key"""
    import json
    g = mg.Csr.rmat(10, 8, 3)
    plan, _ = plan_for(g, 2, 5)
    r = mg.bfs(plan, mg.BfsOptions(source=0))
    j = r.stats.to_json(partitioner="random", duplication="all")
    assert set(j) == {"primitive", "n", "partitioner", "duplication", "communication", "policy",
                      "S", "W", "C", "H", "H_total", "H_per_iter_by_src", "out_per_iter",
                      "edges_per_iter", "wall_ms", "exchange_ms", "h_inflation",
                      "wire_records", "stop_reason", "peak_bytes", "reallocs", "buffers"}
    assert j["primitive"] == "bfs" and j["n"] == 2 and j["S"] == r.stats.supersteps
    assert j["H_total"] == sum(map(sum, j["H"])) == r.stats.h_total()
    assert len(j["buffers"]) == 2
    json.dumps(j)  # serialisable


@pytest.mark.parametrize("scale,ef,seed", [(12, 16, 1), (14, 16, 3)])
def test_bfs_exact_cost_extension_keeps_bfs_semantics(scale, ef, seed):
    """BFS with dobfs_exact_cost: heavy supersteps pull physically; labels, S and
    W equal the plain BFS (and the oracle); preds stay a legal tree"""
    g = mg.Csr.rmat(scale, ef, seed)
    off, col, _ = g.arrays()
    plan = mg.PartitionPlan(g, None, 1)
    for src in (0, 5):
        a = mg.bfs(plan, mg.BfsOptions(source=src))
        b = mg.bfs(plan, mg.BfsOptions(source=src, mark_preds=True),
                   mg.EngineConfig(dobfs_exact_cost=True))
        assert np.array_equal(b.labels, seq.bfs_levels(off, col, src))
        assert np.array_equal(a.labels, b.labels)
        assert a.stats.supersteps == b.stats.supersteps
        assert a.stats.edges_examined == b.stats.edges_examined
        for v in np.nonzero(b.labels != mg.kInfLabel)[0][:500]:
            if v == src:
                continue
            p = int(b.preds[v])
            assert b.labels[p] + 1 == b.labels[v] and v in col[off[p]:off[p + 1]]


@pytest.mark.parametrize("n", [2, 3, 4])
def test_dobfs_exact_cost_several_partitions(n):
    """exact-cost DOBFS on several partitions: one global physical direction per
    superstep; labels, direction log, S and W stay the reference's; the records
    sent (H) can only shrink (a pull discovers hosted vertices once)"""
    g = mg.Csr.rmat(13, 16, 2)
    off, col, _ = g.arrays()
    plan, owner = plan_for(g, n, 9 * n + 1)
    want = seq.bfs_levels(off, col, 0)
    for do_a in (0.01, 0.001):
        a = mg.dobfs(plan, mg.DobfsOptions(source=0, do_a=do_a))
        b = mg.dobfs(plan, mg.DobfsOptions(source=0, do_a=do_a, mark_preds=True),
                     mg.EngineConfig(dobfs_exact_cost=True))
        assert np.array_equal(b.labels, want)
        assert list(a.direction_log) == list(b.direction_log)
        assert a.stats.supersteps == b.stats.supersteps
        assert a.stats.edges_examined == b.stats.edges_examined
        assert b.stats.h_total() <= a.stats.h_total()
        for v in np.nonzero(b.labels != mg.kInfLabel)[0][:300]:
            if v == 0:
                continue
            p = int(b.preds[v])
            assert b.labels[p] + 1 == b.labels[v] and v in col[off[p]:off[p + 1]]


GRAPH_CFG = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                            dobfs_exact_cost=True)


def _host_loop(fn):
    import os
    os.environ["MG_NO_GRAPH"] = "1"
    try:
        return fn()
    finally:
        del os.environ["MG_NO_GRAPH"]


@pytest.mark.parametrize("scale,ef,seed", [(12, 16, 1), (14, 16, 3), (12, 32, 6)])
def test_dobfs_graph_loop_equals_host_loop(scale, ef, seed):
    """the device-driven superstep loop (one CUDA graph with WHILE/IF nodes)
    reproduces the host-driven run: labels, direction log, S, W and the
    per-superstep frontier sizes and edge counts"""
    g = mg.Csr.rmat(scale, ef, seed)
    off, col, _ = g.arrays()
    plan = mg.PartitionPlan(g, None, 1)
    for src in (0, 3, 77):
        for do_a in (0.01, 0.001):
            opt = mg.DobfsOptions(source=src, do_a=do_a, mark_preds=True)
            a = mg.dobfs(plan, opt, GRAPH_CFG)
            b = _host_loop(lambda: mg.dobfs(plan, opt, GRAPH_CFG))
            assert np.array_equal(a.labels, seq.bfs_levels(off, col, src))
            assert np.array_equal(a.labels, b.labels)
            assert list(a.direction_log) == list(b.direction_log)
            assert a.stats.supersteps == b.stats.supersteps
            assert a.stats.edges_examined == b.stats.edges_examined
            assert np.array_equal(a.stats.edges_per_iter, b.stats.edges_per_iter)
            assert np.array_equal(a.stats.out_per_iter, b.stats.out_per_iter)
            assert a.forward_edges == b.forward_edges and a.backward_edges == b.backward_edges
            for v in np.nonzero(a.labels != mg.kInfLabel)[0][:300]:
                if v == src:
                    continue
                p = int(a.preds[v])
                assert a.labels[p] + 1 == a.labels[v] and v in col[off[p]:off[p + 1]]
    # the BFS schedule through the same graph
    a = mg.bfs(plan, mg.BfsOptions(source=0), GRAPH_CFG)
    b = mg.bfs(plan, mg.BfsOptions(source=0))
    assert np.array_equal(a.labels, b.labels)
    assert a.stats.supersteps == b.stats.supersteps
    assert a.stats.edges_examined == b.stats.edges_examined


def test_dobfs_graph_loop_max_supersteps_and_isolated_source():
    g = mg.Csr.rmat(12, 16, 1)
    off, col, _ = g.arrays()
    plan = mg.PartitionPlan(g, None, 1)
    cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                          dobfs_exact_cost=True, max_supersteps=2)
    a = mg.dobfs(plan, mg.DobfsOptions(source=0), cfg)
    b = _host_loop(lambda: mg.dobfs(plan, mg.DobfsOptions(source=0), cfg))
    assert a.stats.supersteps == b.stats.supersteps == 2
    assert np.array_equal(a.labels, b.labels)
    assert a.stats.stop_reason == b.stats.stop_reason
    iso = int(np.nonzero(np.diff(off) == 0)[0][0])
    r = mg.dobfs(plan, mg.DobfsOptions(source=iso), GRAPH_CFG)
    assert r.labels[iso] == 0 and int((r.labels != mg.kInfLabel).sum()) == 1
    assert r.stats.supersteps == 1


FIRST_HIT_POS = list(range(15)) + [17, 18, 19, 25, 26, 33, 42, 43, 50, 58, 75, 90]


def _first_hit_graph():
    """source 0 -> hub 1 -> rows x whose first frontier neighbour (the hub) sits at
    arc position k, followed by 0/1/5/20 more arcs: the pull's record arcs
    (0-1), its in-thread stages (arcs 2-17) and the cooperative stage (18+),
    whose first round tests 8 arcs and later rounds 8 * kGroupSectors"""
    adj = [[1], [0]]
    for k in FIRST_HIT_POS:
        for t in (0, 1, 5, 20):
            x = len(adj)
            adj.append([])
            adj[1].append(x)
            fill = []
            for _ in range(k):
                f = len(adj)
                adj.append([x])
                fill.append(f)
            tail = []
            for _ in range(t):
                f = len(adj)
                adj.append([x])
                tail.append(f)
            adj[x] = fill + [1] + tail
    off = np.zeros(len(adj) + 1, np.uint32)
    off[1:] = np.cumsum([len(a) for a in adj])
    col = np.array([v for a in adj for v in a], np.uint32)
    return mg.Csr.from_csr(off, col)


@pytest.mark.parametrize("n", [1, 2])
@pytest.mark.parametrize("do_a", [1e-9, 0.01])
def test_dobfs_pull_first_hit_positions(n, do_a):
    """W (the first-hit scan count) and labels equal the reference's for first
    hits at every arc position across the pull's three stages"""
    g = _first_hit_graph()
    off, col, _ = g.arrays()
    plan, owner = plan_for(g, n, seed=5)
    for exact in (False, True):
        cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                              dobfs_exact_cost=exact)
        r = mg.dobfs(plan, mg.DobfsOptions(source=0, do_a=do_a, do_b=0.1, mark_preds=True), cfg)
        assert np.array_equal(r.labels, seq.bfs_levels(off, col, 0))
        x = np.nonzero(r.labels == 2)[0]
        assert np.all(r.preds[x] == 1) and len(x) == 4 * len(FIRST_HIT_POS)
        if do_a < 1e-6:
            assert r.backward_edges > 0  # the rows were pulled
        if ref.available():
            rr = ref.RefPlan(ref.RefGraph.from_csr(off, col), owner, n).dobfs(0, do_a, 0.1)
            assert list(r.direction_log) == list(rr.direction_log)
            assert r.stats.edges_examined == rr.stats.edges_examined
            assert r.stats.supersteps == rr.stats.supersteps


def _two_components():
    """RMAT-10 on [0, 1024), RMAT-9 shifted to [1024, 1536), plus 64 isolated
    vertices at the end: sources in different components reach disjoint sets"""
    def edges(g, shift):
        off, col, _ = g.arrays()
        src = np.repeat(np.arange(len(off) - 1), np.diff(off))
        return np.stack([src + shift, col.astype(np.int64) + shift], axis=1)
    e = np.concatenate([edges(mg.Csr.rmat(10, 8, 3), 0), edges(mg.Csr.rmat(9, 8, 5), 1024)])
    g = mg.Csr.from_edges(1536 + 64, e)
    return g, g.arrays()


@pytest.mark.parametrize("n,loop", [(1, "graph"), (1, "host"), (2, "host"), (3, "host")])
def test_dobfs_labels_across_runs_without_fill(n, loop):
    """a DOBFS run that follows a completed DOBFS run skips the |V| label
    fill and resets only what the previous run reached and this one did not:
    labels stay exact across sources in different components, an isolated
    source, a max_supersteps cut and interleaved runs of other primitives
    (which clear the reuse)"""
    import os
    g, (off, col, _) = _two_components()
    plan = mg.PartitionPlan(g, mg.partition_random(g.num_vertices, n, 3) if n > 1 else None, n)
    comp_a = int(np.nonzero(np.diff(off)[:1024])[0][0])
    comp_b = 1024 + int(np.nonzero(np.diff(off)[1024:1536])[0][0])
    iso = 1536 + 5
    cut = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                          dobfs_exact_cost=True, max_supersteps=2)
    if loop == "host":
        os.environ["MG_NO_GRAPH"] = "1"
    try:
        for src, cfg, other in ((comp_a, GRAPH_CFG, None), (comp_b, GRAPH_CFG, None),
                                (iso, GRAPH_CFG, None), (comp_a, GRAPH_CFG, "bc"),
                                (comp_a, cut, None), (comp_b, GRAPH_CFG, None),
                                (comp_b, GRAPH_CFG, "bfs"), (comp_a, None, None)):
            if other == "bc":
                mg.bc(plan, comp_b)
            elif other == "bfs":
                mg.bfs(plan, mg.BfsOptions(source=comp_a))
            r = mg.dobfs(plan, mg.DobfsOptions(source=src), cfg)
            want = seq.bfs_levels(off, col, src)
            if cfg is cut:
                want = np.where(want <= 2, want, mg.kInfLabel).astype(want.dtype)
            assert np.array_equal(r.labels, want), (src, other)
    finally:
        os.environ.pop("MG_NO_GRAPH", None)
