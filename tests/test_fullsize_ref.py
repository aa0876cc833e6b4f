"""Full-size parity against the reference itself (GPU): the BASELINE.json
configurations at their own sizes, run by the UNMODIFIED reference engine
(oracle/_ref, compiled from /root/reference/proj/core/src) on the same CSR,
owner map and sources, and compared with the sm_100a path — at one partition
and at n = 2/4/8 partitions hosted on one GPU.

  C2  DOBFS RMAT-26/16, partition_random(|V|, n, 7), sources 0 and 4301304:
      labels bit-exact; direction log, S and W (first-hit scan count, the
      reference's accounting, primitives.cpp:227-252) equal; under the
      reference schedule H equals the reference's H matrix.
  C3  SSSP RMAT-24/16 w in [1,64] (assign_random_weights seed 102), the
      border-minimising partition_biased_random(g, n, 7, 1.0), source 0:
      distances bit-exact vs the reference engine and vs Dijkstra
      (reference.cpp:63-90); S and the H matrix equal.
  C5  BC RMAT-24/16, partition_random(|V|, n, 7), source 0: sigma and labels
      bit-exact, bc within 1e-5 relative (tools/mgraph.cpp:478-489), S and H
      equal.
  C4  RGG n = 2^24: CC bit-exact (S, H equal at n = 8) and PageRank
      (d = 0.85, eps = 1e-6) with the reference's iteration count and ranks
      within 1e-6 per vertex at n = 1 and n = 8.

Both sides get the graph from their own builder (device gen.cu for the
product, gen_oracle.cpp for the reference); the first test checks they are
the same bytes.  The reference runs n worker threads (engine.hpp:951-959).
"""
import gc

import numpy as np
import pytest

import paper_1504_04804_b200 as mg
from oracle import ref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]

MAXCFG = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On)
EXACT = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                        dobfs_exact_cost=True)
C2_SOURCES = (0, 4301304)


def owner_random(nv, n):
    return ref.partition_random(nv, n, 7) if n > 1 else np.zeros(nv, np.uint32)


def rel_close(a, b, tol):
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-12)
    return bool(np.all(np.abs(a - b) / scale <= tol))


# --------------------------------------------------------------------------- C2
@pytest.fixture(scope="module")
def rmat26():
    g = ref.RefGraph.rmat_hashed(26, 16, 1)
    yield g
    del g
    gc.collect()


def test_c2_device_rmat26_is_the_reference_side_graph(rmat26):
    plan = mg.PartitionPlan.rmat_device(26, 16, 1)
    a = plan.download_graph()
    del plan
    off_a, col_a, _ = a.arrays()
    del a
    nv, ne, _ = rmat26.info()
    assert (nv, ne) == (len(off_a) - 1, len(col_a))
    off_b, col_b, _ = rmat26.arrays()
    assert np.array_equal(off_a, off_b)
    assert np.array_equal(col_a, col_b)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_c2_dobfs_rmat26_equals_reference_engine(rmat26, n):
    nv = rmat26.info()[0]
    owner = owner_random(nv, n)
    rp = ref.RefPlan(rmat26, owner, n)
    plan = mg.PartitionPlan.rmat_device(26, 16, 1, owner=owner if n > 1 else None, n=n)
    for src in C2_SOURCES:
        w = rp.dobfs(src)
        for cfg in (EXACT, MAXCFG):
            r = mg.dobfs(plan, mg.DobfsOptions(source=src), cfg)
            assert np.array_equal(r.labels, w.labels), f"labels differ (src {src})"
            assert list(r.direction_log) == list(w.direction_log)
            assert r.stats.supersteps == w.stats.supersteps
            assert r.stats.edges_examined == w.stats.edges_examined
            if cfg is MAXCFG:
                assert r.forward_edges == w.forward_edges
                assert r.backward_edges == w.backward_edges
                assert np.array_equal(r.stats.h_matrix, w.h_matrix)
            else:  # pulls in place of heavy pushes can only ship less
                assert r.stats.h_total() <= int(w.h_matrix.sum())
    del rp, plan
    gc.collect()


# --------------------------------------------------------------------------- C3 / C5
@pytest.fixture(scope="module")
def rmat24w():
    g = ref.RefGraph.rmat_hashed(24, 16, 1).weighted(1, 64, 102)
    yield g, g.seq_dijkstra(0)
    del g
    gc.collect()


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_c3_sssp_rmat24_biased_partition_equals_reference_engine(rmat24w, n):
    g, dijkstra = rmat24w
    owner = ref.partition_biased(g, n, 7, 1.0) if n > 1 else np.zeros(g.info()[0], np.uint32)
    rp = ref.RefPlan(g, owner, n)
    w = rp.sssp(0)
    del rp
    plan = mg.PartitionPlan.rmat_device(24, 16, 1, owner=owner if n > 1 else None, n=n,
                                        weights=(1, 64, 102))
    r = mg.sssp(plan, 0, False, MAXCFG)
    assert np.array_equal(w.dists, dijkstra)
    assert np.array_equal(r.dists, dijkstra)
    assert r.stats.supersteps == w.stats.supersteps
    assert np.array_equal(r.stats.h_matrix, w.h_matrix)
    del plan
    gc.collect()


@pytest.fixture(scope="module")
def rmat24():
    g = ref.RefGraph.rmat_hashed(24, 16, 1)
    yield g
    del g
    gc.collect()


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_c5_bc_rmat24_equals_reference_engine(rmat24, n):
    owner = owner_random(rmat24.info()[0], n)
    rp = ref.RefPlan(rmat24, owner, n)
    w = rp.bc(0)
    del rp
    plan = mg.PartitionPlan.rmat_device(24, 16, 1, owner=owner if n > 1 else None, n=n)
    r = mg.bc(plan, 0, MAXCFG)
    assert np.array_equal(r.labels, w.labels)
    assert np.array_equal(r.sigma, w.sigma)
    assert rel_close(r.bc, w.bc, 1e-5)
    assert r.stats.supersteps == w.stats.supersteps
    assert np.array_equal(r.stats.h_matrix, w.h_matrix)
    del plan
    gc.collect()


# --------------------------------------------------------------------------- C4
@pytest.fixture(scope="module")
def rgg24():
    plan = mg.PartitionPlan.rgg_device(1 << 24, 1)
    off, col, _ = plan.download_graph().arrays()
    del plan
    g = ref.RefGraph.from_csr(off, col)
    del off, col
    owner8 = ref.partition_random(1 << 24, 8, 7)
    rp = ref.RefPlan(g, owner8, 8)
    cc8 = rp.cc()
    pr8 = rp.pagerank(0.85, 1e-6, 1000)
    del rp
    gc.collect()
    yield g, owner8, cc8, pr8
    del g
    gc.collect()


@pytest.mark.parametrize("n", [1, 8])
def test_c4_cc_rgg24_equals_reference_engine(rgg24, n):
    _, owner8, w, _ = rgg24
    plan = mg.PartitionPlan.rgg_device(1 << 24, 1, owner=owner8 if n == 8 else None, n=n)
    r = mg.cc(plan, MAXCFG)
    assert np.array_equal(r.components, w.components)
    if n == 8:
        assert r.stats.supersteps == w.stats.supersteps
        assert np.array_equal(r.stats.h_matrix, w.h_matrix)


@pytest.mark.parametrize("n", [1, 8])
def test_c4_pagerank_rgg24_equals_reference_engine(rgg24, n):
    _, owner8, _, w = rgg24
    plan = mg.PartitionPlan.rgg_device(1 << 24, 1, owner=owner8 if n == 8 else None, n=n)
    r = mg.pagerank(plan, mg.PrOptions(damping=0.85, epsilon=1e-6, max_iter=1000), MAXCFG)
    assert r.iterations == w.iterations
    assert float(np.max(np.abs(r.ranks - w.ranks))) <= 1e-6
    if n == 8:
        assert r.stats.supersteps == w.stats.supersteps
        assert np.array_equal(r.stats.h_matrix, w.h_matrix)
