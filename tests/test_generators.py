"""Graph preparation pinned to the reference.

f1  the counter-based R-MAT CSR — the product's host twin (host_graph.cpp),
    its device builder (gen.cu) and the oracle's own builder (gen_oracle.cpp,
    used by bench.py's reference arm) — equals the reference's build_csr +
    symmetrize_dedup (csr.cpp:27-108) run on the same raw edge draws; the hash
    weights equal assign_random_weights (generate.cpp:64-79) on the same CSR.
f2  the device Duplicate-All extraction gives the border counts and edge cut
    of the reference's build_partition_plan / border_metrics
    (partition.cpp:121-242), for random and border-minimising assignments.
f3  the device random-geometric graph is exactly {(i, j): i != j,
    |p_i - p_j|^2 < r^2}, r = 0.55 sqrt(ln n / n), with
    the points restated here from their definition (mix64 counter draws).
"""
import numpy as np
import pytest

import paper_1504_04804_b200 as mg
from oracle import ref

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def csr_equal(a, b):
    return np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# --------------------------------------------------------------------------- f1 (CPU)
@needs_ref
@pytest.mark.parametrize("scale,ef,seed", [(8, 4, 3), (12, 16, 1), (16, 16, 1), (14, 32, 9)])
def test_hashed_rmat_equals_reference_symmetrize_dedup(scale, ef, seed):
    src, dst = ref.rmat_hashed_edges(scale, ef, seed)
    assert len(src) == (1 << scale) * ef
    want = ref.RefGraph.from_edges(1 << scale, src, dst).symmetrize().arrays()
    host_twin = mg.Csr.rmat_hashed(scale, ef, seed).arrays()
    oracle_builder = ref.RefGraph.rmat_hashed(scale, ef, seed).arrays()
    assert csr_equal(host_twin, want), "host twin != reference symmetrize_dedup"
    assert csr_equal(oracle_builder, want), "oracle builder != reference symmetrize_dedup"


@needs_ref
def test_hashed_rmat_weights_equal_reference_assign_random_weights():
    g = mg.Csr.rmat_hashed(14, 16, 1)
    rg = ref.RefGraph.rmat_hashed(14, 16, 1)
    for lo, hi, seed in [(1, 64, 102), (0, 7, 5)]:
        a = g.with_weights(lo, hi, seed).arrays()
        b = rg.weighted(lo, hi, seed).arrays()
        assert csr_equal(a, b) and np.array_equal(a[2], b[2])
        assert int(a[2].min()) >= lo and int(a[2].max()) <= hi


# --------------------------------------------------------------------------- f1-f3 (GPU)
@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("scale,ef,seed", [(16, 16, 1), (20, 16, 1), (18, 8, 3)])
def test_device_rmat_equals_host_twin_and_reference(scale, ef, seed):
    dev = mg.PartitionPlan.rmat_device(scale, ef, seed, weights=(1, 64, 102))
    a = dev.download_graph().arrays()
    b = mg.Csr.rmat_hashed(scale, ef, seed).with_weights(1, 64, 102).arrays()
    assert csr_equal(a, b) and np.array_equal(a[2], b[2])
    if scale <= 16:  # the reference's sequential symmetrize_dedup on the raw draws
        src, dst = ref.rmat_hashed_edges(scale, ef, seed)
        c = ref.RefGraph.from_edges(1 << scale, src, dst).symmetrize().weighted(1, 64, 102)
        c = c.arrays()
        assert csr_equal(a, c) and np.array_equal(a[2], c[2])


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("n,biased", [(2, False), (4, False), (8, False), (3, True), (8, True)])
def test_device_partition_extraction_equals_build_partition_plan(n, biased):
    scale = 16
    g = mg.Csr.rmat_hashed(scale, 16, 1)
    rg = ref.RefGraph.rmat_hashed(scale, 16, 1)
    owner = (ref.partition_biased(rg, n, 7, 1.0) if biased
             else ref.partition_random(g.num_vertices, n, 7))
    if biased:
        assert np.array_equal(owner, mg.partition_biased_random(g, n, 7, 1.0))
    dev = mg.PartitionPlan.rmat_device(scale, 16, 1, owner=owner, n=n)
    host = mg.PartitionPlan(g, owner, n)
    rp = ref.RefPlan(rg, owner, n)
    want_pair, want_cut = rp.border_metrics()
    for p in (dev, host):
        pair, cut = p.border_metrics()
        assert np.array_equal(pair, want_pair) and cut == want_cut
    # the extracted sub-graphs carry every hosted row and nothing else: results
    # on the device-extracted plan equal the reference engine's, H included
    r = mg.bfs(dev, mg.BfsOptions(source=0))
    w = rp.bfs(0)
    assert np.array_equal(r.labels, w.labels)
    assert r.stats.supersteps == w.stats.supersteps
    assert r.stats.edges_examined == w.stats.edges_examined
    assert np.array_equal(r.stats.h_matrix, w.h_matrix)


def _mix64(x):
    x = (x + np.uint64(0x9E3779B97F4A7C15))
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def rgg_points(n, seed):
    """gen.cu rgg_coord: x_i = mix64(mix64(seed) + 2i) >> 11 / 2^53, y_i from 2i+1"""
    with np.errstate(over="ignore"):
        sm = _mix64(np.array([seed], np.uint64))[0]
        k = np.arange(2 * n, dtype=np.uint64) + sm
        u = (_mix64(k) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return u[0::2], u[1::2]


@pytest.mark.gpu
@pytest.mark.parametrize("n,seed", [(1 << 14, 1), (50000, 3), (1 << 18, 1)])
def test_rgg_edge_iff_distance_below_radius(n, seed):
    from scipy.spatial import cKDTree
    plan = mg.PartitionPlan.rgg_device(n, seed)
    off, col, _ = plan.download_graph().arrays()
    x, y = rgg_points(n, seed)
    r = 0.55 * np.sqrt(np.log(n) / n)
    # candidates with a little slack, then the exact double test of the generator
    pairs = cKDTree(np.stack([x, y], 1)).query_pairs(r * (1 + 1e-9), output_type="ndarray")
    i, j = pairs[:, 0], pairs[:, 1]
    dx, dy = x[j] - x[i], y[j] - y[i]
    keep = dx * dx + dy * dy < r * r
    i, j = i[keep], j[keep]
    want = np.unique(np.concatenate([i.astype(np.int64) << 32 | j, j.astype(np.int64) << 32 | i]))
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(off.astype(np.int64)))
    got = rows << 32 | col.astype(np.int64)
    assert np.all(np.diff(got) > 0), "rows not sorted / duplicate arcs"
    assert np.array_equal(got, want)
    # mean degree pi r^2 n = 0.9503 ln n up to boundary loss
    assert 0.8 * 0.9503 * np.log(n) < len(col) / n < 1.0 * 0.9503 * np.log(n)
