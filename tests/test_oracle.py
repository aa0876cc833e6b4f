"""Pin the oracle before trusting it (CPU only).

* the plain-C restatement (oracle/seq_oracle.c) against the golden vectors the
  reference's own unit tests hold (tests/golden/reference_pins.json), and
* against the unmodified reference compiled into oracle/_ref — bit-exact,
  floating point included (the restatement keeps the evaluation order).
"""
import numpy as np
import pytest

from oracle import ref, seq


def test_restatement_matches_golden_vectors(golden):
    pins, vec = golden
    off, col = vec["rmat12_off"], vec["rmat12_col"]
    assert np.array_equal(seq.bfs_levels(off, col, 0), vec["rmat12_bfs0"])
    assert np.array_equal(seq.connected_components(off, col), vec["rmat12_cc"])
    assert np.array_equal(seq.dijkstra(off, col, vec["rmat12_w"], 0), vec["rmat12_dijkstra0"])
    bc, sigma, labels = seq.brandes_bc(vec["rmat10_off"], vec["rmat10_col"], 1)
    assert np.array_equal(bc, vec["rmat10_bc1"])  # bit-exact: same evaluation order
    ranks, it, sums = seq.pagerank_power(vec["rmat10s21_off"], vec["rmat10s21_col"], 0.85, 1e-4,
                                         1000)
    assert it == int(vec["rmat10s21_pr_iters"])
    assert np.array_equal(ranks, vec["rmat10s21_pr"])
    assert np.array_equal(sums, vec["rmat10s21_pr_sums"])


def test_restatement_hand_pins(golden):
    pins, _ = golden
    # P4 path 0-1-2-3
    off = np.array([0, 1, 3, 5, 6], np.uint32)
    col = np.array([1, 0, 2, 1, 3, 2], np.uint32)
    assert list(seq.bfs_levels(off, col, 0)) == pins["bfs_p4_two_way"]["labels"]
    bc, _, _ = seq.brandes_bc(off, col, 0)
    assert list(bc) == pins["bc_p4"]["bc"]
    # weighted P4 (weights 2,3,1 mirrored)
    w = np.array([2, 2, 3, 3, 1, 1], np.uint32)
    assert list(seq.dijkstra(off, col, w, 0)) == pins["sssp_p4_weighted"]["dists"]
    # triangle + isolated
    toff = np.array([0, 2, 4, 6, 6], np.uint32)
    tcol = np.array([1, 2, 0, 2, 0, 1], np.uint32)
    assert list(seq.connected_components(toff, tcol)) == pins["cc_triangle_isolated"]["components"]
    eoff = np.zeros(6, np.uint32)
    assert list(seq.connected_components(eoff, np.zeros(0, np.uint32))) == \
        pins["cc_edgeless"]["components"]
    # star from a leaf
    soff = np.array([0, 4, 5, 6, 7, 8], np.uint32)
    scol = np.array([1, 2, 3, 4, 0, 0, 0, 0], np.uint32)
    bc, _, _ = seq.brandes_bc(soff, scol, 1)
    assert bc[0] == pins["bc_star5_leaf"]["bc_center"]
    ranks, it, _ = seq.pagerank_power(np.zeros(2, np.uint32), np.zeros(0, np.uint32), 0.85, 0.01,
                                      1000)
    assert abs(ranks[0] - 1.0) <= 1e-12


def test_direction_rule_table(golden):
    pins, _ = golden
    for cur, fv, bv, a, b, sw, expect in pins["direction_rule_table"]["cases"]:
        assert seq.direction_decide(cur, fv, bv, a, b, sw) == expect
        if ref.available():
            assert ref.lib().ref_direction_decide(cur, fv, bv, a, b, sw) == expect
    e = pins["direction_estimates"]
    fv, bv = seq.direction_estimates(*e["args"])
    assert fv == pytest.approx(e["fv"]) and bv == pytest.approx(e["bv"])


needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("scale,ef,seed", [(9, 8, 4), (11, 16, 3), (12, 32, 6)])
def test_restatement_equals_reference(scale, ef, seed):
    g = ref.RefGraph.rmat(scale, ef, seed)
    off, col, _ = g.arrays()
    for s in (0, 5):
        assert np.array_equal(seq.bfs_levels(off, col, s), g.seq_bfs(s))
        assert np.array_equal(seq.brandes_bc(off, col, s)[0], g.seq_bc(s))
    assert np.array_equal(seq.connected_components(off, col), g.seq_cc())
    gw = g.weighted(1, 64, seed + 101)
    assert np.array_equal(seq.dijkstra(off, col, gw.arrays()[2], 0), gw.seq_dijkstra(0))
    r1 = seq.pagerank_power(off, col, 0.85, 1e-6, 1000)
    r2 = g.seq_pagerank(0.85, 1e-6, 1000)
    assert r1[1] == r2[1] and np.array_equal(r1[0], r2[0])


@needs_ref
def test_reference_engine_agrees_with_restatement_and_pins(golden):
    pins, vec = golden
    p = ref.RefGraph.path(4)
    plan = ref.RefPlan(p, np.array([0, 0, 1, 1], np.uint32), 2)
    r = plan.bfs(0)
    pin = pins["bfs_p4_two_way"]
    assert list(r.labels) == pin["labels"]
    assert r.stats.supersteps == pin["supersteps"] and r.stats.h_total == pin["h_total"]
    assert r.h_matrix.tolist() == pin["h_matrix"] and r.stats.combine_ops == pin["combine_ops"]
    g = ref.RefGraph.from_csr(vec["rmat12_off"], vec["rmat12_col"])
    plan = ref.RefPlan(g, vec["rmat12_n4_owner"], 4)
    r = plan.bfs(0)
    assert np.array_equal(r.labels, vec["rmat12_n4_bfs_labels"])
    assert r.stats.supersteps == int(vec["rmat12_n4_bfs_S"])
    assert np.array_equal(r.h_matrix, vec["rmat12_n4_bfs_H"])
