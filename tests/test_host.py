"""Host logic (CPU only): the kept graph preparation and partitioners produce
the reference's bytes, and the C-ABI library exports what include/ declares."""
import os
import re

import numpy as np
import pytest

import paper_1504_04804_b200 as mg
from paper_1504_04804_b200 import abi
from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "mgraph_b200.h")).read()
    declared = set(re.findall(r"^(?:[\w\s\*]+?)\b(mg_\w+)\(", hdr, re.M))
    assert len(declared) >= 35
    L = mg.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert declared == set(abi.PROTOTYPES), declared ^ set(abi.PROTOTYPES)


def test_config_defaults_match_reference():
    c = abi.mg_config()
    mg.lib().mg_config_default(c)
    assert c.policy == abi.MG_POLICY_JUST and c.h_inflation == 1
    assert c.max_supersteps == 1000000 and c.comm_override == -1  # engine.hpp:308-315


@needs_ref
@pytest.mark.parametrize("scale,ef,seed", [(4, 4, 3), (9, 8, 4), (12, 16, 1), (12, 32, 6)])
def test_rmat_build_symmetrize_bit_identical(scale, ef, seed):
    a = mg.Csr.rmat(scale, ef, seed).arrays()
    b = ref.RefGraph.rmat(scale, ef, seed).arrays()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    raw_a = mg.Csr.rmat(scale, ef, seed, symmetrize=False).arrays()
    raw_b = ref.RefGraph.rmat(scale, ef, seed, symmetrize=False).arrays()
    assert np.array_equal(raw_a[0], raw_b[0]) and np.array_equal(raw_a[1], raw_b[1])


def test_rmat18_matches_golden_digest(golden):
    """config 1 graph (RMAT-18/16 seed 1): |V|, |A| and a checksum of the CSR"""
    _, vec = golden
    off, col, _ = mg.Csr.rmat(18, 16, 1).arrays()
    assert [len(off) - 1, len(col)] == list(vec["rmat18_nv_ne"])
    d = [int(off.astype(np.uint64).sum()),
         int((col.astype(np.uint64) * 2654435761 % (1 << 61)).sum())]
    assert d == list(vec["rmat18_off_digest"])
    assert len(col) == 7610830


@needs_ref
def test_weights_grid_path_bit_identical():
    g = mg.Csr.rmat(10, 8, 5)
    rg = ref.RefGraph.rmat(10, 8, 5)
    for lo, hi, seed in [(0, 64, 6), (1, 64, 106), (1, 1, 0)]:
        assert np.array_equal(g.with_weights(lo, hi, seed).arrays()[2],
                              rg.weighted(lo, hi, seed).arrays()[2])
    for (r, c) in [(1, 1), (3, 5), (32, 32)]:
        a, b = mg.Csr.grid(r, c).arrays(), ref.RefGraph.grid(r, c).arrays()
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    a, b = mg.Csr.path(4).arrays(), ref.RefGraph.path(4).arrays()
    assert np.array_equal(a[1], b[1])


@needs_ref
def test_build_csr_and_symmetrize_with_weights():
    rng = np.random.default_rng(3)
    e = np.stack([rng.integers(0, 50, 400), rng.integers(0, 50, 400),
                  rng.integers(0, 9, 400)], 1)
    a = mg.Csr.from_edges(50, e, weighted=True)
    b = ref.RefGraph.from_edges(50, e[:, 0], e[:, 1], e[:, 2])
    for x, y in zip(a.arrays(), b.arrays()):
        assert np.array_equal(x, y)
    for x, y in zip(a.symmetrize_dedup().arrays(), b.symmetrize().arrays()):
        assert np.array_equal(x, y)  # min weight kept on conflicts (csr.cpp:82-108)


@needs_ref
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_partitioners_bit_identical(n):
    g = mg.Csr.rmat(11, 8, 2)
    rg = ref.RefGraph.rmat(11, 8, 2)
    for seed in (0, 7, 99):
        assert np.array_equal(mg.partition_random(g.num_vertices, n, seed),
                              ref.partition_random(g.num_vertices, n, seed))
        for bias in (0.0, 0.5, 1.0):
            assert np.array_equal(mg.partition_biased_random(g, n, seed, bias),
                                  ref.partition_biased(rg, n, seed, bias))


def test_error_behaviour_without_gpu_is_loud():
    with pytest.raises(ValueError):
        mg.partition_random(10, 0, 1)  # partition.cpp:32
    with pytest.raises(ValueError):
        mg.partition_biased_random(mg.Csr.path(4), 2, 1, 1.5)
    with pytest.raises(ValueError):
        mg.Csr.from_edges(3, [[0, 5]])  # build_csr range check


def test_hashed_rmat_host_generator_is_symmetric_and_deduped():
    off, col, _ = mg.Csr.rmat_hashed(10, 16, 5).arrays()
    nv = len(off) - 1
    src = np.repeat(np.arange(nv), np.diff(off.astype(np.int64)))
    assert np.all(src != col)  # no self-loops
    fwd = set(zip(src.tolist(), col.tolist()))
    assert len(fwd) == len(col)  # no duplicates
    assert all((v, u) in fwd for u, v in list(fwd)[:2000])  # mirrored
    # rows sorted
    for u in range(0, nv, 37):
        row = col[off[u]:off[u + 1]]
        assert np.all(row[:-1] < row[1:])
