"""Dense DOBFS push supersteps (DobfsDev::red): fire-and-forget visited-bit ORs,
labels and the output frontier taken afterwards from vis & ~prev.

The thresholds (MG_DOBFS_DENSE_ARCS host loop, MG_DOBFS_LOOP_DENSE_ARCS
device-driven loop) are read once
per process, so the forced cases run
in a child process with every push dense; the parent checks the default
thresholds.  Labels must equal the oracle's BFS levels; direction log, S, W and
the per-superstep frontier sizes must equal the reference engine's
(oracle/_ref, primitives.cpp:197-253) and the non-dense run's.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1504_04804_b200 as mg
from oracle import ref, seq

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

HOST_CFG = dict(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                dobfs_exact_cost=False)
LOOP_CFG = dict(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On,
                dobfs_exact_cost=True)

CASES = [("rmat", 12, 16, 1), ("rmat", 14, 16, 3), ("rmat", 12, 32, 6), ("grid", 48, 48, 0)]


def _graph(kind, a, b, seed):
    return mg.Csr.rmat(a, b, seed) if kind == "rmat" else mg.Csr.grid(a, b)


def _runs():
    """every case x source x do_a x loop: labels digest and schedule"""
    out = []
    for kind, a, b, seed in CASES:
        g = _graph(kind, a, b, seed)
        off, col, _ = g.arrays()
        plan = mg.PartitionPlan(g, None, 1)
        for src in (0, 5, 301):
            for do_a in (0.01, 0.001):
                for name, cfg in (("host", HOST_CFG), ("loop", LOOP_CFG)):
                    r = mg.dobfs(plan, mg.DobfsOptions(source=src, do_a=do_a),
                                 mg.EngineConfig(**cfg))
                    ok = bool(np.array_equal(r.labels, seq.bfs_levels(off, col, src)))
                    out.append({"case": [kind, a, b, seed], "src": src, "do_a": do_a,
                                "loop": name, "labels_ok": ok,
                                "dir": [int(x) for x in r.direction_log],
                                "S": int(r.stats.supersteps), "W": int(r.stats.edges_examined),
                                "out": [int(x) for x in r.stats.out_per_iter],
                                "device_loop": int(r.stats.device_loop)})
    return out


def _child(env):
    code = ("import json, sys; sys.path.insert(0, %r); sys.path.insert(0, %r); "
            "import test_dense_push as t; print(json.dumps(t._runs()))"
            % (ROOT, os.path.join(ROOT, "tests")))
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       env={**os.environ, **env}, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def forced():
    return _child({"MG_DOBFS_DENSE_ARCS": "1", "MG_DOBFS_LOOP_DENSE_ARCS": "1"})


@pytest.fixture(scope="module")
def never():
    return _child({"MG_DOBFS_DENSE_ARCS": "0", "MG_DOBFS_LOOP_DENSE_ARCS": "0"})


def test_dense_push_labels_exact(forced):
    assert all(r["labels_ok"] for r in forced)
    # the device-driven loop ran (so its dense branch was exercised)
    assert any(r["device_loop"] for r in forced if r["loop"] == "loop")


def test_dense_push_schedule_equals_atomic_push(forced, never):
    assert len(forced) == len(never)
    for a, b in zip(forced, never):
        assert b["labels_ok"]
        for k in ("dir", "S", "W", "out"):
            assert a[k] == b[k], (a["case"], a["src"], a["loop"], k)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_dense_push_matches_reference_engine(forced):
    graphs, bad = {}, []
    for r in forced:
        if r["loop"] != "host":
            continue
        key = tuple(r["case"])
        if key not in graphs:
            off, col, _ = _graph(*key).arrays()
            owner = np.zeros(len(off) - 1, np.uint32)
            graphs[key] = ref.RefPlan(ref.RefGraph.from_csr(off, col), owner, 1)
        rr = graphs[key].dobfs(r["src"], r["do_a"], 0.1)
        want = ([int(x) for x in rr.direction_log], int(rr.stats.supersteps),
                int(rr.stats.edges_examined))
        got = (r["dir"], r["S"], r["W"])
        if got != want:
            bad.append((key, r["src"], r["do_a"], got, want))
    assert not bad, bad[:3]


def test_dense_push_default_thresholds_rmat16():
    """in-process defaults: RMAT-16 pushes cross both thresholds"""
    g = mg.Csr.rmat(16, 16, 2)
    off, col, _ = g.arrays()
    plan = mg.PartitionPlan(g, None, 1)
    for cfg in (HOST_CFG, LOOP_CFG):
        for src in (0, 11):
            r = mg.dobfs(plan, mg.DobfsOptions(source=src), mg.EngineConfig(**cfg))
            assert np.array_equal(r.labels, seq.bfs_levels(off, col, src))


def test_dense_bfs_push_rmat22():
    """single-partition BFS with the visited bitmap (|V| >= 2^22): its big
    pushes run dense at the default threshold; labels equal the oracle's and
    S, W and the per-superstep frontier sizes the reference engine's"""
    plan = mg.PartitionPlan.rmat_device(22, 16, 1)
    off, col, _ = plan.download_graph().arrays()
    cfg = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On)
    rp = None
    if ref.available():
        rp = ref.RefPlan(ref.RefGraph.from_csr(off, col), np.zeros(len(off) - 1, np.uint32), 1)
    for src in (0, 1000):
        r = mg.bfs(plan, mg.BfsOptions(source=src), cfg)
        assert np.array_equal(r.labels, seq.bfs_levels(off, col, src))
        assert r.stats.edges_examined > (1 << 20)  # a dense superstep ran
        if rp is not None:
            rr = rp.bfs(src)
            assert r.stats.supersteps == rr.stats.supersteps
            assert r.stats.edges_examined == rr.stats.edges_examined
            assert list(r.stats.out_per_iter) == list(rr.out_per_iter)
