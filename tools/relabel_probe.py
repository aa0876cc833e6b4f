"""Probe: does a vertex relabelling that packs the probed vertices into fewer
L2 sectors speed up SSSP / BC on RMAT-24?  Builds relabelled copies of the
C3/C5 graph in torch on the GPU, runs the primitives on each, checks the
results map back to the original IDs, prints device times.

    python tools/relabel_probe.py [--scale 24] [--orders deg,bfs]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1504_04804_b200 as mg  # noqa: E402

MAXCFG = mg.EngineConfig(policy=mg.AllocPolicyKind.Maximum, fused=mg.FusedMode.On)


def relabel(off, col, w, perm, dev="cuda"):
    """perm[i] = old vertex at new position i -> (off2, col2, w2) on the host"""
    off_t = torch.from_numpy(off.astype(np.int64)).to(dev)
    perm_t = torch.from_numpy(perm.astype(np.int64)).to(dev)
    nv = len(perm)
    iperm = torch.empty(nv, dtype=torch.int64, device=dev)
    iperm[perm_t] = torch.arange(nv, device=dev)
    deg = off_t[1:] - off_t[:-1]
    ndeg = deg[perm_t]
    noff = torch.zeros(nv + 1, dtype=torch.int64, device=dev)
    noff[1:] = torch.cumsum(ndeg, 0)
    ne = int(noff[-1])
    shift = off_t[:-1][perm_t] - noff[:-1]
    src = torch.repeat_interleave(shift, ndeg, output_size=ne)
    old_arc = src + torch.arange(ne, device=dev)
    del src
    col_t = torch.from_numpy(col.view(np.int32)).to(dev)
    ncol = iperm[col_t[old_arc].long()].to(torch.int32)
    del col_t
    nw = None
    if w is not None:
        w_t = torch.from_numpy(w.view(np.int32)).to(dev)
        nw = w_t[old_arc].cpu().numpy().view(np.uint32)
        del w_t
    out = (noff.cpu().numpy().astype(np.uint32), ncol.cpu().numpy().view(np.uint32), nw,
           iperm.cpu().numpy())
    del old_arc, ncol
    torch.cuda.empty_cache()
    return out


def timeit(fn, reps):
    fn()
    ms = [fn() for _ in range(reps)]
    return float(np.mean(ms)), float(np.min(ms))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--orders", default="deg,bfs,deghub")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    plan = mg.PartitionPlan.rmat_device(a.scale, 16, 1, weights=(1, 64, 102))
    g = plan.download_graph()
    off, col, w = g.arrays()
    nv = len(off) - 1
    deg = np.diff(off.astype(np.int64))
    r0 = mg.sssp(plan, 0, cfg=MAXCFG)
    b0 = mg.bc(plan, 0, cfg=MAXCFG)
    base = dict(order="identity",
                sssp=timeit(lambda: mg.sssp(plan, 0, cfg=MAXCFG, download=False).stats.device_ms,
                            a.reps),
                bc=timeit(lambda: mg.bc(plan, 0, cfg=MAXCFG, download=False).stats.device_ms,
                          a.reps))
    print(json.dumps(base), flush=True)
    del plan
    for name in a.orders.split(","):
        if name == "deg":  # degree descending, ties by ID
            perm = np.lexsort((np.arange(nv), -deg))
        elif name == "deghub":  # rows of degree >= 64 first (by degree), the rest in ID order
            hub = deg >= 64
            hp = np.nonzero(hub)[0]
            hp = hp[np.argsort(-deg[hp], kind="stable")]
            perm = np.concatenate([hp, np.nonzero(~hub)[0]])
        elif name == "bfs":  # the library's FIFO-BFS locality order from the hub
            import scipy.sparse as sp
            from scipy.sparse.csgraph import breadth_first_order
            m = sp.csr_matrix((np.ones(len(col), np.int8), col, off), shape=(nv, nv))
            start = int(np.argmax(deg))
            o = breadth_first_order(m, start, directed=True, return_predecessors=False)
            seen = np.zeros(nv, bool)
            seen[o] = True
            perm = np.concatenate([o, np.nonzero(~seen)[0]])
            del m
        else:
            raise SystemExit(name)
        off2, col2, w2, iperm = relabel(off, col, w, perm)
        g2 = mg.Csr.from_csr(off2, col2, w2)
        p2 = mg.PartitionPlan(g2, None, 1, devices=[0])
        s = int(iperm[0])
        r = mg.sssp(p2, s, cfg=MAXCFG)
        ok_s = bool(np.array_equal(r.dists[iperm], r0.dists))
        b = mg.bc(p2, s, cfg=MAXCFG)
        ok_b = bool(np.array_equal(b.sigma[iperm], b0.sigma))
        out = dict(order=name, sssp_ok=ok_s, bc_sigma_ok=ok_b,
                   S=int(r.stats.supersteps), S0=int(r0.stats.supersteps),
                   W=int(r.stats.edges_examined), W0=int(r0.stats.edges_examined),
                   sssp=timeit(lambda: mg.sssp(p2, s, cfg=MAXCFG, download=False).stats.device_ms,
                               a.reps),
                   bc=timeit(lambda: mg.bc(p2, s, cfg=MAXCFG, download=False).stats.device_ms,
                             a.reps))
        print(json.dumps(out), flush=True)
        del p2, g2, r, b


if __name__ == "__main__":
    main()
