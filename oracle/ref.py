"""ctypes binding of the unmodified reference (oracle/_ref/libmgraph_ref.so). TEST-ONLY.

The shared object is compiled from /root/reference/proj/core/src by
oracle/Makefile in the dev container and travels to the GPU box prebuilt.
"""
import ctypes as C
import os

import numpy as np

from paper_1504_04804_b200.abi import (MG_ARR_H_MATRIX, default_config, mg_config, mg_stats)

from . import REF_DIR

_lib = None


def available():
    return os.path.exists(os.path.join(REF_DIR, "libmgraph_ref.so"))


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(REF_DIR, "libmgraph_ref.so")
        if not os.path.exists(path):
            from . import build
            build()
        L = C.CDLL(path)
        P, PP = C.c_void_p, C.POINTER(C.c_void_p)
        u32, u64, i32, dbl = C.c_uint32, C.c_uint64, C.c_int, C.c_double
        CFG, ST = C.POINTER(mg_config), C.POINTER(mg_stats)
        protos = {
            "ref_last_error": (C.c_char_p, []),
            "ref_graph_from_csr": (i32, [u32, u64, P, P, P, PP]),
            "ref_graph_from_edges": (i32, [u32, u64, P, P, P, PP]),
            "ref_graph_rmat": (i32, [i32, i32, u64, i32, PP]),
            "ref_graph_symmetrize": (i32, [P, PP]),
            "ref_graph_assign_weights": (i32, [P, u32, u32, u64, PP]),
            "ref_graph_grid": (i32, [u32, u32, PP]),
            "ref_graph_path": (i32, [u32, PP]),
            "ref_graph_info": (None, [P, C.POINTER(u32), C.POINTER(u64), C.POINTER(i32)]),
            "ref_graph_copy": (None, [P, P, P, P]),
            "ref_graph_destroy": (None, [P]),
            "ref_partition_random": (i32, [u32, u32, u64, P]),
            "ref_partition_biased": (i32, [P, u32, u64, dbl, P]),
            "ref_plan_create": (i32, [P, P, u32, i32, PP]),
            "ref_plan_destroy": (None, [P]),
            "ref_plan_border_metrics": (None, [P, P, C.POINTER(u64)]),
            "ref_plan_subgraph_info": (None, [P, u32, C.POINTER(u32), C.POINTER(u64),
                                              C.POINTER(u32)]),
            "ref_plan_subgraph_copy": (None, [P, u32, P, P, P, P]),
            "ref_bfs": (i32, [P, u32, i32, CFG, P, P, ST]),
            "ref_dobfs": (i32, [P, u32, dbl, dbl, i32, CFG, P, P, P, u64, C.POINTER(u64),
                                C.POINTER(u64), C.POINTER(u64), ST]),
            "ref_sssp": (i32, [P, u32, i32, CFG, P, P, ST]),
            "ref_cc": (i32, [P, CFG, P, ST]),
            "ref_bc": (i32, [P, u32, CFG, P, P, P, ST]),
            "ref_pagerank": (i32, [P, dbl, dbl, u64, CFG, P, C.POINTER(u64), P, u64,
                                   C.POINTER(u64), ST]),
            "ref_last_array": (u64, [i32, P, u64]),
            "ref_last_buffer_stats": (None, [u32, i32, C.POINTER(u64), C.POINTER(u64),
                                             C.POINTER(u64)]),
            "ref_direction_decide": (i32, [i32, dbl, dbl, dbl, dbl, i32]),
            "ref_seq_bfs": (None, [P, u32, P]),
            "ref_seq_dijkstra": (None, [P, u32, P]),
            "ref_seq_cc": (None, [P, P]),
            "ref_seq_bc": (None, [P, u32, P]),
            "ref_seq_pagerank": (u64, [P, dbl, dbl, u64, P, P, u64]),
            "ref_gen_last_error": (C.c_char_p, []),
            "ref_rmat_hashed_edges": (i32, [i32, i32, u64, P, P]),
            "ref_graph_rmat_hashed": (i32, [i32, i32, u64, i32, PP]),
        }
        for name, (res, args) in protos.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class RefGraph:
    """reference mgraph::Csr owned by the shim"""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_graph_destroy(self.h)
            self.h = None

    @classmethod
    def _make(cls, fn, *args):
        out = C.c_void_p()
        _check(fn(*args, C.byref(out)))
        return cls(out.value)

    @classmethod
    def rmat(cls, scale, ef, seed, symmetrize=True):
        return cls._make(lib().ref_graph_rmat, scale, ef, seed, int(symmetrize))

    @classmethod
    def rmat_hashed(cls, scale, ef, seed, threads=0):
        """counter-based R-MAT, symmetrized + deduplicated by the oracle's parallel
        builder (gen_oracle.cpp) into a reference Csr: the reference side's copy of
        the benchmark graph, made without the product library"""
        out = C.c_void_p()
        rc = lib().ref_graph_rmat_hashed(scale, ef, seed, threads, C.byref(out))
        if rc != 0:
            raise RefError(rc, lib().ref_gen_last_error().decode())
        return cls(out.value)

    @classmethod
    def from_csr(cls, off, col, w=None):
        off = np.ascontiguousarray(off, np.uint32)
        col = np.ascontiguousarray(col, np.uint32)
        w = None if w is None else np.ascontiguousarray(w, np.uint32)
        return cls._make(lib().ref_graph_from_csr, len(off) - 1, len(col), _p(off), _p(col), _p(w))

    @classmethod
    def from_edges(cls, nv, src, dst, w=None):
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        w = None if w is None else np.ascontiguousarray(w, np.uint32)
        return cls._make(lib().ref_graph_from_edges, nv, len(src), _p(src), _p(dst), _p(w))

    @classmethod
    def grid(cls, rows, cols):
        return cls._make(lib().ref_graph_grid, rows, cols)

    @classmethod
    def path(cls, n):
        return cls._make(lib().ref_graph_path, n)

    def symmetrize(self):
        return RefGraph._make(lib().ref_graph_symmetrize, self.h)

    def weighted(self, lo, hi, seed):
        return RefGraph._make(lib().ref_graph_assign_weights, self.h, lo, hi, seed)

    def info(self):
        nv, ne, w = C.c_uint32(), C.c_uint64(), C.c_int()
        lib().ref_graph_info(self.h, C.byref(nv), C.byref(ne), C.byref(w))
        return nv.value, ne.value, bool(w.value)

    def offsets(self):
        """row offsets only (no copy of the columns)"""
        nv = self.info()[0]
        off = np.empty(nv + 1, np.uint32)
        lib().ref_graph_copy(self.h, _p(off), None, None)
        return off

    def arrays(self):
        nv, ne, has_w = self.info()
        off = np.empty(nv + 1, np.uint32)
        col = np.empty(ne, np.uint32)
        w = np.empty(ne, np.uint32) if has_w else None
        lib().ref_graph_copy(self.h, _p(off), _p(col), _p(w))
        return off, col, w

    # sequential oracles (reference.cpp)
    def seq_bfs(self, src):
        out = np.empty(self.info()[0], np.uint32)
        lib().ref_seq_bfs(self.h, src, _p(out))
        return out

    def seq_dijkstra(self, src):
        out = np.empty(self.info()[0], np.uint64)
        lib().ref_seq_dijkstra(self.h, src, _p(out))
        return out

    def seq_cc(self):
        out = np.empty(self.info()[0], np.uint32)
        lib().ref_seq_cc(self.h, _p(out))
        return out

    def seq_bc(self, src):
        out = np.empty(self.info()[0], np.float64)
        lib().ref_seq_bc(self.h, src, _p(out))
        return out

    def seq_pagerank(self, d, eps, max_iter):
        nv = self.info()[0]
        ranks = np.empty(nv, np.float64)
        cap = int(min(max_iter, 1 << 20))
        sums = np.empty(max(cap, 1), np.float64)
        it = lib().ref_seq_pagerank(self.h, d, eps, max_iter, _p(ranks), _p(sums), cap)
        return ranks, int(it), sums[:it].copy()


def rmat_hashed_edges(scale, ef, seed):
    """the raw counter-based R-MAT draws (src, dst), 2^scale * ef of them"""
    m = (1 << scale) * ef
    src = np.empty(m, np.uint32)
    dst = np.empty(m, np.uint32)
    rc = lib().ref_rmat_hashed_edges(scale, ef, seed, _p(src), _p(dst))
    if rc != 0:
        raise RefError(rc, lib().ref_gen_last_error().decode())
    return src, dst


def partition_random(nv, n, seed):
    out = np.empty(nv, np.uint32)
    _check(lib().ref_partition_random(nv, n, seed, _p(out)))
    return out


def partition_biased(g, n, seed, bias):
    out = np.empty(g.info()[0], np.uint32)
    _check(lib().ref_partition_biased(g.h, n, seed, bias, _p(out)))
    return out


class RefResult:
    pass


def _cfg(cfg):
    return cfg if cfg is not None else default_config()


def _collect_stats(st, n):
    r = RefResult()
    r.stats = st
    k = lib().ref_last_array(MG_ARR_H_MATRIX, None, 0)
    hm = np.zeros(k, np.uint64)
    lib().ref_last_array(MG_ARR_H_MATRIX, _p(hm), k)
    r.h_matrix = hm.reshape(n, n) if k else np.zeros((n, n), np.uint64)
    arrs = {}
    for which in range(1, 5):
        k = lib().ref_last_array(which, None, 0)
        a = np.zeros(k, np.uint64)
        lib().ref_last_array(which, _p(a), k)
        arrs[which] = a
    r.h_per_iter = arrs[1].reshape(-1, n) if n else arrs[1]
    r.out_per_iter, r.edges_per_iter, r.combine_per_iter = arrs[2], arrs[3], arrs[4]
    r.buffers = {}
    for wk in range(n):
        for role in range(5):
            a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
            lib().ref_last_buffer_stats(wk, role, C.byref(a), C.byref(b), C.byref(c))
            r.buffers[(wk, role)] = (a.value, b.value, c.value)
    return r


class RefPlan:
    def __init__(self, g, owner, n, dup=0):
        self.g = g
        self.n = n
        self.nv = g.info()[0]
        owner = np.ascontiguousarray(owner, np.uint32)
        out = C.c_void_p()
        _check(lib().ref_plan_create(g.h, _p(owner), n, dup, C.byref(out)))
        self.h = out

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_plan_destroy(self.h)
            self.h = None

    def border_metrics(self):
        pair = np.zeros(self.n * self.n, np.uint64)
        cut = C.c_uint64()
        lib().ref_plan_border_metrics(self.h, _p(pair), C.byref(cut))
        return pair.reshape(self.n, self.n), cut.value

    def subgraph(self, p):
        nv, ne, nl = C.c_uint32(), C.c_uint64(), C.c_uint32()
        lib().ref_plan_subgraph_info(self.h, p, C.byref(nv), C.byref(ne), C.byref(nl))
        off = np.empty(nv.value + 1, np.uint32)
        col = np.empty(ne.value, np.uint32)
        w = np.empty(ne.value, np.uint32)
        l2g = np.empty(nv.value, np.uint32)
        lib().ref_plan_subgraph_copy(self.h, p, _p(off), _p(col), _p(w), _p(l2g))
        return off, col, w, l2g, nl.value

    def bfs(self, src, mark_preds=False, cfg=None):
        labels = np.empty(self.nv, np.uint32)
        preds = np.empty(self.nv, np.uint32) if mark_preds else None
        st = mg_stats()
        _check(lib().ref_bfs(self.h, src, int(mark_preds), C.byref(_cfg(cfg)), _p(labels),
                             _p(preds), C.byref(st)))
        r = _collect_stats(st, self.n)
        r.labels, r.preds = labels, preds
        return r

    def dobfs(self, src, do_a=0.01, do_b=0.1, mark_preds=False, cfg=None):
        labels = np.empty(self.nv, np.uint32)
        preds = np.empty(self.nv, np.uint32) if mark_preds else None
        dl = np.zeros(4096, np.int32)
        ln, fw, bw = C.c_uint64(), C.c_uint64(), C.c_uint64()
        st = mg_stats()
        _check(lib().ref_dobfs(self.h, src, do_a, do_b, int(mark_preds), C.byref(_cfg(cfg)),
                               _p(labels), _p(preds), _p(dl), len(dl), C.byref(ln), C.byref(fw),
                               C.byref(bw), C.byref(st)))
        r = _collect_stats(st, self.n)
        r.labels, r.preds = labels, preds
        r.direction_log = dl[:ln.value].copy()
        r.forward_edges, r.backward_edges = fw.value, bw.value
        return r

    def sssp(self, src, mark_preds=False, cfg=None):
        d = np.empty(self.nv, np.uint64)
        preds = np.empty(self.nv, np.uint32) if mark_preds else None
        st = mg_stats()
        _check(lib().ref_sssp(self.h, src, int(mark_preds), C.byref(_cfg(cfg)), _p(d),
                              _p(preds), C.byref(st)))
        r = _collect_stats(st, self.n)
        r.dists, r.preds = d, preds
        return r

    def cc(self, cfg=None):
        comp = np.empty(self.nv, np.uint32)
        st = mg_stats()
        _check(lib().ref_cc(self.h, C.byref(_cfg(cfg)), _p(comp), C.byref(st)))
        r = _collect_stats(st, self.n)
        r.components = comp
        return r

    def bc(self, src, cfg=None):
        bc = np.empty(self.nv, np.float64)
        sigma = np.empty(self.nv, np.float64)
        labels = np.empty(self.nv, np.uint32)
        st = mg_stats()
        _check(lib().ref_bc(self.h, src, C.byref(_cfg(cfg)), _p(bc), _p(sigma), _p(labels),
                            C.byref(st)))
        r = _collect_stats(st, self.n)
        r.bc, r.sigma, r.labels = bc, sigma, labels
        return r

    def pagerank(self, damping=0.85, epsilon=0.01, max_iter=1000, cfg=None):
        ranks = np.empty(self.nv, np.float64)
        cap = int(min(max_iter + 1, 1 << 20))
        sums = np.empty(cap, np.float64)
        it, ln = C.c_uint64(), C.c_uint64()
        st = mg_stats()
        _check(lib().ref_pagerank(self.h, damping, epsilon, max_iter, C.byref(_cfg(cfg)),
                                  _p(ranks), C.byref(it), _p(sums), cap, C.byref(ln),
                                  C.byref(st)))
        r = _collect_stats(st, self.n)
        r.ranks, r.iterations, r.rank_sums = ranks, it.value, sums[:ln.value].copy()
        return r
