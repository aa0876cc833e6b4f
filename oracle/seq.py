"""ctypes binding of the plain-C restatement (oracle/seq_oracle.c). TEST-ONLY."""
import ctypes as C
import os

import numpy as np

from . import REF_DIR

_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(REF_DIR, "libmgoracle.so")
        if not os.path.exists(path):
            from . import build
            build()
        _lib = C.CDLL(path)
        P = C.c_void_p
        _lib.mgo_bfs_levels.argtypes = [C.c_uint32, P, P, C.c_uint32, P]
        _lib.mgo_dijkstra.argtypes = [C.c_uint32, P, P, P, C.c_uint32, P]
        _lib.mgo_connected_components.argtypes = [C.c_uint32, P, P, P]
        _lib.mgo_brandes_bc.argtypes = [C.c_uint32, P, P, C.c_uint32, P, P, P]
        _lib.mgo_pagerank.argtypes = [C.c_uint32, P, P, C.c_double, C.c_double, C.c_uint64, P,
                                      P, C.c_uint64]
        _lib.mgo_pagerank.restype = C.c_uint64
        _lib.mgo_direction_decide.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double,
                                              C.c_double, C.c_int]
        _lib.mgo_direction_decide.restype = C.c_int
        _lib.mgo_direction_estimates.argtypes = [C.c_uint64] * 5 + [P, P]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _csr(off, col):
    off = np.ascontiguousarray(off, dtype=np.uint32)
    col = np.ascontiguousarray(col, dtype=np.uint32)
    return off, col, len(off) - 1


def bfs_levels(off, col, source):
    off, col, nv = _csr(off, col)
    out = np.empty(nv, np.uint32)
    lib().mgo_bfs_levels(nv, _p(off), _p(col), source, _p(out))
    return out


def dijkstra(off, col, w, source):
    off, col, nv = _csr(off, col)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.uint32)
    out = np.empty(nv, np.uint64)
    lib().mgo_dijkstra(nv, _p(off), _p(col), _p(w), source, _p(out))
    return out


def connected_components(off, col):
    off, col, nv = _csr(off, col)
    out = np.empty(nv, np.uint32)
    lib().mgo_connected_components(nv, _p(off), _p(col), _p(out))
    return out


def brandes_bc(off, col, source):
    """returns (bc, sigma, labels)"""
    off, col, nv = _csr(off, col)
    bc = np.empty(nv, np.float64)
    sigma = np.empty(nv, np.float64)
    dist = np.empty(nv, np.uint32)
    lib().mgo_brandes_bc(nv, _p(off), _p(col), source, _p(bc), _p(sigma), _p(dist))
    return bc, sigma, dist


def pagerank_power(off, col, damping, epsilon, max_iter):
    """returns (ranks, iterations, rank_sums)"""
    off, col, nv = _csr(off, col)
    ranks = np.empty(nv, np.float64)
    cap = int(min(max_iter, 1 << 20))
    sums = np.empty(max(cap, 1), np.float64)
    it = lib().mgo_pagerank(nv, _p(off), _p(col), damping, epsilon, max_iter, _p(ranks),
                            _p(sums), cap)
    return ranks, int(it), sums[:min(it, cap)].copy()


def direction_decide(current, fv, bv, do_a, do_b, switched):
    return lib().mgo_direction_decide(current, fv, bv, do_a, do_b, switched)


def direction_estimates(q, u, p, edges, vertices):
    fv, bv = C.c_double(), C.c_double()
    lib().mgo_direction_estimates(q, u, p, edges, vertices, C.byref(fv), C.byref(bv))
    return fv.value, bv.value
