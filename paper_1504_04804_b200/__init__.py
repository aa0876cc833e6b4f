"""mgraph-b200: B200-native multi-GPU graph hot path (Pan et al., arXiv 1504.04804).

Host-side mirror of the reference's C++ interface (proj/core/include/mgraph/
primitives.hpp, engine.hpp, partition.hpp) over the C-ABI library
``libmgraph_b200.so`` (include/mgraph_b200.h).  Same names, argument meaning
and error behaviour:

    g = Csr.rmat(18, 16, seed=1)                      # fixtures::rmat
    owner = partition_random(g.num_vertices, 4, 7)     # partition.cpp:31
    plan = PartitionPlan(g, owner, 4)                  # build_partition_plan + upload
    r = bfs(plan, BfsOptions(source=0))                # primitives.hpp:40
    r.labels, r.stats.supersteps, r.stats.h_matrix

Every compute call runs the hand-written sm_100a kernels; there is no CPU
fallback — if the shared object is missing or no GPU is visible the calls
raise.
"""
import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import abi
from .abi import (MG_COMM_BROADCAST, MG_COMM_DEFAULT, MG_COMM_SELECTIVE, MG_DUP_ALL, MG_DUP_ONEHOP,
                  MG_FUSED_AUTO, MG_FUSED_OFF, MG_FUSED_ON, MG_INF_DIST, MG_INF_LABEL,
                  MG_INVALID_VERTEX, MG_POLICY_FIXED, MG_POLICY_FUSED, MG_POLICY_JUST,
                  MG_POLICY_MAX, ROLES, STOP_REASONS)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmgraph_b200.so")

kInfLabel = MG_INF_LABEL
kInfDist = MG_INF_DIST
kInvalidVertex = MG_INVALID_VERTEX

_lib = None


def lib():
    """Load the in-tree CUDA library (built by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is None:
        path = os.environ.get("MG_LIB_PATH", LIB_PATH)  # experiment variants (build.py)
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: run `python -m paper_1504_04804_b200.build`"
                               " (there is no CPU fallback)")
        _lib = abi.bind(C.CDLL(path))
    return _lib


# ----------------------------------------------------------------------------- errors
class CapacityError(RuntimeError):
    """mgraph::CapacityError (frontier.hpp:98-102)"""


class CudaError(RuntimeError):
    pass


def _raise(code):
    msg = lib().mg_last_error().decode()
    if code == abi.MG_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if code == abi.MG_ECAPACITY:
        raise CapacityError(msg)
    if code == abi.MG_ECUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)  # std::runtime_error (missing proxy, worker failure)


def _check(code):
    if code != abi.MG_OK:
        _raise(code)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------------------- graphs
class Csr:
    """Host CSR graph (reference Csr, csr.hpp:38-52), owned by the library."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.mg_graph_destroy(self._h)
            self._h = None

    @classmethod
    def _make(cls, fn, *args):
        out = C.c_void_p()
        _check(fn(*args, C.byref(out)))
        return cls(out.value)

    @classmethod
    def from_csr(cls, row_offsets, col_indices, edge_values=None):
        off = np.ascontiguousarray(row_offsets, np.uint32)
        col = np.ascontiguousarray(col_indices, np.uint32)
        w = None if edge_values is None else np.ascontiguousarray(edge_values, np.uint32)
        return cls._make(lib().mg_graph_from_csr, len(off) - 1, len(col), _p(off), _p(col), _p(w))

    @classmethod
    def from_edges(cls, num_vertices, edges, weighted=False):
        """build_csr (csr.cpp:27-69) from (src, dst[, w]) rows"""
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 3 if weighted else 2) if len(edges) else \
            np.zeros((0, 3 if weighted else 2), np.int64)
        src = np.ascontiguousarray(e[:, 0], np.uint32)
        dst = np.ascontiguousarray(e[:, 1], np.uint32)
        w = np.ascontiguousarray(e[:, 2], np.uint32) if weighted else None
        return cls._make(lib().mg_graph_from_edges, num_vertices, len(src), _p(src), _p(dst), _p(w))

    @classmethod
    def rmat(cls, scale, edge_factor, seed, a=0.57, b=0.19, c=0.19, d=0.05, symmetrize=True):
        """rmat_generate -> build_csr -> symmetrize_dedup (fixtures.hpp:56-63)"""
        return cls._make(lib().mg_graph_rmat, scale, edge_factor, a, b, c, d, seed, int(symmetrize))

    @classmethod
    def rmat_hashed(cls, scale, edge_factor, seed, threads=0):
        """counter-based R-MAT (host twin of the device generator)"""
        return cls._make(lib().mg_graph_rmat_hashed, scale, edge_factor, seed, threads)

    @classmethod
    def grid(cls, rows, cols):
        return cls._make(lib().mg_graph_grid, rows, cols)

    @classmethod
    def path(cls, n):
        return cls._make(lib().mg_graph_path, n)

    def symmetrize_dedup(self):
        return Csr._make(lib().mg_graph_symmetrize, self._h)

    def with_weights(self, lo, hi, seed):
        """assign_random_weights (generate.cpp:64-79)"""
        return Csr._make(lib().mg_graph_assign_weights, self._h, lo, hi, seed)

    @property
    def num_vertices(self):
        return self._info()[0]

    @property
    def num_edges(self):
        return self._info()[1]

    def has_weights(self):
        return bool(self._info()[2])

    def _info(self):
        nv, ne, w = C.c_uint32(), C.c_uint64(), C.c_int()
        _check(lib().mg_graph_info(self._h, C.byref(nv), C.byref(ne), C.byref(w)))
        return nv.value, ne.value, w.value

    def arrays(self):
        """(row_offsets, col_indices, edge_values|None) as numpy copies"""
        nv, ne, has_w = self._info()
        po, pc, pw = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(lib().mg_graph_arrays(self._h, C.byref(po), C.byref(pc), C.byref(pw)))
        off = np.ctypeslib.as_array(C.cast(po, C.POINTER(C.c_uint32)), (nv + 1,)).copy()
        col = np.ctypeslib.as_array(C.cast(pc, C.POINTER(C.c_uint32)), (max(ne, 1),))[:ne].copy() \
            if ne else np.zeros(0, np.uint32)
        w = None
        if has_w:
            w = np.ctypeslib.as_array(C.cast(pw, C.POINTER(C.c_uint32)), (max(ne, 1),))[:ne].copy() \
                if ne else np.zeros(0, np.uint32)
        return off, col, w


# ----------------------------------------------------------------------------- partitioners
def partition_random(num_vertices, n, seed):
    """Uniform owner per vertex (partition.cpp:31-40)."""
    out = np.empty(num_vertices, np.uint32)
    _check(lib().mg_partition_random(num_vertices, n, seed, _p(out)))
    return out


def partition_biased_random(g: Csr, n, seed, bias):
    """Border-minimising biased random partitioner (partition.cpp:42-85)."""
    out = np.empty(g.num_vertices, np.uint32)
    _check(lib().mg_partition_biased_random(g._h, n, seed, bias, _p(out)))
    return out


class Duplication:
    All = MG_DUP_ALL
    OneHop = MG_DUP_ONEHOP


class CommMode:
    Selective = MG_COMM_SELECTIVE
    Broadcast = MG_COMM_BROADCAST


class AllocPolicyKind:
    JustEnough = MG_POLICY_JUST
    FixedPrealloc = MG_POLICY_FIXED
    Maximum = MG_POLICY_MAX
    PreallocFused = MG_POLICY_FUSED


class FusedMode:
    Auto = MG_FUSED_AUTO
    On = MG_FUSED_ON
    Off = MG_FUSED_OFF


@dataclass
class DropPackage:
    src: int = 0
    dst: int = 0
    iteration: int = 0


@dataclass
class EngineConfig:
    """EngineConfig (engine.hpp:308-315) + AllocationPolicy (frontier.hpp:63-69)"""
    policy: int = MG_POLICY_JUST
    factors: Dict[str, float] = field(default_factory=dict)
    hard_cap_bytes: int = 0
    fused: int = MG_FUSED_AUTO
    comm_override: Optional[int] = None
    h_inflation: int = 1
    drop_package: Optional[DropPackage] = None
    max_supersteps: int = 1000000
    dobfs_exact_cost: bool = False

    def to_c(self):
        c = abi.default_config()
        c.policy = self.policy
        c.fused = self.fused
        c.comm_override = MG_COMM_DEFAULT if self.comm_override is None else self.comm_override
        c.h_inflation = self.h_inflation
        c.max_supersteps = self.max_supersteps
        c.hard_cap_bytes = self.hard_cap_bytes
        c.dobfs_exact_cost = int(self.dobfs_exact_cost)
        for k, v in self.factors.items():
            c.factors[ROLES.index(k)] = v
        if self.drop_package is not None:
            c.drop_enabled = 1
            c.drop_src, c.drop_dst = self.drop_package.src, self.drop_package.dst
            c.drop_iteration = self.drop_package.iteration
        return c


class PartitionPlan:
    """build_partition_plan (partition.cpp:121-209) uploaded to the GPU(s).

    ``devices[p]`` is the CUDA ordinal of worker p (default: all on device 0;
    co-located workers exercise the multi-partition engine on one GPU)."""

    def __init__(self, g: Optional[Csr], owner=None, n=1, duplication=MG_DUP_ALL, devices=None,
                 _handle=None):
        if _handle is not None:
            self._h = C.c_void_p(_handle)
        else:
            own = None if owner is None else np.ascontiguousarray(owner, np.uint32)
            devs = None if devices is None else (C.c_int * n)(*devices)
            out = C.c_void_p()
            _check(lib().mg_plan_create(g._h, _p(own), n, duplication, devs, C.byref(out)))
            self._h = out
        nv, ne, np_ = C.c_uint32(), C.c_uint64(), C.c_uint32()
        _check(lib().mg_plan_info(self._h, C.byref(nv), C.byref(ne), C.byref(np_)))
        self.num_global_vertices, self.num_global_edges, self.n = nv.value, ne.value, np_.value

    @classmethod
    def rmat_device(cls, scale, edge_factor, seed, owner=None, n=1, weights=None, devices=None):
        """hashed R-MAT generated, symmetrized and partitioned on the GPU.
        weights = (lo, hi, seed) for mirrored hash weights."""
        own = None if owner is None else np.ascontiguousarray(owner, np.uint32)
        devs = None if devices is None else (C.c_int * n)(*devices)
        lo, hi, ws = weights if weights else (0, 0, 0)
        out = C.c_void_p()
        _check(lib().mg_plan_create_rmat_device(scale, edge_factor, seed, int(bool(weights)), lo,
                                                hi, ws, _p(own), n, devs, C.byref(out)))
        return cls(None, _handle=out.value)

    @classmethod
    def rgg_device(cls, num_vertices, seed, owner=None, n=1, devices=None):
        """random geometric graph generated + partitioned on the GPU (r = 0.55 sqrt(ln n/n))"""
        own = None if owner is None else np.ascontiguousarray(owner, np.uint32)
        devs = None if devices is None else (C.c_int * n)(*devices)
        out = C.c_void_p()
        _check(lib().mg_plan_create_rgg_device(num_vertices, seed, _p(own), n, devs,
                                               C.byref(out)))
        return cls(None, _handle=out.value)

    @classmethod
    def multiprocess(cls, g: Csr, owner, n, rank, device, key, duplication=MG_DUP_ALL):
        """One process per GPU: this rank uploads partition `rank` to `device`
        and rendezvous with its peers through the job-unique `key`
        (include/mgraph_b200.h, mg_plan_create_mp)."""
        own = np.ascontiguousarray(owner, np.uint32)
        out = C.c_void_p()
        _check(lib().mg_plan_create_mp(g._h, _p(own), n, duplication, rank, device,
                                       key.encode(), C.byref(out)))
        p = cls(None, _handle=out.value)
        p.rank = rank
        return p

    @classmethod
    def rmat_device_multiprocess(cls, scale, edge_factor, seed, owner, n, rank, device, key,
                                 weights=None):
        own = np.ascontiguousarray(owner, np.uint32)
        lo, hi, ws = weights if weights else (0, 0, 0)
        out = C.c_void_p()
        _check(lib().mg_plan_create_rmat_device_mp(scale, edge_factor, seed, int(bool(weights)),
                                                   lo, hi, ws, _p(own), n, rank, device,
                                                   key.encode(), C.byref(out)))
        p = cls(None, _handle=out.value)
        p.rank = rank
        return p

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.mg_plan_destroy(self._h)
            self._h = None

    def num_partitions(self):
        return self.n

    def border_metrics(self):
        """(pair_border n x n, edge_cut) — BorderMetrics (partition.cpp:211-242)"""
        pair = np.zeros(self.n * self.n, np.uint64)
        cut = C.c_uint64()
        _check(lib().mg_plan_border_metrics(self._h, _p(pair), C.byref(cut)))
        return pair.reshape(self.n, self.n), cut.value

    def pair_border(self):
        pair = np.zeros(self.n * self.n, np.uint64)
        _check(lib().mg_plan_border_metrics(self._h, _p(pair), None))
        return pair.reshape(self.n, self.n)

    def download_graph(self):
        return Csr._make(lib().mg_plan_download_graph, self._h)

    def fetch(self, which, dtype):
        out = np.empty(self.num_global_vertices, dtype)
        _check(lib().mg_plan_fetch(self._h, which, _p(out)))
        return out


# ----------------------------------------------------------------------------- results
@dataclass
class BufferStats:
    realloc_count: int
    peak_items: int
    peak_bytes: int


class RunStats:
    """RunStats (engine.hpp:261-298)"""

    def __init__(self, plan: PartitionPlan, st, primitive="?"):
        n = st.n
        self.primitive = primitive
        self.n = n
        self.supersteps = st.supersteps
        self.edges_examined = st.edges_examined
        self.combine_ops = st.combine_ops
        self.wire_records = st.wire_records
        self.peak_bytes = st.peak_bytes
        self.reallocs = st.reallocs
        self.wall_ms = st.wall_ms
        self.exchange_ms = st.exchange_ms
        self.device_ms = st.device_ms
        self.gpu_launches = st.gpu_launches
        self.device_loop = bool(st.device_loop)  # supersteps ran as one CUDA graph
        self.exchange_bytes = st.exchange_bytes
        self.stop_reason = STOP_REASONS[st.stop_reason]
        self.communication = "broadcast" if st.communication == MG_COMM_BROADCAST else "selective"
        self.policy = ("just", "fixed", "max", "fused")[st.policy]

        def arr(which):
            ln = C.c_uint64()
            _check(lib().mg_plan_last_array(plan._h, which, None, 0, C.byref(ln)))
            a = np.zeros(ln.value, np.uint64)
            _check(lib().mg_plan_last_array(plan._h, which, _p(a), ln.value, C.byref(ln)))
            return a

        self.h_matrix = arr(abi.MG_ARR_H_MATRIX).reshape(n, n) if n else np.zeros((0, 0))
        self.h_per_iter_by_src = arr(abi.MG_ARR_H_PER_ITER).reshape(-1, n)
        self.out_per_iter = arr(abi.MG_ARR_OUT_PER_ITER)
        self.edges_per_iter = arr(abi.MG_ARR_EDGES_PER_ITER)
        self.combine_per_iter = arr(abi.MG_ARR_COMBINE_PER_ITER)
        self.worker_buffers: List[Dict[str, BufferStats]] = []
        for wk in range(n):
            d = {}
            for r, name in enumerate(ROLES):
                a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
                if lib().mg_plan_last_buffer_stats(plan._h, wk, r, C.byref(a), C.byref(b),
                                                   C.byref(c)) == 0:
                    d[name] = BufferStats(a.value, b.value, c.value)
            self.worker_buffers.append(d)

    def h_total(self):
        return int(self.h_matrix.sum())

    def to_json(self, partitioner="unspecified", duplication="all", h_inflation=1):
        """the reference's RunStats JSON document (stats_json.hpp:28-61), same keys"""
        return {
            "primitive": self.primitive, "n": int(self.n), "partitioner": partitioner,
            "duplication": duplication, "communication": self.communication,
            "policy": self.policy, "S": int(self.supersteps), "W": int(self.edges_examined),
            "C": int(self.combine_ops), "H": self.h_matrix.astype(int).tolist(),
            "H_total": self.h_total(),
            "H_per_iter_by_src": self.h_per_iter_by_src.astype(int).tolist(),
            "out_per_iter": self.out_per_iter.astype(int).tolist(),
            "edges_per_iter": self.edges_per_iter.astype(int).tolist(),
            "wall_ms": float(self.wall_ms), "exchange_ms": float(self.exchange_ms),
            "h_inflation": int(h_inflation), "wire_records": int(self.wire_records),
            "stop_reason": self.stop_reason, "peak_bytes": int(self.peak_bytes),
            "reallocs": int(self.reallocs),
            "buffers": [{role: {"reallocs": int(b.realloc_count), "peak_items": int(b.peak_items),
                                "peak_bytes": int(b.peak_bytes)} for role, b in wb.items()}
                        for wb in self.worker_buffers],
        }

    def h_from(self, i):
        return int(self.h_matrix[i].sum())


class Result:
    pass


def _cfg(cfg):
    return (cfg or EngineConfig()).to_c()


@dataclass
class BfsOptions:
    source: int = 0
    mark_preds: bool = False


@dataclass
class DobfsOptions:
    source: int = 0
    do_a: float = 0.01
    do_b: float = 0.1
    mark_preds: bool = False


@dataclass
class PrOptions:
    damping: float = 0.85
    epsilon: float = 0.01
    max_iter: int = 1000


def bfs(plan: PartitionPlan, opt: BfsOptions = BfsOptions(), cfg: EngineConfig = None,
        download=True):
    """BfsResult bfs(plan, opt, cfg) (primitives.hpp:40)"""
    nv = plan.num_global_vertices
    labels = np.empty(nv, np.uint32) if download else None
    preds = np.empty(nv, np.uint32) if (download and opt.mark_preds) else None
    st = abi.mg_stats()
    _check(lib().mg_bfs(plan._h, opt.source, int(opt.mark_preds), C.byref(_cfg(cfg)), _p(labels),
                        _p(preds), C.byref(st)))
    r = Result()
    r.labels, r.preds, r.stats = labels, preds, RunStats(plan, st, "bfs")
    return r


def dobfs(plan: PartitionPlan, opt: DobfsOptions = DobfsOptions(), cfg: EngineConfig = None,
          download=True):
    """DobfsResult dobfs(plan, opt, cfg) (primitives.hpp:85)"""
    nv = plan.num_global_vertices
    labels = np.empty(nv, np.uint32) if download else None
    preds = np.empty(nv, np.uint32) if (download and opt.mark_preds) else None
    dl = np.zeros(4096, np.int32)
    ln, fw, bw = C.c_uint64(), C.c_uint64(), C.c_uint64()
    st = abi.mg_stats()
    _check(lib().mg_dobfs(plan._h, opt.source, opt.do_a, opt.do_b, int(opt.mark_preds),
                          C.byref(_cfg(cfg)), _p(labels), _p(preds), _p(dl), len(dl), C.byref(ln),
                          C.byref(fw), C.byref(bw), C.byref(st)))
    r = Result()
    r.labels, r.preds, r.stats = labels, preds, RunStats(plan, st, "dobfs")
    if ln.value > len(dl):  # longer than the buffer: the library keeps the whole log
        full = np.zeros(ln.value, np.uint64)
        got = C.c_uint64()
        _check(lib().mg_plan_last_array(plan._h, abi.MG_ARR_DIRECTION_LOG, _p(full), ln.value,
                                        C.byref(got)))
        r.direction_log = full.astype(np.int32)
    else:
        r.direction_log = dl[:ln.value].copy()
    r.forward_edges, r.backward_edges = fw.value, bw.value
    return r


def make_direction_state(current, q, u, p, edges, vertices, do_a, do_b, switched_once):
    s = abi.mg_direction_state()
    lib().mg_make_direction_state(current, q, u, p, edges, vertices, do_a, do_b,
                                  int(switched_once), C.byref(s))
    return s


def direction_decide(s):
    """0 = forward, 1 = backward (primitives.cpp:147-154)"""
    return lib().mg_direction_decide(C.byref(s))


def sssp(plan: PartitionPlan, source=0, mark_preds=False, cfg: EngineConfig = None, download=True):
    """SsspResult sssp(plan, source, mark_preds, cfg) (primitives.hpp:97)"""
    nv = plan.num_global_vertices
    d = np.empty(nv, np.uint64) if download else None
    preds = np.empty(nv, np.uint32) if (download and mark_preds) else None
    st = abi.mg_stats()
    _check(lib().mg_sssp(plan._h, source, int(mark_preds), C.byref(_cfg(cfg)), _p(d), _p(preds),
                         C.byref(st)))
    r = Result()
    r.dists, r.preds, r.stats = d, preds, RunStats(plan, st, "sssp")
    return r


def cc(plan: PartitionPlan, cfg: EngineConfig = None, download=True):
    """CcResult cc(plan, cfg) (primitives.hpp:108)"""
    comp = np.empty(plan.num_global_vertices, np.uint32) if download else None
    st = abi.mg_stats()
    _check(lib().mg_cc(plan._h, C.byref(_cfg(cfg)), _p(comp), C.byref(st)))
    r = Result()
    r.components, r.stats = comp, RunStats(plan, st, "cc")
    return r


def bc(plan: PartitionPlan, source=0, cfg: EngineConfig = None, download=True):
    """BcResult bc(plan, source, cfg) (primitives.hpp:120)"""
    nv = plan.num_global_vertices
    b = np.empty(nv, np.float64) if download else None
    s = np.empty(nv, np.float64) if download else None
    lab = np.empty(nv, np.uint32) if download else None
    st = abi.mg_stats()
    _check(lib().mg_bc(plan._h, source, C.byref(_cfg(cfg)), _p(b), _p(s), _p(lab), C.byref(st)))
    r = Result()
    r.bc, r.sigma, r.labels, r.stats = b, s, lab, RunStats(plan, st, "bc")
    return r


def pagerank(plan: PartitionPlan, opt: PrOptions = PrOptions(), cfg: EngineConfig = None,
             download=True):
    """PrResult pagerank(plan, opt, cfg) (primitives.hpp:138)"""
    nv = plan.num_global_vertices
    ranks = np.empty(nv, np.float64) if download else None
    cap = int(min(opt.max_iter + 2, 1 << 20))
    sums = np.empty(cap, np.float64)
    it, ln = C.c_uint64(), C.c_uint64()
    st = abi.mg_stats()
    _check(lib().mg_pagerank(plan._h, opt.damping, opt.epsilon, opt.max_iter, C.byref(_cfg(cfg)),
                             _p(ranks), C.byref(it), _p(sums), cap, C.byref(ln), C.byref(st)))
    r = Result()
    r.ranks, r.iterations, r.rank_sums = ranks, it.value, sums[:ln.value].copy()
    r.stats = RunStats(plan, st, "pagerank")
    return r


def kernel_launch_count():
    return lib().mg_kernel_launch_count()
