// prims.cu — the six primitives of primitives.cpp as device functor sets +
// host hooks for the enactor (engine.cuh), and their C-ABI entry points.
//
// Each primitive mirrors its reference PrimitiveSpec field by field:
// init / iteration_body / combine / gather / send_filter / comm_selector /
// stop_condition / finalize (engine.hpp:587-626).  Device functors implement
// the per-vertex hooks with atomics whose outcome is independent of thread
// order (atomicCAS / atomicMin / atomicExch stamps), so labels, distances and
// components are bit-identical to the sequential reference.
#include <cub/block/block_reduce.cuh>
#include <cub/device/device_radix_sort.cuh>

#include <cmath>
#include <cstring>

#include "engine.cuh"

namespace mgb {

void gather_u32(Plan& P, const std::vector<const uint32_t*>& pw, uint32_t* out);
void gather_labels_u32(Plan& P, const std::vector<const uint32_t*>& pw, uint32_t* out,
                       uint64_t max_label);
void gather_u64(Plan& P, const std::vector<const unsigned long long*>& pw, uint64_t* out);
void gather_f64(Plan& P, const std::vector<const double*>& pw, double* out);

namespace {

// defaults of the PrimitiveSpec hooks
struct PrimBase {
  const char* name = "?";
  int nva = 0, nvv = 0;
  int communication = MG_COMM_SELECTIVE;
  bool allow_comm_override = false;
  int dup_required = MG_DUP_ALL;
  bool has_stop_condition = false;
  bool reports_deg = false;  // body leaves Σdeg(next frontier) in ctr->next_deg
  uint64_t inbox_bound(Plan& P, uint32_t src, uint32_t dst, int comm) const {
    // selective: each proxy at most once per superstep (keep dedup) -> |B_{src,dst}|;
    // broadcast: the whole output, bounded by |V_src| local IDs
    return comm == MG_COMM_BROADCAST ? P.workers[src] ? P.workers[src]->nv : P.nv
                                     : P.pair_border[src][dst];
  }
  int comm_selector(Ctx&, int comm) { return comm; }
  DenseView dense_view(Ctx&) const { return {}; }  // records only
  bool stop_condition(const GlobalView&) { return false; }
  void after_merge(Ctx&) {}
  void finalize(Ctx&, const GlobalView&) {}
};

template <class T>
void fill(DevArray<T>& a, uint64_t n, int byte, cudaStream_t s) {
  if (a.n < n || !a.ptr) a.alloc(n ? n : 1);
  MGB_CUDA(cudaMemsetAsync(a.ptr, byte, sizeof(T) * (n ? n : 1), s));
}

template <class T>
__global__ void set_one_kernel(T* a, uint32_t i, T v) {
  a[i] = v;
}

__global__ void fill_f64_kernel(double* a, uint32_t n, double v) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[i] = v;
}

__global__ void fill_hosted_f64_kernel(double* a, const uint32_t* hosted, uint32_t n, double v) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[hosted[i]] = v;
}

__global__ void or_word_kernel(uint32_t* w, uint32_t bit) { *w |= bit; }

__global__ void iota_kernel(uint32_t* a, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[i] = i;
}

// atomicMax on non-negative doubles through their ordered bit patterns
__device__ __forceinline__ void atomic_max_pos_f64(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

// ===========================================================================
// BFS (primitives.cpp:60-126)

// Single partition of >= 2^22 vertices: visited state as a bitmap (|V|/8 bytes,
// L2-resident at RMAT-26) instead of probing the 4-byte label of every arc's
// head (RMAT-26 BFS 20.1 -> 16.4 ms); the
// test-and-set makes each discovery unique, so the keep stamp is not needed.
// Several partitions keep the label CAS (remote combines lower labels).
struct BfsDev {
  uint32_t* labels;
  uint32_t* preds;
  uint32_t* seen;
  uint32_t* vis;  // visited bitmap (single partition) or nullptr
  OwnerView ow;
  uint32_t iter;
  int mark_preds;
  // dense push (bitmap, no predecessors; as DobfsDev::red): when the
  // advance's arc count reaches red_min, visits only set visited bits with a
  // fire-and-forget OR; labels and the output come from vis & ~prev
  const unsigned long long* red_total = nullptr;
  unsigned long long red_min = 0;
  __device__ bool dense() const { return vis && red_min && *red_total >= red_min; }
  // visit: unvisited -> label iter+1 (+pred); the CAS / test-and-set makes the
  // discovery unique (called only for arcs whose prefilter() saw it unvisited)
  __device__ bool visit(uint32_t u, uint32_t v, uint32_t) const {
    if (vis) {
      const uint32_t bit = 1u << (v & 31);
      if (atomicOr(&vis[v >> 5], bit) & bit) return false;
      labels[v] = iter + 1;
    } else if (atomicCAS(&labels[v], kInfLabel, iter + 1) != kInfLabel) {
      return false;
    }
    if (mark_preds) preds[v] = ow.to_global(u);
    return true;
  }
  // keep: per-superstep stamp dedup (primitives.cpp:89-94)
  __device__ bool keep(uint32_t v) const {
    return vis || atomicExch(&seen[v], iter + 1) != iter + 1;
  }
  __device__ bool prefilter(uint32_t v) const {
    return vis ? !((__ldcg(&vis[v >> 5]) >> (v & 31)) & 1u) : __ldcg(&labels[v]) == kInfLabel;
  }
  // combine (primitives.cpp:98-107): iter+1 < label -> set, enqueue iff hosted
  __device__ bool combine(uint32_t v, const uint32_t* va, const double*, uint32_t it) const {
    uint32_t cand = it + 1;
    uint32_t old = atomicMin(&labels[v], cand);
    if (cand < old) {
      if (mark_preds) preds[v] = va[0];
      return ow.hosts(v);
    }
    return false;
  }
  __device__ void gather(uint32_t v, uint32_t* va, double*) const {
    if (mark_preds) va[0] = preds[v];
  }
  __device__ bool send_filter(uint32_t, uint32_t) const { return true; }
  __device__ uint32_t peer_id(uint32_t v, uint32_t, uint32_t) const { return v; }
};

// batched visits: the whole batch's test-and-sets in flight together
template <int K>
__device__ __forceinline__ void visit_batch(const BfsDev& f, const uint32_t* src,
                                            const uint32_t* nb, const uint32_t* eid,
                                            const bool* pass, bool* acc) {
  if (!f.vis) {
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = pass[k] && f.visit(src[k], nb[k], eid[k]);
    return;
  }
  if (f.dense()) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (pass[k])
        asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(&f.vis[nb[k] >> 5]),
                     "r"(1u << (nb[k] & 31))
                     : "memory");
      acc[k] = false;
    }
    return;
  }
  uint32_t old[K];
#pragma unroll
  for (int k = 0; k < K; ++k)
    old[k] = pass[k] ? atomicOr(&f.vis[nb[k] >> 5], 1u << (nb[k] & 31)) : ~0u;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    acc[k] = !(old[k] & (1u << (nb[k] & 31)));
    if (acc[k]) {
      f.labels[nb[k]] = f.iter + 1;
      if (f.mark_preds) f.preds[nb[k]] = f.ow.to_global(src[k]);
    }
  }
}

__device__ __forceinline__ bool expand_quiet(const BfsDev& f) { return f.dense(); }
__device__ __forceinline__ bool expand_needs_src(const BfsDev& f) { return f.mark_preds != 0; }
}  // namespace
template <>
struct expand_long_rows<BfsDev> {
  static constexpr bool value = true;
};
namespace {

static unsigned long long dense_push_arcs();
__global__ void bitmap_diff_list_kernel(const uint32_t* __restrict__ vis, uint32_t* prev,
                                        uint32_t nw, uint32_t* out, uint32_t* cnt, int set_prev,
                                        const struct DobfsLoop* st, uint32_t* labels,
                                        uint32_t level, const unsigned long long* need_total,
                                        unsigned long long need_min);

struct BfsPrim : PrimBase {
  uint32_t source;
  bool mark_preds;
  bool bitmap = false;  // single partition: visited bitmap in su32[3]
  BfsPrim(uint32_t s, bool m) : source(s), mark_preds(m) {
    name = "bfs";
    nva = m ? 1 : 0;
    allow_comm_override = true;
  }
  void init(Ctx& c) {  // primitives.cpp:71-79
    Worker& w = *c.w;
    // the bitmap pays off once the label array outgrows L2 (small graphs keep
    // the label CAS: one launch less at init, same result)
    bitmap = c.P->n == 1 && w.nv >= (1u << 22);
    fill(w.su32[0], w.nv, 0xFF, w.stream);  // labels = inf
    if (bitmap) {
      fill(w.su32[3], (w.nv + 31) / 32 + 1, 0, w.stream);  // visited bitmap
      MGB_LAUNCH(or_word_kernel, 1, 1, 0, w.stream, w.su32[3].ptr + (source >> 5),
                 1u << (source & 31));
    } else {
      fill(w.su32[2], w.nv, 0, w.stream);  // seen
    }
    if (mark_preds) fill(w.su32[1], w.nv, 0xFF, w.stream);
    MGB_LAUNCH(set_one_kernel<uint32_t>, 1, 1, 0, w.stream, w.su32[0].ptr, source, 0u);
    if (c.P->owner_host[source] == w.p) c.push_initial({source});
  }
  BfsDev dev(Ctx& c) {
    Worker& w = *c.w;
    return {w.su32[0].ptr, w.su32[1].ptr, w.su32[2].ptr, bitmap ? w.su32[3].ptr : nullptr,
            c.owner_view(), (uint32_t)c.iter, mark_preds ? 1 : 0};
  }
  void body(Ctx& c) {
    Worker& w = *c.w;
    if (bitmap && c.fused && !mark_preds && dense_push_arcs() && c.in_count) {
      // dense when the advance examines >= dense_push_arcs() arcs (DobfsPrim)
      const uint64_t nw = w.nv / 32 + 1;
      if (w.su32[2].n < nw || !w.su32[2].ptr) w.su32[2].alloc(nw);  // prev (seen is unused)
      MGB_CUDA(cudaMemcpyAsync(w.su32[2].ptr, w.su32[3].ptr, 4 * nw, cudaMemcpyDeviceToDevice,
                               w.stream));
      const uint32_t nb = (c.in_count + kLbBlock - 1) / kLbBlock;  // lb_advance's total slot
      if (w.lb_bsum.n < nb + 1ull) w.lb_bsum.alloc(nb + 1ull);
      BfsDev f = dev(c);
      f.red_total = w.lb_bsum.ptr + nb;
      f.red_min = dense_push_arcs();
      c.pipeline(f, w.nv);
      MGB_LAUNCH(bitmap_diff_list_kernel, grid_for(nw, 256, num_sms() * 8), 256, 0, w.stream,
                 w.su32[3].ptr, w.su32[2].ptr, (uint32_t)nw, w.output.ptr, &c.ctr()->out_cnt, 0,
                 (const DobfsLoop*)nullptr, w.su32[0].ptr, (uint32_t)c.iter + 1, f.red_total,
                 f.red_min);
      return;
    }
    c.pipeline(dev(c), c.w->nv);
  }
};

// ===========================================================================
// DOBFS (primitives.cpp:131-289)
//
// B200 layout: visited and frontier sets are BITMAPS (|V|/8 bytes each: 8 MiB
// at scale 26, resident in the 126 MB L2), so the per-arc membership tests of
// both directions hit L2 instead of HBM.  The pull step walks a compacted
// unvisited list (the paper's split of the unvisited queue),
// seeded from the plan's list of non-isolated hosted vertices so the ~half of
// an RMAT graph that is isolated is never touched.  Results and the
// examined-edge count W are those of the reference's scan (first hit in arc
// order), so labels, direction log and W match it exactly.

// exact-cost physical direction: pull when Σdeg(Q) > ratio * |unvisited list|
// (MG_PULL_RATIO overrides the default, for the sweep in DESIGN.md §7)
// A push superstep of the host-driven loop that examines at least this many
// arcs runs dense (DobfsDev::red) on one partition without predecessors under
// the fused policy (MG_DOBFS_DENSE_ARCS, 0 = never).  Reference schedule over
// the bench sources: 27.4 ms never, 17.2 ms at 2^20 arcs.
static unsigned long long dense_push_arcs() {
  static const unsigned long long a = [] {
    const char* e = getenv("MG_DOBFS_DENSE_ARCS");
    return e ? (unsigned long long)atoll(e) : (1ull << 20);
  }();
  return a;
}

// The device-driven (exact-cost) loop: dense pushes from 2^20 arcs
// (MG_DOBFS_LOOP_DENSE_ARCS, 0 = never).  They lost while the end kernel ran
// 4 CTAs per SM (MG_LOOP_END_CTAS above); at 8 they win (6.89 -> 6.78 ms).
static unsigned long long loop_dense_push_arcs() {
  static const unsigned long long a = [] {
    const char* e = getenv("MG_DOBFS_LOOP_DENSE_ARCS");
    return e ? (unsigned long long)atoll(e) : (1ull << 20);
  }();
  return a;
}

static double pull_ratio() {
  static const double r = [] {
    const char* e = getenv("MG_PULL_RATIO");
    return e ? atof(e) : 3.0;
  }();
  return r;
}

// ---- device-driven supersteps (see DobfsGraph below) ------------------------
struct DobfsLoop {
  // per-run parameters, written by the host before the graph launch
  double nv_d, ne_d, do_a, do_b, pull_ratio;
  uint32_t nv, source, max_supersteps, exact;
  // superstep state, owned by the device
  uint32_t iter, dir, switched, physical;
  uint32_t in_count, ul_src, ul_len, n_nonisolated;
  unsigned long long in_degsum, visited;
  uint32_t prev_physical;        // the last superstep was a pull (its list is clean)
  uint32_t end_ticket;           // CTAs of a branch's last kernel that finished
};
struct DobfsHist {
  uint32_t dir, physical, out, pad;
  unsigned long long edges;
};
// the pull kernels read their per-superstep arguments from the loop state
// when dyn.st is set (graph-captured launches have fixed arguments)
struct DobfsDyn {
  const DobfsLoop* st;
  uint32_t* ub0;
  uint32_t* ub1;
};

constexpr uint32_t kLoopHist = 65536;  // supersteps recorded per run

// the direction of superstep st->iter (primitives.cpp:197-205, the reference
// rule on global quantities) and the exact-cost physical choice, in the host
// path's double arithmetic; returns the physical direction (1: pull)
__device__ uint32_t dobfs_loop_decide(DobfsLoop* st, DobfsHist* hist) {
  const uint32_t t = st->iter;
  if (t >= 1) {
    st->visited += st->in_count;
    const double fv = st->nv > 0 ? (double)st->in_count * st->ne_d / st->nv_d : 0.0;
    const double bv = st->visited > 0 ? (double)((unsigned long long)st->nv - st->visited) *
                                            st->nv_d / (double)st->visited
                                      : 0.0;
    uint32_t next;
    if (st->dir == 0) next = (!st->switched && fv > bv * st->do_a) ? 1u : 0u;
    else next = fv < bv * st->do_b ? 0u : 1u;
    if (next == 1 && st->dir == 0) st->switched = 1;
    st->dir = next;
  }
  uint32_t phys = st->dir == 1;
  if (!phys && st->exact && t > 0 && st->in_count &&
      (double)st->in_degsum > st->pull_ratio * st->ul_len)
    phys = 1;
  st->physical = phys;
  hist[t].dir = st->dir;
  hist[t].physical = phys;
  hist[t].pad = 0u;
  if (!phys && t > 0) st->in_count = 0;  // the push recounts its list from the bitmap
  return phys;
}

// superstep 0 is always a push: its decision is taken here, before the graph
// (the graph's IF handles default to push at every launch); every later
// decision is taken by the end kernel of the superstep before it, so a
// superstep costs no separate decide launch
__global__ void dobfs_loop_init_kernel(DobfsLoop* st, DobfsHist* hist, uint32_t* labels,
                                       uint32_t* vis, uint32_t* prev, uint32_t* front) {
  const uint32_t s = st->source;
  labels[s] = 0u;
  vis[s >> 5] |= 1u << (s & 31);
  prev[s >> 5] |= 1u << (s & 31);  // superstep 0's list is seeded here (prev = vis)
  front[0] = s;
  st->iter = 0;
  st->dir = 0;
  st->switched = 0;
  st->physical = 0;
  st->in_count = 1;
  st->ul_src = 2;  // every non-isolated record, no list
  st->ul_len = st->n_nonisolated;
  st->in_degsum = 0;
  st->visited = 1;
  st->prev_physical = 0;
  dobfs_loop_decide(st, hist);
}

// end of a device-driven superstep (the whole CTA): history, loop state,
// counters cleared, loop condition, the next superstep's direction
__device__ void dobfs_loop_end_cta(DobfsLoop* st, Counters* ctr, DobfsHist* hist,
                                   cudaGraphConditionalHandle h_while,
                                   cudaGraphConditionalHandle h_pull,
                                   cudaGraphConditionalHandle h_push) {
  __shared__ uint32_t s_out;
  const uint32_t t = st->iter;
  if (threadIdx.x == 0) {
    const uint32_t out = ctr->out_cnt;
    s_out = out;
    hist[t].out = out;
    hist[t].edges = ctr->edges;
    if (st->physical) {  // the pull compacted the unvisited list (ping-pong)
      st->ul_len = ctr->misc;
      st->ul_src = st->ul_src == 0 ? 1 : 0;
    }
    st->prev_physical = st->physical;
    st->in_count = out;
    st->in_degsum = ctr->next_deg;
  }
  __syncthreads();
  uint32_t* c = reinterpret_cast<uint32_t*>(ctr);
  for (uint32_t i = threadIdx.x; i < sizeof(Counters) / 4; i += blockDim.x) c[i] = 0u;
  if (threadIdx.x == 0) {
    st->iter = t + 1;
    const bool more = s_out > 0 && t + 1 < st->max_supersteps && t + 1 < kLoopHist;
    cudaGraphSetConditional(h_while, more ? 1u : 0u);
    if (more) {  // the next superstep's direction
      const uint32_t phys = dobfs_loop_decide(st, hist);
      cudaGraphSetConditional(h_pull, phys);
      cudaGraphSetConditional(h_push, phys ? 0u : 1u);
    }
  }
}

// the superstep end folded into the last kernel of each branch: the last CTA
// to finish (atomic ticket) runs it, so a superstep needs no end launch
struct DobfsLoopEnd {
  DobfsLoop* st = nullptr;
  DobfsHist* hist = nullptr;
  cudaGraphConditionalHandle h_while = 0, h_pull = 0, h_push = 0;
};

__device__ void dobfs_loop_end_last_cta(const DobfsLoopEnd& le, Counters* ctr) {
  __shared__ uint32_t s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&le.st->end_ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) le.st->end_ticket = 0u;
  dobfs_loop_end_cta(le.st, ctr, le.hist, le.h_while, le.h_pull, le.h_push);
}

// a device-loop push whose advance examines at least `min` arcs (*total) runs
// dense (DobfsDev::red): the end kernel then takes the discoveries from
// vis & ~prev (prev = vis as of the superstep's start) and writes their labels
struct DensePush {
  const unsigned long long* total;  // the advance's arc count (lb_scan)
  unsigned long long min;           // 0: never
  const uint32_t* vis;
  const uint32_t* prev;
  uint32_t* labels;
  uint32_t nw;
  __device__ bool on() const { return min && *total >= min; }
};

// CTAs per SM of the push branch's end kernel: its dense branch walks the
// whole visited bitmap (labels + degree sum of every discovery), and at 4 it
// made dense pushes lose in the device loop (bench sources: off 6.89-6.95 ms,
// dense 6.99; at 8: dense 6.77-6.78, off 6.88)
#ifndef MG_LOOP_END_CTAS
#define MG_LOOP_END_CTAS 8
#endif
// push branch's last kernel: the degree sum of the discoveries, then the end
__global__ void __launch_bounds__(256)
    dobfs_degsum_end_kernel(GraphView g, const uint32_t* __restrict__ in, Counters* ctr,
                            DobfsLoopEnd le, DensePush dp) {
  unsigned long long d = 0;
  if (dp.on()) {
    const uint32_t level = le.st->iter + 1;
    uint32_t cnt = 0;
    const uint32_t lane = lane_id();
    // warp-uniform trip count; word by word, lane l takes bit l (coalesced
    // label stores and offset loads)
    for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; b < dp.nw;
         b += gridDim.x * blockDim.x) {
      const uint32_t i = b + lane;
      const uint32_t x = i < dp.nw ? __ldcg(&dp.vis[i]) & ~__ldcs(&dp.prev[i]) : 0u;
      cnt += __popc(x);
      for (unsigned m = __ballot_sync(0xffffffffu, x != 0); m; m &= m - 1) {
        const int src = __ffs(m) - 1;
        const uint32_t xj = __shfl_sync(0xffffffffu, x, src);
        if ((xj >> lane) & 1u) {
          const uint32_t v = (b + src) * 32 + lane;
          dp.labels[v] = level;
          d += g.off[v + 1] - g.off[v];
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane_id() == 0 && cnt) atomicAdd(&ctr->out_cnt, cnt);
  } else {
    const uint32_t n = ctr->out_cnt;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += gridDim.x * blockDim.x) {
      const uint32_t v = in[i];
      d += g.off[v + 1] - g.off[v];
    }
  }
  unsigned long long* const dst[1] = {&ctr->next_deg};
  const uint64_t val[1] = {d};
  block_add_u64<1>(dst, val);
  dobfs_loop_end_last_cta(le, ctr);
}

#ifndef MG_DENSE_LDCA
#define MG_DENSE_LDCA 0
#endif
#ifndef MG_DENSE_NOPROBE
#define MG_DENSE_NOPROBE 0
#endif
struct DobfsDev {
  uint32_t* labels;
  uint32_t* preds;
  uint32_t* vis;             // visited bitmap (live)
  const uint32_t* vis_snap;  // visited bitmap as of the start of the superstep
  OwnerView ow;
  uint32_t iter;
  int mark_preds;
  const uint32_t* iter_ptr;  // device-driven supersteps: the superstep index in memory
  // forward visit (primitives.cpp:216-222): test-and-set on the visited bitmap.
  // The pre-test reads L2 (ld.cg): an L1 copy would keep showing bits other
  // SMs have since set, turning every later test into an atomic.
  // (called only for arcs whose prefilter() saw the bit clear)
  __device__ bool visit(uint32_t u, uint32_t v, uint32_t) const {
    const uint32_t bit = 1u << (v & 31);
    if (atomicOr(&vis[v >> 5], bit) & bit) return false;
    labels[v] = iter + 1;
    if (mark_preds) preds[v] = ow.to_global(u);
    return true;
  }
  __device__ bool keep(uint32_t) const { return true; }
  // pre-test on the live bitmap in L2 (ld.cg).  Measured: L1-cached (ld.ca)
  // and read-only (ld.nc) probes are no faster on RMAT-26 — the probes are
  // spread too widely for L1 reuse.
  __device__ bool prefilter(uint32_t v) const {
#if MG_DENSE_NOPROBE
    if (red || red_min) return true;  // experiment: every arc issues its RED
#endif
#if MG_DENSE_LDCA
    // a dense push tolerates stale L1 copies (a stale clear bit costs one
    // more RED, a set bit is never stale): hub words stay in L1
    if (red || red_min) return !(__ldca(&vis[v >> 5]) & (1u << (v & 31)));
#endif
    return !(__ldcg(&vis[v >> 5]) & (1u << (v & 31)));
  }
  // combine (primitives.cpp:255-265): an unvisited vertex takes the remote
  // label; accepted discoveries join the (global) next frontier everywhere
  __device__ bool combine(uint32_t v, const uint32_t* va, const double*, uint32_t it) const {
    const uint32_t bit = 1u << (v & 31);
    if (vis[v >> 5] & bit) return false;
    if (atomicOr(&vis[v >> 5], bit) & bit) return false;
    labels[v] = it + 1;
    if (mark_preds) preds[v] = va[0];
    return true;
  }
  __device__ void gather(uint32_t v, uint32_t* va, double*) const {
    if (mark_preds) va[0] = preds[v];
  }
  __device__ bool send_filter(uint32_t, uint32_t) const { return true; }
  __device__ uint32_t peer_id(uint32_t v, uint32_t, uint32_t) const { return v; }
  // dense push superstep (one partition, no predecessors): an arc whose
  // pre-test saw the bit clear sets it with a fire-and-forget OR (RED: the
  // thread never waits on the L2 for a return value) and accepts nothing; the
  // labels and the output list come afterwards from vis & ~prev
  // (bitmap_diff_list_kernel with labels), in ID order
  int red = 0;
  // device loop: dense when the advance's arc count reaches red_min (DensePush)
  const unsigned long long* red_total = nullptr;
  unsigned long long red_min = 0;
  __device__ bool dense() const { return red || (red_min && *red_total >= red_min); }
};

}  // namespace
#ifndef MG_DOBFS_EXPAND_CTAS
#define MG_DOBFS_EXPAND_CTAS 4
#endif
// The DOBFS push is bound on its visited-bit probes (L2 latency).  Compiled
// for 4, 5 and 6 resident CTAs per SM (64 / 48 / 40 registers, the last with
// spills): reference schedule over the bench sources 17.15 / 17.35 / 19.5 ms.
template <>
struct expand_min_ctas<DobfsDev> {
  static constexpr int value = MG_DOBFS_EXPAND_CTAS;
};
// hub rows: whole batches inside one row (reference schedule 18.1 -> 17.2 ms)
template <>
struct expand_long_rows<DobfsDev> {
  static constexpr bool value = true;
};
namespace {

// a dense push accepts nothing: no output queue work in the expansion
__device__ __forceinline__ bool expand_quiet(const DobfsDev& f) { return f.dense(); }
// the source vertex is read only for predecessors
__device__ __forceinline__ bool expand_needs_src(const DobfsDev& f) { return f.mark_preds != 0; }

// batched forward visit: all test-and-set atomics of the batch in flight
// before any result is consumed (see visit_batch in operators.cuh)
template <int K>
__device__ __forceinline__ void visit_batch(const DobfsDev& f, const uint32_t* src,
                                            const uint32_t* nb, const uint32_t*,
                                            const bool* pass, bool* acc) {
  if (f.dense()) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      // explicit red: a plain atomicOr shares its ATOMG with the path below
      if (pass[k])
        asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(&f.vis[nb[k] >> 5]),
                     "r"(1u << (nb[k] & 31))
                     : "memory");
      acc[k] = false;
    }
    return;
  }
  uint32_t old[K];
#pragma unroll
  for (int k = 0; k < K; ++k)
    old[k] = pass[k] ? atomicOr(&f.vis[nb[k] >> 5], 1u << (nb[k] & 31)) : ~0u;
  const uint32_t label = (f.iter_ptr ? *f.iter_ptr : f.iter) + 1;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    acc[k] = !(old[k] & (1u << (nb[k] & 31)));
    if (acc[k]) {
      f.labels[nb[k]] = label;
      if (f.mark_preds) f.preds[nb[k]] = f.ow.to_global(src[k]);
    }
  }
}

// fb = vis & ~prev (the level just discovered); prev = vis.  Thread 0 also
// resets the pull step's queue counters and stores the superstep's logical W
// (forward superstep run as a pull), saving two tiny copies per pull step.
__global__ void frontier_diff_kernel(const uint32_t* __restrict__ vis, uint32_t* prev,
                                     uint32_t* __restrict__ fb, uint32_t nw, uint32_t* zero2,
                                     unsigned long long* w_dst, unsigned long long w_val,
                                     const DobfsLoop* st = nullptr,
                                     unsigned long long* w_dyn = nullptr) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    zero2[0] = zero2[1] = 0u;
    if (st && st->dir == 0) *w_dyn = st->in_degsum;  // forward superstep run as a pull
    if (w_dst) *w_dst = w_val;
  }
  const uint4* v4 = reinterpret_cast<const uint4*>(vis);
  uint4* p4 = reinterpret_cast<uint4*>(prev);
  uint4* f4 = reinterpret_cast<uint4*>(fb);
  const uint32_t n4 = nw / 4;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
    uint4 a = v4[i], b = p4[i];
    f4[i] = make_uint4(a.x & ~b.x, a.y & ~b.y, a.z & ~b.z, a.w & ~b.w);
    p4[i] = a;
  }
  for (uint32_t i = n4 * 4 + blockIdx.x * blockDim.x + threadIdx.x; i < nw;
       i += gridDim.x * blockDim.x) {
    fb[i] = vis[i] & ~prev[i];
    prev[i] = vis[i];
  }
}

__global__ void bitmap_set_kernel(const uint32_t* __restrict__ in, uint32_t n, uint32_t* bits) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t v = in[i];
    atomicOr(&bits[v >> 5], 1u << (v & 31));
  }
}

// end of a DOBFS run whose label fill was skipped: every vertex the previous
// run reached and this one did not goes back to infinity (lastvis & ~vis;
// in RMAT runs from the giant component that is no vertex at all).  Two
// streaming 16-byte reads per 128 vertices; the next run's begin copies vis
// into lastvis.
__device__ __forceinline__ void reset_unreached(uint32_t d, uint32_t word, uint32_t* labels,
                                                uint32_t nv) {
  while (d) {
    const uint32_t v = word * 32 + (__ffs(d) - 1);
    if (v < nv) labels[v] = kInfLabel;
    d &= d - 1;
  }
}
__global__ void dobfs_label_fixup_kernel(const uint32_t* __restrict__ lastvis,
                                         const uint32_t* __restrict__ vis, uint32_t nw,
                                         uint32_t* labels, uint32_t nv) {
  const uint32_t n4 = nw / 4;
  const uint4* l4 = reinterpret_cast<const uint4*>(lastvis);
  const uint4* v4 = reinterpret_cast<const uint4*>(vis);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
    const uint4 a = __ldcs(&l4[i]), b = __ldcs(&v4[i]);
    const uint32_t d0 = a.x & ~b.x, d1 = a.y & ~b.y, d2 = a.z & ~b.z, d3 = a.w & ~b.w;
    if (d0 | d1 | d2 | d3) {
      reset_unreached(d0, 4 * i, labels, nv);
      reset_unreached(d1, 4 * i + 1, labels, nv);
      reset_unreached(d2, 4 * i + 2, labels, nv);
      reset_unreached(d3, 4 * i + 3, labels, nv);
    }
  }
  for (uint32_t i = n4 * 4 + blockIdx.x * blockDim.x + threadIdx.x; i < nw;
       i += gridDim.x * blockDim.x)
    reset_unreached(lastvis[i] & ~vis[i], i, labels, nv);
}

// start of a DOBFS run on worker w: the labels are filled with infinity only
// when the array does not hold a completed DOBFS result; otherwise the
// previous run's visited bitmap is kept for the end-of-run fixup (16 MB of
// bitmap traffic instead of the 268 MB fill at RMAT-26)
void dobfs_labels_begin(Worker& w, uint64_t nw) {
  if (w.dobfs_lastvis.n < nw || !w.dobfs_lastvis.ptr) {
    w.dobfs_lastvis.alloc(nw);
    w.dobfs_labels_ok = false;
  }
  if (w.dobfs_labels_ok && w.su32[0].ptr && w.su32[0].n >= w.nv && w.su32[2].ptr &&
      w.su32[2].n >= nw && !getenv("MG_DOBFS_FILL")) {
    MGB_CUDA(cudaMemcpyAsync(w.dobfs_lastvis.ptr, w.su32[2].ptr, 4 * nw, cudaMemcpyDeviceToDevice,
                             w.stream));
  } else {
    if (w.su32[0].n < w.nv || !w.su32[0].ptr) w.su32[0].alloc(w.nv ? w.nv : 1);
    MGB_CUDA(cudaMemsetAsync(w.su32[0].ptr, 0xFF, 4ull * (w.nv ? w.nv : 1), w.stream));
    MGB_CUDA(cudaMemsetAsync(w.dobfs_lastvis.ptr, 0, 4 * nw, w.stream));
  }
  w.dobfs_labels_ok = false;  // until this run completes
}

void dobfs_labels_end(Worker& w, uint64_t nw) {
  MGB_LAUNCH(dobfs_label_fixup_kernel, grid_for(nw / 4 + 1, 256, num_sms() * 8), 256, 0, w.stream,
             w.dobfs_lastvis.ptr, w.su32[2].ptr, (uint32_t)nw, w.su32[0].ptr, w.nv);
}

__global__ void select_nonisolated_kernel(const uint32_t* __restrict__ hosted, uint32_t nh,
                                          const uint32_t* __restrict__ off, uint32_t* out,
                                          uint32_t* cnt) {
  for (uint32_t base = blockIdx.x * blockDim.x; base < nh; base += gridDim.x * blockDim.x) {
    uint32_t i = base + threadIdx.x;
    uint32_t v = i < nh ? hosted[i] : 0;
    bool keep = i < nh && off[v + 1] > off[v];
    uint32_t s = warp_append(cnt, keep);
    if (keep) out[s] = v;
  }
}

// Pull records (plan lifetime, one per non-isolated hosted vertex, ascending):
// {v, deg(v), col[off[v]], col[off[v]+1]} — 16 bytes, the first two arcs of the
// row stored next to the vertex (0xFFFFFFFF past the end of a short row).  In
// R-MAT rows the lowest-ID neighbours (hubs) come first, so most unvisited
// vertices find a frontier parent within the first two arcs; the pull step
// then reads one coalesced 16-byte record per vertex instead of an offset pair
// plus a random 32-byte col_indices sector.  Unvisited lists hold record
// positions; the first pull of a run walks all records without a list.
constexpr int kPullK = 2;      // arcs held in the record
constexpr int kPullGroup = 8;  // lanes per vertex in the long-row pass
#ifndef MG_PV
#define MG_PV 8
#endif
constexpr int kPV = MG_PV;     // records per thread per iteration (loads in flight)
#ifndef MG_PULL_QX
#define MG_PULL_QX 0
#endif
#ifndef MG_PULL_BLOCK
#define MG_PULL_BLOCK 128  // 128: 7.08 ms over the bench sources, 256: 7.16
#endif
#ifndef MG_PULL_OCC
#define MG_PULL_OCC 4  // resident 256-thread CTAs' worth of warps per SM
#endif
constexpr uint32_t kPullBlock = MG_PULL_BLOCK;  // threads per CTA of the pull thread kernel
constexpr uint32_t kPullCtas = MG_PULL_OCC * 256 / kPullBlock;  // resident CTAs per SM
constexpr uint32_t kPullQ = kPullBlock * kPV + MG_PULL_QX;  // CTA queue capacity (>= one chunk)
#ifndef MG_PULL_MID
#define MG_PULL_MID 8
#endif
// arcs [kPullK, kPullK + kPullMid) of rows the record did not settle are tested
// by the thread stage itself (one offset load + one or two col sectors per row);
// only rows longer than kPullStart go on to the cooperative stage
constexpr int kPullMid = MG_PULL_MID;
static_assert(kPullMid == 8, "stage 1b takes arcs 2-9 from the 32-byte record extension");
// arc-0 frontier probe issued beside the visited probe (first pull of source
// 0: 297 -> 284 us under ncu; 8 bench sources 6.816 -> 6.789 ms, same box)
// experiment: the warp's visited-word window computed after the probes are
// issued (bench sources 6.91 -> 6.89 / 6.99 ms: noise), off
#ifndef MG_PULL_LATE_WINDOW
#define MG_PULL_LATE_WINDOW 0
#endif
#ifndef MG_PULL_EAGER_FB
#define MG_PULL_EAGER_FB 1
#endif
#ifndef MG_A1_LAZY
#define MG_A1_LAZY 1
#endif
#ifndef MG_MID_WAVE
#define MG_MID_WAVE 5
#endif
constexpr int kMidWave = MG_MID_WAVE;  // stage-1b probes in the first wave (3: 7.26 ms, 5: 7.17, 8: 7.31)
#ifndef MG_EXT2
#define MG_EXT2 1  // 7.36 -> 7.30 ms over the bench sources (source 8582448: 1.13 -> 1.08)
#endif
// MG_EXT2: a second extension sector (arcs 10..17), read only by rows that
// arcs 2..9 did not settle
constexpr int kExtSlots = MG_EXT2 ? 4 : 2;  // uint4 per record extension
constexpr uint32_t kPullStart = kPullK + kPullMid + (MG_EXT2 ? 8 : 0);
// (measured: stage 1b as its own kernel over the long-row queue, one row per
// thread and no CTA barrier, is slower — 8.93 -> 10.61 ms over the bench
// sources — the inline stage reuses the record already in registers)
constexpr bool kInline1b = kPullMid > 0;
#ifndef MG_MID_PARTS
#define MG_MID_PARTS 1
#endif
constexpr int kMidParts = MG_MID_PARTS;

__global__ void pull_records_kernel(GraphView g, const uint32_t* __restrict__ ni, uint32_t n,
                                    uint4* rec) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t v = ni[i];
    uint32_t b = g.off[v], d = g.off[v + 1] - b;
    rec[i] = make_uint4(v, d, d > 0 ? g.col[b] : kInfLabel, d > 1 ? g.col[b + 1] : kInfLabel);
  }
}

// record extensions (plan lifetime, same positions, one 32-byte sector each):
// arcs 2..9 of the row for stage 1b, so a row the record's two arcs did not
// settle tests its next 8 arcs from one sector, with no offset load and no
// col_indices sector (measured: {off, arc2-4} 7.90 -> 7.55 ms over the bench
// sources, {off, arc2-8} 7.27, {arc2-9} below)
__global__ void pull_ext_kernel(GraphView g, const uint32_t* __restrict__ ni, uint32_t n,
                                uint4* ext) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t v = ni[i];
    const uint32_t b = g.off[v], d = g.off[v + 1] - b;
    for (int q = 0; q < kExtSlots; ++q) {
      uint32_t a[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t arc = 2u + 4u * q + k;
        a[k] = d > arc ? g.col[b + arc] : kInfLabel;
      }
      ext[(uint64_t)kExtSlots * i + q] = make_uint4(a[0], a[1], a[2], a[3]);
    }
  }
}

__device__ __forceinline__ bool bit_set(const uint32_t* bits, uint32_t v) {
  return (__ldg(&bits[v >> 5]) >> (v & 31)) & 1u;
}

// Warp-level append of up to kPV items per lane into a CTA queue: ONE shared
// atomic per warp per call (the ballots of all kPV slots are summed first).
template <int K, int kCap>
__device__ __forceinline__ void warp_queue_append(BlockQueue<kCap>& q, const bool* pred,
                                                  const uint32_t* val) {
  unsigned m[K];
  uint32_t tot = 0;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    m[j] = __ballot_sync(0xffffffffu, pred[j]);
    tot += __popc(m[j]);
  }
  if (!tot) return;
  uint32_t base = 0;
  if (lane_id() == 0) base = atomicAdd(&q.n, tot);
  base = __shfl_sync(0xffffffffu, base, 0);
  const unsigned lt = (1u << lane_id()) - 1u;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (pred[j]) q.buf[base + __popc(m[j] & lt)] = val[j];
    base += __popc(m[j]);
  }
}

constexpr uint32_t kVisWin = 128;   // per-warp visited-word window of the pull thread kernel

// pull step, stage 1 (primitives.cpp:230-251): one thread per unvisited record
// tests the record's two arcs against the frontier bitmap; a hit labels the
// vertex, a short row without a hit stays unvisited, a longer row is tested on
// up to kPullStart arcs by stage 1b below and only then goes to the
// cooperative stage.  CTA queues with one shared atomic per warp and one
// global atomic per queue per 256*kPV records.  With emit_found == 0 (single
// partition) the discovered vertices are only counted (and their degrees
// summed into deg_out when non-null): the next superstep rebuilds the frontier
// list from the visited bitmap only if it pushes.
// kEmit: discoveries listed (several partitions); otherwise only counted and
// the found queue takes no shared memory
template <bool kEmit>
__global__ void __launch_bounds__(kPullBlock, kPullCtas)
    dobfs_pull_thread_kernel(GraphView g, const uint4* __restrict__ rec,
                             const uint4* __restrict__ ext, const uint32_t* __restrict__ ul,
                             uint32_t nul, uint32_t* labels, uint32_t* preds, uint32_t* vis,
                             const uint32_t* __restrict__ fb, uint32_t next_label, int mark_preds,
                             OwnerView ow, int emit_found, uint32_t* out, uint32_t* ul_out,
                             uint32_t* ul_out_cnt, uint32_t* longq, uint32_t* long_cnt,
                             Counters* ctr, unsigned long long* scanned_out,
                             unsigned long long* deg_out, DobfsDyn dyn, int list_clean = 0) {
  if (dyn.st) {
    list_clean = dyn.st->prev_physical;
    const uint32_t src = dyn.st->ul_src;
    nul = dyn.st->ul_len;
    ul = src == 2 ? nullptr : (src == 0 ? dyn.ub0 : dyn.ub1);
    ul_out = src == 0 ? dyn.ub1 : dyn.ub0;
    next_label = dyn.st->iter + 1;
    scanned_out = dyn.st->dir == 1 ? &ctr->edges : &ctr->u[3];
  }
  uint32_t scanned = 0, opened = 0, degs = 0;  // per-thread partials fit 32 bits
  uint32_t found_n = 0;
  // queues hold up to kPullQ entries and are flushed only when one could
  // overflow in the next chunk (one barrier per chunk otherwise)
  __shared__ BlockQueue<kEmit ? kPullQ : 1> q_found;
  __shared__ BlockQueue<kPullQ> q_keep, q_long;
  __shared__ uint32_t s_found;
  // per-warp window of visited words: a warp's 32 * kPV records are one
  // contiguous run of the (sorted) record array, so their vertices usually
  // fall in a few dozen bitmap words; discoveries are ORed into the window in
  // shared memory and each touched word gets ONE global atomicOr per chunk
  // (measured: also loading the window's words for the open tests, instead
  // of one visited probe per record, is slower — 8.28 -> 8.89 ms)
  __shared__ uint32_t s_nw[kPullBlock / 32][kVisWin];
  __shared__ uint32_t s_mid[kInline1b ? kPullBlock / 32 : 1][kInline1b ? 32 * kPV / kMidParts : 1];
  for (uint32_t i = threadIdx.x; i < (kPullBlock / 32) * kVisWin; i += blockDim.x) (&s_nw[0][0])[i] = 0u;
  uint32_t* nwin = s_nw[threadIdx.x >> 5];
  q_found.reset();
  q_keep.reset();
  q_long.reset();
  if (threadIdx.x == 0) s_found = 0;
  __syncthreads();
  const uint32_t chunk = kPullBlock * kPV;
  const bool clean = ul != nullptr && list_clean;
  for (uint32_t base = blockIdx.x * chunk; base < nul; base += gridDim.x * chunk) {
    uint32_t pos[kPV];
    uint4 r[kPV];
#pragma unroll
    for (int j = 0; j < kPV; ++j) {  // the warp's run: 32 consecutive entries per slot
      uint32_t i = base + (threadIdx.x >> 5) * (32 * kPV) + j * 32 + lane_id();
      pos[j] = i < nul ? (ul ? __ldg(&ul[i]) : i) : kInfLabel;
    }
#pragma unroll
    for (int j = 0; j < kPV; ++j)  // coalesced 16-byte records, kPV in flight, evict-first
      r[j] = pos[j] != kInfLabel ? __ldcs(&rec[pos[j]]) : make_uint4(0, 0, kInfLabel, kInfLabel);
#if !MG_PULL_LATE_WINDOW
    // the window: bitmap words [w0, w0 + span) hold every vertex of the run
    uint32_t vlo = 0xFFFFFFFFu, vhi = 0u;
#pragma unroll
    for (int j = 0; j < kPV; ++j)
      if (pos[j] != kInfLabel) {
        vlo = min(vlo, r[j].x);
        vhi = max(vhi, r[j].x);
      }
    vlo = __reduce_min_sync(0xffffffffu, vlo);
    vhi = __reduce_max_sync(0xffffffffu, vhi);
    const uint32_t w0 = vlo >> 5;
    const uint32_t span = vlo <= vhi ? (vhi >> 5) - w0 + 1 : 0u;
    const bool inwin = span <= kVisWin;  // warp-uniform
#endif
    bool open[kPV], h0[kPV], h1[kPV];
#pragma unroll
    for (int j = 0; j < kPV; ++j) {
      // a list written by the previous superstep's pull holds only unvisited
      // vertices (no push ran since): no visited probe
#if MG_PULL_EAGER_FB
      // the arc-0 frontier probe does not wait for the visited probe: both
      // depend only on the record (a visited vertex's probe is wasted)
      const bool valid = pos[j] != kInfLabel;
      const uint32_t vw = valid && !clean ? __ldcg(&vis[r[j].x >> 5]) : 0u;
      const uint32_t fw = valid ? __ldg(&fb[r[j].z >> 5]) : 0u;
      open[j] = valid && !((vw >> (r[j].x & 31)) & 1u);
      h0[j] = open[j] && ((fw >> (r[j].z & 31)) & 1u);
#else
      open[j] = pos[j] != kInfLabel &&
                (clean || !((__ldcg(&vis[r[j].x >> 5]) >> (r[j].x & 31)) & 1u));
      h0[j] = open[j] && bit_set(fb, r[j].z);
#endif
#if !MG_A1_LAZY
      h1[j] = open[j] && r[j].y > 1 && bit_set(fb, r[j].w);
#endif
    }
#if MG_A1_LAZY
#pragma unroll
    for (int j = 0; j < kPV; ++j) h1[j] = open[j] && !h0[j] && r[j].y > 1 && bit_set(fb, r[j].w);
#endif
#if MG_PULL_LATE_WINDOW
    // (after the probes are issued: the warp reductions no longer hold them back)
    // the window: bitmap words [w0, w0 + span) hold every vertex of the run
    uint32_t vlo = 0xFFFFFFFFu, vhi = 0u;
#pragma unroll
    for (int j = 0; j < kPV; ++j)
      if (pos[j] != kInfLabel) {
        vlo = min(vlo, r[j].x);
        vhi = max(vhi, r[j].x);
      }
    vlo = __reduce_min_sync(0xffffffffu, vlo);
    vhi = __reduce_max_sync(0xffffffffu, vhi);
    const uint32_t w0 = vlo >> 5;
    const uint32_t span = vlo <= vhi ? (vhi >> 5) - w0 + 1 : 0u;
    const bool inwin = span <= kVisWin;  // warp-uniform
#endif
    bool found[kPV], keep[kPV], lng[kPV];
    uint32_t vv[kPV];
#pragma unroll
    for (int j = 0; j < kPV; ++j) {
      const uint32_t v = r[j].x, d = r[j].y;
      vv[j] = v;
      const bool f = open[j] && (h0[j] || h1[j]);
      found[j] = f;
      keep[j] = open[j] && !f && d <= (uint32_t)kPullK;
      lng[j] = open[j] && !f && d > (uint32_t)kPullK;
      // counters without branches; one branch for the discovery's stores
      opened += open[j];
      found_n += f;
      degs += f ? d : 0u;
      scanned += f ? (h0[j] ? 1u : 2u) : (open[j] ? min(d, (uint32_t)kPullK) : 0u);
      if (f) {
        __stcs(&labels[v], next_label);
        if (mark_preds) preds[v] = ow.to_global(h0[j] ? r[j].z : r[j].w);
        if (inwin) atomicOr(&nwin[(v >> 5) - w0], 1u << (v & 31));
        else atomicOr(&vis[v >> 5], 1u << (v & 31));
      }
    }

    if constexpr (kEmit) warp_queue_append<kPV>(q_found, found, vv);
    warp_queue_append<kPV>(q_keep, keep, pos);
    if constexpr (!kInline1b) {
      warp_queue_append<kPV>(q_long, lng, pos);
    } else {
      // stage 1b: the warp compacts its unsettled rows and spreads them over
      // all 32 lanes; each lane tests arcs [kPullK, kPullStart) of one row
      // with independent loads, first hit in arc order wins (exact W)
      // (in kMidParts passes over the lane's records: a smaller shared list)
      uint32_t* lst = s_mid[threadIdx.x >> 5];
      const unsigned lt = (1u << lane_id()) - 1u;
#pragma unroll
      for (int part = 0; part < kMidParts; ++part) {
      uint32_t cnt = 0;
#pragma unroll
      for (int jj = 0; jj < kPV / kMidParts; ++jj) {
        const int j = part * (kPV / kMidParts) + jj;
        const unsigned m = __ballot_sync(0xffffffffu, lng[j]);
        if (lng[j]) lst[cnt + __popc(m & lt)] = pos[j];
        cnt += __popc(m);
      }
      __syncwarp();
      for (uint32_t t0 = 0; t0 < cnt; t0 += 32) {
        const uint32_t t = t0 + lane_id();
        const bool act = t < cnt;
        uint32_t p = act ? lst[t] : 0u;
        // the record again (L1/L2) and its 32-byte extension (arcs 2-9), both
        // addressed by the position: no offset load, no col_indices sector
        const uint4 rr = act ? rec[p] : make_uint4(0, 0, 0, 0);
        const uint4 ex = act ? __ldcs(&ext[(uint64_t)kExtSlots * p]) : make_uint4(0, 0, 0, 0);
        const uint4 ex2 = act ? __ldcs(&ext[(uint64_t)kExtSlots * p + 1]) : make_uint4(0, 0, 0, 0);
        uint32_t v = rr.x;
        const uint32_t d = rr.y;
        const uint32_t e = d < kPullStart ? d : kPullStart;
        const uint32_t wv[kPullMid] = {ex.x, ex.y, ex.z, ex.w, ex2.x, ex2.y, ex2.z, ex2.w};
        bool h[kPullMid];
        // two waves of frontier probes: arcs 2-6, then 7-9 only past a miss
        // (probes are L2 requests; most rows hit early)
#pragma unroll
        for (int k = 0; k < kMidWave; ++k) h[k] = act && kPullK + k < e && bit_set(fb, wv[k]);
        bool early = false;
#pragma unroll
        for (int k = 0; k < kMidWave; ++k) early |= h[k];
#pragma unroll
        for (int k = kMidWave; k < kPullMid; ++k)
          h[k] = act && !early && kPullK + k < e && bit_set(fb, wv[k]);
        int f = -1;
        uint32_t pw = 0;
#pragma unroll
        for (int k = kPullMid - 1; k >= 0; --k)
          if (h[k]) {
            f = k;
            pw = wv[k];
          }
#if MG_EXT2
        if (f < 0 && act && d > kPullK + kPullMid) {  // arcs 10..17 from the second sector
          const uint4 e3 = __ldcs(&ext[(uint64_t)kExtSlots * p + 2]);
          const uint4 e4 = __ldcs(&ext[(uint64_t)kExtSlots * p + 3]);
          const uint32_t w2[8] = {e3.x, e3.y, e3.z, e3.w, e4.x, e4.y, e4.z, e4.w};
          bool h2[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) h2[k] = kPullK + kPullMid + k < e && bit_set(fb, w2[k]);
#pragma unroll
          for (int k = 7; k >= 0; --k)
            if (h2[k]) {
              f = kPullMid + k;
              pw = w2[k];
            }
        }
#endif
        bool fnd = f >= 0;
        bool kp = act && !fnd && d <= kPullStart;
        bool lg = act && !fnd && d > kPullStart;
        scanned += fnd ? (uint32_t)(f + 1) : (act ? e - kPullK : 0u);
        found_n += fnd;
        degs += fnd ? d : 0u;
        if (fnd) {
          __stcs(&labels[v], next_label);
          if (mark_preds) preds[v] = ow.to_global(pw);
          if (inwin) atomicOr(&nwin[(v >> 5) - w0], 1u << (v & 31));
          else atomicOr(&vis[v >> 5], 1u << (v & 31));
        }
        if constexpr (kEmit) warp_queue_append<1>(q_found, &fnd, &v);
        warp_queue_append<1>(q_keep, &kp, &p);
        warp_queue_append<1>(q_long, &lg, &p);
      }
      __syncwarp();
      }
    }
    if (inwin) {  // one global atomicOr per word that gained a bit
      __syncwarp();
      for (uint32_t k = lane_id(); k < span; k += 32) {
        const uint32_t m = nwin[k];
        if (m) {
          atomicOr(&vis[w0 + k], m);
          nwin[k] = 0u;
        }
      }
    }
    __syncthreads();
    const bool last = base + gridDim.x * chunk >= nul;
    if (last || q_found.n > kPullQ - chunk || q_keep.n > kPullQ - chunk ||
        q_long.n > kPullQ - chunk) {  // CTA-uniform: read after the barrier
      if (threadIdx.x == 0) {
        q_found.base = q_found.n ? atomicAdd(&ctr->out_cnt, q_found.n) : 0u;
        q_keep.base = q_keep.n ? atomicAdd(ul_out_cnt, q_keep.n) : 0u;
        q_long.base = q_long.n ? atomicAdd(long_cnt, q_long.n) : 0u;
      }
      __syncthreads();
      for (uint32_t k = threadIdx.x; k < q_found.n; k += kPullBlock) out[q_found.base + k] = q_found.buf[k];
      for (uint32_t k = threadIdx.x; k < q_keep.n; k += kPullBlock) ul_out[q_keep.base + k] = q_keep.buf[k];
      for (uint32_t k = threadIdx.x; k < q_long.n; k += kPullBlock) longq[q_long.base + k] = q_long.buf[k];
      __syncthreads();
      if (threadIdx.x == 0) q_found.n = q_keep.n = q_long.n = 0;
      __syncthreads();
    }
  }
  if constexpr (!kEmit) {
    unsigned m = __reduce_add_sync(0xffffffffu, found_n);
    if (lane_id() == 0 && m) atomicAdd(&s_found, m);
    __syncthreads();
    if (threadIdx.x == 0 && s_found) atomicAdd(&ctr->out_cnt, s_found);
  }
  unsigned long long* const dst[3] = {scanned_out, &ctr->u[2], deg_out};
  const uint64_t val[3] = {scanned, opened, degs};
  block_add_u64<3>(dst, val);
}

// pull step, stage 2: rows longer than the record, 8 lanes per vertex from arc
// kPullK on; each round tests one 32-byte sector of col_indices and the first
// hit in arc order wins, so W equals the reference's sequential count.  Queue
// appends are CTA-aggregated like stage 1.
constexpr int kGroupIters = 4;  // vertices per group between CTA flushes
#ifndef MG_GROUP_SECTORS
#define MG_GROUP_SECTORS 4
#endif
constexpr int kGroupSectors = MG_GROUP_SECTORS;  // 8-arc sectors per group per round

__global__ void __launch_bounds__(256)
    dobfs_pull_group_kernel(GraphView g, const uint4* __restrict__ rec,
                            const uint32_t* __restrict__ longq, const uint32_t* long_cnt,
                            uint32_t* labels, uint32_t* preds, uint32_t* vis,
                            const uint32_t* __restrict__ fb, uint32_t next_label, int mark_preds,
                            OwnerView ow, int emit_found, uint32_t* out, uint32_t* ul_out,
                            uint32_t* ul_out_cnt, Counters* ctr,
                            unsigned long long* scanned_out, unsigned long long* deg_out,
                            DobfsDyn dyn, DobfsLoopEnd le = {}) {
  if (dyn.st) {
    ul_out = dyn.st->ul_src == 0 ? dyn.ub1 : dyn.ub0;
    next_label = dyn.st->iter + 1;
    scanned_out = dyn.st->dir == 1 ? &ctr->edges : &ctr->u[3];
  }
  __shared__ BlockQueue<256 / kPullGroup * kGroupIters> q_found, q_keep;
  unsigned long long degs = 0;
  __shared__ uint32_t s_found;
  const uint32_t nl = *long_cnt;
  // CTAs past the queue leave at once (an empty stage used to cost ~5 us);
  // with the superstep end folded in they only take their ticket
  if (blockIdx.x * (256 / kPullGroup * kGroupIters) >= nl) {
    if (le.st) dobfs_loop_end_last_cta(le, ctr);
    return;
  }
  const unsigned lane = threadIdx.x & 31u;
  const unsigned sub = lane & (kPullGroup - 1);
  const unsigned gbase = lane & ~(kPullGroup - 1);
  const unsigned gmask = ((1u << kPullGroup) - 1u) << gbase;
  unsigned long long scanned = 0;
  uint32_t found_n = 0;
  q_found.reset();
  q_keep.reset();
  if (threadIdx.x == 0) s_found = 0;
  __syncthreads();
  const uint32_t gpb = 256 / kPullGroup;  // groups per CTA
  const uint32_t per_cta = gpb * kGroupIters;
  for (uint32_t cbase = blockIdx.x * per_cta; cbase < nl; cbase += gridDim.x * per_cta) {
    for (int it = 0; it < kGroupIters; ++it) {
      const uint32_t i = cbase + it * gpb + threadIdx.x / kPullGroup;
      bool found = false, keep = false;
      uint32_t v = 0, pos = 0;
      uint4 r;
      if (i < nl) {
        pos = longq[i];
        r = rec[pos];
        v = r.x;
        const uint32_t row = g.off[v];
        const uint32_t b = row + kPullStart, e = row + r.y;
        keep = true;
        // the first round tests one sector (most rows hit early); later rounds
        // keep kGroupSectors sectors of the row in flight per group, since a
        // row that got this far is likely to be scanned to its end
        uint32_t span = kPullGroup;
        for (uint32_t k = b; k < e; k += span, span = kPullGroup * kGroupSectors) {
          uint32_t w[kGroupSectors];
          bool hit[kGroupSectors];
#pragma unroll
          for (int j = 0; j < kGroupSectors; ++j) {
            const uint32_t idx = k + j * kPullGroup + sub;
            const bool ok = idx < e && (j == 0 || span > kPullGroup);
            w[j] = ok ? __ldg(&g.col[idx]) : 0u;
            hit[j] = ok;
          }
#pragma unroll
          for (int j = 0; j < kGroupSectors; ++j) hit[j] = hit[j] && bit_set(fb, w[j]);
          int fj = -1;
          unsigned m = 0;
#pragma unroll
          for (int j = kGroupSectors - 1; j >= 0; --j) {  // lowest sector with a hit
            const unsigned mj = __ballot_sync(gmask, hit[j]) & gmask;
            if (mj) {
              fj = j;
              m = mj;
            }
          }
          if (fj >= 0) {
            const unsigned first = __ffs(m) - 1 - gbase;
            uint32_t sel = w[0];
#pragma unroll
            for (int j = 1; j < kGroupSectors; ++j)
              if (j == fj) sel = w[j];
            const uint32_t pw = __shfl_sync(gmask, sel, gbase + first);
            if (sub == 0) {
              // the rounds before this one already counted their spans
              scanned += fj * kPullGroup + first + 1;
              found = true;
              keep = false;
              labels[v] = next_label;
              atomicOr(&vis[v >> 5], 1u << (v & 31));
              if (mark_preds) preds[v] = ow.to_global(pw);
              ++found_n;
              degs += r.y;
            }
            break;
          }
          if (sub == 0) scanned += (e - k < span) ? (e - k) : span;
        }
        if (sub != 0) keep = false;
      }
      if (emit_found) q_found.push(found, v);
      q_keep.push(keep, pos);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      q_found.base = q_found.n ? atomicAdd(&ctr->out_cnt, q_found.n) : 0u;
      q_keep.base = q_keep.n ? atomicAdd(ul_out_cnt, q_keep.n) : 0u;
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < q_found.n; k += 256) out[q_found.base + k] = q_found.buf[k];
    for (uint32_t k = threadIdx.x; k < q_keep.n; k += 256) ul_out[q_keep.base + k] = q_keep.buf[k];
    __syncthreads();
    if (threadIdx.x == 0) q_found.n = q_keep.n = 0;
    __syncthreads();
  }
  if (!emit_found) {
    unsigned m = __reduce_add_sync(0xffffffffu, found_n);
    if (lane_id() == 0 && m) atomicAdd(&s_found, m);
    __syncthreads();
    if (threadIdx.x == 0 && s_found) atomicAdd(&ctr->out_cnt, s_found);
  }
  unsigned long long* const dst[2] = {scanned_out, deg_out};
  const uint64_t val[2] = {scanned, degs};
  block_add_u64<2>(dst, val);
  if (le.st) dobfs_loop_end_last_cta(le, ctr);
}

// frontier list = vis & ~prev (the vertices discovered in the previous
// superstep), rebuilt for a push step that follows a list-free pull step:
// per round 256 words, a CTA scan of their popcounts, one atomic per round
__global__ void __launch_bounds__(256)
    bitmap_diff_list_kernel(const uint32_t* __restrict__ vis, uint32_t* prev, uint32_t nw,
                            uint32_t* out, uint32_t* cnt, int set_prev = 0,
                            const DobfsLoop* st = nullptr, uint32_t* labels = nullptr,
                            uint32_t level = 0, const unsigned long long* need_total = nullptr,
                            unsigned long long need_min = 0) {
  // after a host-loop push: list only when it ran dense (DobfsDev::dense)
  if (need_total && *need_total < need_min) return;
  // device-driven loop, superstep 0: the list is the source, seeded by the
  // init kernel together with prev (no 8 MB bitmap pass for one vertex)
  if (st && st->iter == 0) return;
  __shared__ uint32_t s_warp[8];
  __shared__ uint32_t s_base;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  for (uint32_t base = blockIdx.x * 256; base < nw; base += gridDim.x * 256) {
    const uint32_t i = base + threadIdx.x;
    uint32_t d = 0;
    if (i < nw) {
      const uint32_t a = __ldg(&vis[i]);
      d = a & ~prev[i];
      if (set_prev) prev[i] = a;  // prev = vis in the same pass (push step follows)
    }
    // CTA exclusive scan of the popcounts: warp shuffles, then the 8 warp sums
    const uint32_t c = __popc(d);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t run = 0;
      for (int k = 0; k < 8; ++k) {
        const uint32_t t = s_warp[k];
        s_warp[k] = run;
        run += t;
      }
      s_base = run ? atomicAdd(cnt, run) : 0u;
    }
    __syncthreads();
    const uint32_t o = s_base + s_warp[warp] + x - c;
    // the warp writes word by word (the non-empty ones): lane l stores bit l,
    // so each store instruction fills consecutive list entries and one
    // 128-byte line of labels (a thread walking its own word would put 32
    // lanes on 32 different lines per store)
    const unsigned lt = (1u << lane) - 1u;
    for (unsigned m = __ballot_sync(0xffffffffu, d != 0); m; m &= m - 1) {
      const int src = __ffs(m) - 1;
      const uint32_t dj = __shfl_sync(0xffffffffu, d, src);
      const uint32_t oj = __shfl_sync(0xffffffffu, o, src);
      if ((dj >> lane) & 1u) {
        const uint32_t v = (base + warp * 32 + src) * 32 + lane;
        out[oj + __popc(dj & lt)] = v;
        if (labels) labels[v] = level;  // a dense push's discoveries (DobfsDev::red)
      }
    }
    __syncthreads();
  }
}

// u[0] = the worker's unvisited-list length after this superstep (the pull's
// kept count, or unchanged), u[1] = Σdeg of its next frontier
__global__ void dobfs_share_kernel(Counters* ctr, int pulled, uint32_t ul_keep) {
  ctr->u[0] = pulled ? ctr->misc : ul_keep;
  ctr->u[1] = ctr->next_deg;
}

// ---------------------------------------------------------------------------
// Device-driven DOBFS (single partition, exact-cost direction, max policy):
// the whole superstep loop is ONE CUDA graph — a WHILE node whose body is
//   decide  (the reference direction rule, primitives.cpp:131-154, and the
//            exact-cost physical choice, evaluated on the device in the same
//            double arithmetic as the host path)
//   IF pull { frontier_diff, pull_thread, pull_group }
//   IF push { frontier list from vis & ~prev, prev = vis, degree / scan /
//             tiles / expand, degree sum of the discoveries }
//   end     (history, loop state, counters cleared, loop condition)
// so no superstep waits for the host.  Results and statistics equal the
// host-driven path's (tests/test_gpu_parity.py::test_dobfs_graph_*).

struct DobfsPrim : PrimBase {
  uint32_t source;
  double do_a, do_b;
  bool mark_preds;
  // host-side mirror of the per-worker state (identical on every worker)
  uint64_t visited = 1;
  int dir = 0;
  bool switched_once = false;
  std::vector<int> dir_log;
  // unvisited-list bookkeeping per worker: which aux buffer holds it, length
  std::vector<int> ul_src;  // -1: the plan's non-isolated list
  std::vector<uint32_t> ul_len;
  bool exact_cost = false;
  uint64_t physical_pull_steps = 0;
  static constexpr bool keeps_dobfs_labels = true;
  DobfsPrim(uint32_t s, double a, double b, bool m, bool exact, uint32_t nparts)
      : source(s), do_a(a), do_b(b), mark_preds(m), exact_cost(exact) {
    reports_deg = exact;  // n = 1: by the pull / push kernels; n > 1: by split + merge
    name = "dobfs";
    nva = m ? 1 : 0;
    communication = MG_COMM_BROADCAST;
  }
  static uint64_t words(uint32_t nv) { return (nv + 31) / 32 + 1; }
  // several partitions: a superstep's discoveries go to the peers as IDs, or as
  // the discovery bitmap vis & ~vis_prev once they number >= |V|/32 (engine.cuh
  // DenseView); the inbox then needs room for only |V|/32 records.  Predecessors
  // travel as associates, so mark_preds keeps the record form.
  uint64_t inbox_bound(Plan& P, uint32_t src, uint32_t dst, int comm) const {
    if (!mark_preds && comm == MG_COMM_BROADCAST) return words(P.nv);
    return PrimBase::inbox_bound(P, src, dst, comm);
  }
  DenseView dense_view(Ctx& c) const {
    if (mark_preds) return {};
    Worker& w = *c.w;
    DenseView d;
    d.kind = 1;
    d.cur = w.su32[2].ptr;
    d.prev = w.aux[4].ptr;
    d.vis = w.su32[2].ptr;
    d.words = (uint32_t)words(w.nv);
    d.threshold = d.words;
    return d;
  }
  static void ensure_nonisolated(Worker& w) {
    if (w.nonisolated_ready) return;
    uint32_t nh = (uint32_t)w.hosted_host.size();
    w.nonisolated.alloc(nh ? nh : 1);
    DevArray<uint32_t> cnt;
    cnt.alloc(1);
    MGB_CUDA(cudaMemsetAsync(cnt.ptr, 0, 4, w.stream));
    if (nh)
      MGB_LAUNCH(select_nonisolated_kernel, grid_for(nh, 256, 4096), 256, 0, w.stream,
                 w.hosted.ptr, nh, w.off.ptr, w.nonisolated.ptr, cnt.ptr);
    uint32_t k = 0;
    MGB_CUDA(cudaMemcpyAsync(&k, cnt.ptr, 4, cudaMemcpyDeviceToHost, w.stream));
    MGB_CUDA(cudaStreamSynchronize(w.stream));
    cnt.free_();
    // ascending order keeps the pull step's record reads coalesced
    std::vector<uint32_t> h(k);
    MGB_CUDA(cudaMemcpy(h.data(), w.nonisolated.ptr, 4ull * k, cudaMemcpyDeviceToHost));
    std::sort(h.begin(), h.end());
    MGB_CUDA(cudaMemcpy(w.nonisolated.ptr, h.data(), 4ull * k, cudaMemcpyHostToDevice));
    w.n_nonisolated = k;
    w.pull_rec.alloc(k ? k : 1);
    w.pull_ext.alloc((uint64_t)kExtSlots * (k ? k : 1));
    if (k) {
      MGB_LAUNCH(pull_records_kernel, grid_for(k, 256, num_sms() * 16), 256, 0, w.stream, w.graph(),
                 w.nonisolated.ptr, k, w.pull_rec.ptr);
      MGB_LAUNCH(pull_ext_kernel, grid_for(k, 256, num_sms() * 16), 256, 0, w.stream, w.graph(),
                 w.nonisolated.ptr, k, w.pull_ext.ptr);
    }
    MGB_CUDA(cudaStreamSynchronize(w.stream));
    w.nonisolated_ready = true;
  }
  void init(Ctx& c) {  // primitives.cpp:185-195
    Worker& w = *c.w;
    ensure_nonisolated(w);  // plan-lifetime precomputation, outside the timed region on reuse
    const uint64_t k = w.n_nonisolated ? w.n_nonisolated : 1;
    // unvisited lists (ping-pong) and the long-row queue: plan-lifetime buffers
    for (int i = 0; i < 3; ++i)
      if (w.ul_buf[i].n < k + 1 || !w.ul_buf[i].ptr) w.ul_buf[i].alloc(k + 1);
    if (w.su32[2].n < words(w.nv) || !w.su32[2].ptr) w.dobfs_labels_ok = false;
    dobfs_labels_begin(w, words(w.nv));           // labels (fill or fixup)
    fill(w.su32[2], words(w.nv), 0, w.stream);    // visited bitmap
    fill(w.aux[4], words(w.nv), 0, w.stream);     // visited as of the previous superstep
    if (w.su32[3].n < words(w.nv) || !w.su32[3].ptr) w.su32[3].alloc(words(w.nv));  // frontier
    if (w.aux[2].n < 4 || !w.aux[2].ptr) w.aux[2].alloc(4);
    if (mark_preds) fill(w.su32[1], w.nv, 0xFF, w.stream);
    MGB_LAUNCH(set_one_kernel<uint32_t>, 1, 1, 0, w.stream, w.su32[0].ptr, source, 0u);
    uint32_t sw = 1u << (source & 31);
    set_bit_host(w, source, sw);
    if (c.P->owner_host[source] == w.p) c.push_initial({source});
    if (ul_src.empty()) {
      ul_src.assign(c.P->n, -1);
      ul_len.assign(c.P->n, 0);
      list_free.assign(c.P->n, false);
    }
    ul_src[w.p] = -1;
    ul_len[w.p] = w.n_nonisolated;
    list_free[w.p] = false;
  }
  static void set_bit_host(Worker& w, uint32_t v, uint32_t bit) {
    MGB_LAUNCH(or_word_kernel, 1, 1, 0, w.stream, w.su32[2].ptr + (v >> 5), bit);
  }
  DobfsDev dev(Ctx& c) {
    Worker& w = *c.w;
    return {w.su32[0].ptr, w.su32[1].ptr, w.su32[2].ptr, w.su32[3].ptr, c.owner_view(),
            (uint32_t)c.iter, mark_preds ? 1 : 0};
  }
  void body(Ctx& c) {  // primitives.cpp:197-253
    Worker& w = *c.w;
    collect_profile(c);
    if (pending_ul_[w.p]) {  // length of the list compacted by the last pull step
      ul_len[w.p] = w.host_ctr->misc;
      pending_ul_[w.p] = false;
    }
    if (c.worker() == c.P->local_workers.front()) {
      // decision on global quantities; identical on every worker
      if (c.iter >= 1) {
        if (c.prev) visited += c.prev->reports[c.worker()].next_frontier;
        double fv = c.P->nv > 0 ? (double)c.in_count * (double)c.P->ne / (double)c.P->nv : 0.0;
        double bv = visited > 0 ? (double)(c.P->nv - visited) * (double)c.P->nv / (double)visited
                                : 0.0;
        int next;
        if (dir == 0) next = (!switched_once && fv > bv * do_a) ? 1 : 0;
        else next = fv < bv * do_b ? 0 : 1;
        if (next == 1 && dir == 0) switched_once = true;
        dir = next;
      }
      dir_log.push_back(dir);
    }
    const uint64_t nw = words(w.nv);
    pulled_ = false;
    const bool prev_pull = prev_pull_[w.p];  // the unvisited list is clean
    prev_pull_[w.p] = false;                 // set again below if this step pulls
    if (list_free[w.p]) {
      // the previous (pull) superstep only counted its discoveries: rebuild the
      // input frontier list from the visited bitmap (vis & ~vis_prev); a pull
      // step needs no list, only the bitmap
      list_free[w.p] = false;
      if (dir == 0) {  // this superstep advances (or sizes) from the list
        uint32_t* cnt = w.aux[2].ptr + 2;
        MGB_CUDA(cudaMemsetAsync(cnt, 0, 4, w.stream));
        w.input.ensure(c.in_count, w.stream);
        MGB_LAUNCH(bitmap_diff_list_kernel, grid_for(nw, 256, num_sms() * 8), 256, 0, w.stream,
                   w.su32[2].ptr, w.aux[4].ptr, (uint32_t)nw, w.input.ptr, cnt);
      }
    }
    // extension (mg_config.dobfs_exact_cost, single partition): a logically
    // forward superstep whose exact edge count Σdeg(Q) dwarfs the unvisited
    // list is computed by the pull kernels instead.  For one partition both
    // produce the same set (the unvisited neighbours of Q); W is reported as
    // the reference counts the forward step (E:66), i.e. Σdeg(Q).
    bool physical_pull = dir == 1;
    uint64_t logical_w = 0;
    if (dir == 0 && exact_cost && c.P->n == 1 && c.in_count && c.iter > 0) {
      logical_w = c.degsum();
      physical_pull = (double)logical_w > pull_ratio() * ul_len[w.p];
      if (physical_pull) ++physical_pull_steps;
    } else if (dir == 0 && exact_cost && c.P->n > 1 && c.iter > 0) {
      // several partitions: every worker must take the same physical direction
      // (a pull covers only the hosted vertices, a push only the hosted
      // frontier), so the test uses the global sums every worker reported
      // last superstep: u[1] = Σdeg of its next frontier, u[0] = its list length
      uint64_t gw = 0, gul = 0;
      for (const WorkerReport& r : c.prev->reports) {
        gw += r.u[1];
        gul += r.u[0];
      }
      physical_pull = (double)gw > pull_ratio() * gul;
      logical_w = c.in_degsum == kUnknownDeg ? c.degsum() : c.in_degsum;
      if (physical_pull) ++physical_pull_steps;
    }
    if (!physical_pull) {
      MGB_CUDA(cudaMemcpyAsync(w.aux[4].ptr, w.su32[2].ptr, 4 * nw, cudaMemcpyDeviceToDevice,
                               w.stream));
      if (c.P->profile) MGB_CUDA(cudaEventRecord(w.ev_k0, w.stream));
      if (c.P->n == 1 && !mark_preds && c.fused && dense_push_arcs() && c.in_count) {
        // dense when the advance examines >= dense_push_arcs() arcs (its scan
        // total, read on the device): visited bits only, out_cnt stays 0, then
        // labels and the output list from vis & ~prev
        const uint32_t nb = (c.in_count + kLbBlock - 1) / kLbBlock;  // lb_advance's total slot
        if (w.lb_bsum.n < nb + 1ull) w.lb_bsum.alloc(nb + 1ull);
        DobfsDev f = dev(c);
        f.red_total = w.lb_bsum.ptr + nb;
        f.red_min = dense_push_arcs();
        c.pipeline(f, w.nv);
        MGB_LAUNCH(bitmap_diff_list_kernel, grid_for(nw, 256, num_sms() * 8), 256, 0, w.stream,
                   w.su32[2].ptr, w.aux[4].ptr, (uint32_t)nw, w.output.ptr, &c.ctr()->out_cnt, 0,
                   (const DobfsLoop*)nullptr, w.su32[0].ptr, (uint32_t)c.iter + 1, f.red_total,
                   f.red_min);
      } else {
        c.pipeline(dev(c), w.nv);
      }
      if (c.P->profile) {
        MGB_CUDA(cudaEventRecord(w.ev_k1, w.stream));
        prof_pending_[w.p] = true;
        prof_kind_[w.p] = 1;
        prof_nul_[w.p] = c.in_count;
      }
      if (reports_deg && !c.want_deg && c.P->n == 1)
        MGB_LAUNCH(degsum_dev_kernel, num_sms() * 4, 256, 0, w.stream, w.graph(), w.output.ptr,
                   &c.ctr()->out_cnt, &c.ctr()->next_deg);
      return;
    }
    pulled_ = true;
    // backward: the (global) input frontier is exactly what became visited in
    // the previous superstep, so its bitmap is vis & ~vis_prev — one streaming
    // pass over |V|/32 words instead of an atomic per frontier vertex
    uint32_t* cnts = w.aux[2].ptr;     // [1] long-row queue length (zeroed below)
    MGB_LAUNCH(frontier_diff_kernel, grid_for(nw, 256, num_sms() * 8), 256, 0, w.stream,
               w.su32[2].ptr, w.aux[4].ptr, w.su32[3].ptr, (uint32_t)nw, cnts,
               dir == 0 ? &c.ctr()->edges : nullptr, (unsigned long long)logical_w);
    const int src = ul_src[w.p];
    const uint32_t* ul = src < 0 ? nullptr : w.ul_buf[src].ptr;  // null: every record
    const int dst = src == 0 ? 1 : 0;
    const uint32_t nul = ul_len[w.p];
    uint32_t* ulcnt = &c.ctr()->misc;  // reported with the superstep's counters
    // one partition under the max policy: discoveries are counted, not listed
    // (the next superstep rebuilds a list from the bitmap only if it pushes)
    const bool emit = c.P->n > 1 || c.want_deg;
    if (emit) c.ensure_output(nul);
    const uint32_t next_label = (uint32_t)c.iter + 1;
    if (c.P->profile) {
      MGB_CUDA(cudaEventRecord(w.ev_k0, w.stream));
      prof_nul_[w.p] = nul;
      prof_kind_[w.p] = dir == 1 ? 0 : 2;  // 2: forward superstep run as a pull
    }
    // examined arcs: the reference's W in a backward step; a scratch counter
    // when a forward step runs physically as a pull (W = Σdeg(Q) then)
    unsigned long long* scanned = dir == 1 ? &c.ctr()->edges : &c.ctr()->u[3];
    // exact-cost runs report Σdeg of the next frontier so the next superstep's
    // cost test needs no extra host round trip
    unsigned long long* deg_out =
        reports_deg && !c.want_deg && c.P->n == 1 ? &c.ctr()->next_deg : nullptr;
    if (nul) {
      auto* kern = emit ? dobfs_pull_thread_kernel<true> : dobfs_pull_thread_kernel<false>;
      MGB_LAUNCH(kern, grid_for(nul, kPullBlock * kPV, num_sms() * kPullCtas), kPullBlock, 0,
                 w.stream, w.graph(), w.pull_rec.ptr, w.pull_ext.ptr, ul, nul, w.su32[0].ptr,
                 w.su32[1].ptr, w.su32[2].ptr,
                 w.su32[3].ptr, next_label, mark_preds ? 1 : 0, c.owner_view(), emit ? 1 : 0,
                 w.output.ptr, w.ul_buf[dst].ptr, ulcnt, w.ul_buf[2].ptr, cnts + 1, c.ctr(),
                 scanned, deg_out, DobfsDyn{nullptr, nullptr, nullptr}, prev_pull ? 1 : 0);
      uint32_t* gq = w.ul_buf[2].ptr;  // cooperative-stage input
      uint32_t* gq_cnt = cnts + 1;
      MGB_LAUNCH(dobfs_pull_group_kernel, num_sms() * 8, 256, 0, w.stream, w.graph(),
                 w.pull_rec.ptr, gq, gq_cnt, w.su32[0].ptr, w.su32[1].ptr,
                 w.su32[2].ptr, w.su32[3].ptr, next_label, mark_preds ? 1 : 0, c.owner_view(),
                 emit ? 1 : 0, w.output.ptr, w.ul_buf[dst].ptr, ulcnt, c.ctr(), scanned, deg_out,
                 DobfsDyn{nullptr, nullptr, nullptr});
    }
    list_free[w.p] = !emit;
    prev_pull_[w.p] = true;
    if (c.P->profile) {
      MGB_CUDA(cudaEventRecord(w.ev_k1, w.stream));
      prof_pending_[w.p] = true;
    }
    pending_ul_[w.p] = true;  // new length arrives with this superstep's report
    ul_src[w.p] = dst;
  }
  // Pull-step timing + algorithmic bytes (SURVEY §8(d) DOBFS term, per launch
  // pair): unvisited list 4 B/entry, row offsets 8 B per opened vertex, 4 B per
  // examined arc, label + output 8 B per discovery, 4 B per kept entry.  The
  // visited / frontier bitmaps are L2-resident and not counted.  Read after the
  // superstep's report synchronised the stream.
  void collect_profile(Ctx& c) {
    Worker& w = *c.w;
    if (!prof_pending_[w.p]) return;
    prof_pending_[w.p] = false;
    float ms = 0;
    MGB_CUDA(cudaEventElapsedTime(&ms, w.ev_k0, w.ev_k1));
    const Counters& h = *w.host_ctr;
    if (prof_kind_[w.p] == 1) {
      // push advance: frontier IDs 4 B + row offsets 8 B per frontier vertex,
      // 4 B per examined arc, label + output 8 B per discovery
      double bytes = 12.0 * prof_nul_[w.p] + 4.0 * (double)h.edges + 8.0 * (double)h.out_cnt;
      c.P->prof2_ms += ms;
      c.P->prof2_bytes += bytes;
      c.P->prof2_launches += 1;
      return;
    }
    // arcs the pull kernels examined: W of a backward superstep; in a forward
    // superstep run as a pull W is the logical push count, the scan sits in u[3]
    const double examined = prof_kind_[w.p] == 0 ? (double)h.edges : (double)h.u[3];
    double bytes = 4.0 * prof_nul_[w.p] + 8.0 * (double)h.u[2] + 4.0 * examined +
                   8.0 * (double)h.out_cnt + 4.0 * (double)h.misc;
    c.P->prof_ms += ms;
    c.P->prof_bytes += bytes;
    c.P->prof_launches += 1;
  }
  std::vector<int> prof_kind_ = std::vector<int>(kMaxWorkers, 0);
  void finalize(Ctx& c, const GlobalView&) {
    collect_profile(c);
    dobfs_labels_end(*c.w, words(c.w->nv));
  }
  // several partitions with the exact-cost test: share this worker's list
  // length and next-frontier degree sum through the report (u[0], u[1])
  bool pulled_ = false;
  void after_merge(Ctx& c) {
    if (!(exact_cost && c.P->n > 1)) return;
    MGB_LAUNCH(dobfs_share_kernel, 1, 1, 0, c.w->stream, c.ctr(), pulled_ ? 1 : 0,
               ul_len[c.w->p]);
  }
  // several processes (one partition per rank, device fabric): the whole
  // superstep loop as one CUDA graph per rank (DobfsMpGraphRunner below)
  bool device_loop(Plan& P, std::vector<Ctx>& ctx, RunState& rs, const mg_config& cfg,
                   DeviceLoopOut& o);
  std::vector<bool> pending_ul_ = std::vector<bool>(kMaxWorkers, false);
  std::vector<bool> prev_pull_ = std::vector<bool>(kMaxWorkers, false);
  std::vector<bool> list_free;  // per worker: last pull step counted, did not list
  std::vector<bool> prof_pending_ = std::vector<bool>(kMaxWorkers, false);
  std::vector<uint32_t> prof_nul_ = std::vector<uint32_t>(kMaxWorkers, 0);
};

// one graph per (worker, mark_preds), built on first use
struct DobfsGraph {
  cudaGraphExec_t exec;
  uint32_t n_pull, n_push;  // kernels in each branch (launch accounting)
};

struct DobfsGraphRun {
  std::vector<int> dir_log;
  std::vector<uint64_t> edges, out;
  uint64_t launches = 0;
  bool complete = true;
};

class DobfsGraphRunner {
 public:
  static bool eligible(const Plan& P, const mg_config& c) {
    // The graph removes the per-superstep host round trip (~4 us each): 7-10%
    // less device time on RMAT-18..22; on RMAT-26 1.6% (8.18 -> 8.05 ms over
    // the bench sources, tools/gpu/graph_vs_host.sh, after the round-2 pull
    // changes; the host loop had been 1.3% faster before them).
    // MG_GRAPH_LOOP=0 or MG_NO_GRAPH (any value) forces the host loop.
    const char* force = getenv("MG_GRAPH_LOOP");
    const bool off = getenv("MG_NO_GRAPH") != nullptr || (force && force[0] == '0');
    const bool fused = c.fused == MG_FUSED_ON || (c.fused == MG_FUSED_AUTO &&
                                                  c.policy == MG_POLICY_FUSED);
    return !off && P.n == 1 && P.dup == MG_DUP_ALL && c.dobfs_exact_cost && !P.profile &&
           c.policy == MG_POLICY_MAX && fused && !c.drop_enabled && c.hard_cap_bytes == 0;
  }

  // runs one DOBFS (or the BFS schedule with do_a = inf); fills P.last & co.
  static DobfsGraphRun run(Plan& P, uint32_t source, double do_a, double do_b, bool mark_preds,
                           const mg_config& cfg, const char* name, int comm) {
    auto t0 = std::chrono::steady_clock::now();
    Worker& w = *P.workers[P.local_workers.front()];
    DeviceGuard dg(w.dev);
    DobfsPrim::ensure_nonisolated(w);
    ensure_buffers(w);
    const DobfsGraph G = graph(w, mark_preds);
    const uint64_t nw = (w.nv + 31) / 32 + 1;
    DobfsLoop h{};
    h.nv_d = (double)P.nv;
    h.ne_d = (double)P.ne;
    h.do_a = do_a;
    h.do_b = do_b;
    h.nv = P.nv;
    h.source = source;
    h.max_supersteps = (uint32_t)(cfg.max_supersteps < kLoopHist ? cfg.max_supersteps : kLoopHist);
    h.exact = 1;
    h.pull_ratio = pull_ratio();
    h.n_nonisolated = w.n_nonisolated;
    DobfsLoop* lh = static_cast<DobfsLoop*>(w.loop_host);
    DobfsHist* hh = static_cast<DobfsHist*>(w.loop_hist_host);
    *lh = h;
    MGB_CUDA(cudaEventRecord(w.ev_start, w.stream));
    MGB_CUDA(cudaMemcpyAsync(w.loop_state.ptr, w.loop_host, sizeof(DobfsLoop),
                             cudaMemcpyHostToDevice, w.stream));
    MGB_CUDA(cudaMemsetAsync(w.ctr.ptr, 0, sizeof(Counters), w.stream));
    dobfs_labels_begin(w, nw);                                              // labels
    MGB_CUDA(cudaMemsetAsync(w.su32[2].ptr, 0, 4 * nw, w.stream));          // visited
    MGB_CUDA(cudaMemsetAsync(w.aux[4].ptr, 0, 4 * nw, w.stream));           // visited (prev)
    if (mark_preds) MGB_CUDA(cudaMemsetAsync(w.su32[1].ptr, 0xFF, 4ull * w.nv, w.stream));
    MGB_LAUNCH(dobfs_loop_init_kernel, 1, 1, 0, w.stream,
               reinterpret_cast<DobfsLoop*>(w.loop_state.ptr),
               reinterpret_cast<DobfsHist*>(w.loop_hist.ptr), w.su32[0].ptr, w.su32[2].ptr,
               w.aux[4].ptr, w.loop_front[0].ptr);
    MGB_CUDA(cudaGraphLaunch(G.exec, w.stream));
    dobfs_labels_end(w, nw);
    MGB_CUDA(cudaEventRecord(w.ev_end, w.stream));
    MGB_CUDA(cudaMemcpyAsync(w.loop_host, w.loop_state.ptr, sizeof(DobfsLoop),
                             cudaMemcpyDeviceToHost, w.stream));
    MGB_CUDA(cudaStreamSynchronize(w.stream));
    const uint32_t S = lh->iter;
    w.dobfs_labels_ok = true;  // labels = this run's result (fixup done)
    MGB_CUDA(cudaMemcpy(hh, w.loop_hist.ptr, sizeof(DobfsHist) * S, cudaMemcpyDeviceToHost));
    DobfsGraphRun r;
    uint64_t W = 0, launches = 2;  // init kernel + graph
    for (uint32_t t = 0; t < S; ++t) {
      const DobfsHist& e = hh[t];
      r.dir_log.push_back((int)e.dir);
      r.edges.push_back(e.edges);
      r.out.push_back(e.out);
      W += e.edges;
      launches += e.physical ? G.n_pull : G.n_push;  // the branch (its last kernel ends the superstep)
    }
    r.launches = launches;
    const bool hit_cap = S >= kLoopHist && cfg.max_supersteps > kLoopHist && S && r.out.back();
    r.complete = !hit_cap;
    float ms = 0;
    cudaEventElapsedTime(&ms, w.ev_start, w.ev_end);
    // statistics in the engine's shapes (run_primitive)
    mg_stats& st = P.last;
    st = mg_stats{};
    st.n = 1;
    st.stop_reason = (S && r.out.back() == 0) ? MG_STOP_FRONTIERS_EMPTY : MG_STOP_MAX_SUPERSTEPS;
    st.communication = comm;
    st.policy = cfg.policy;
    st.supersteps = S;
    st.edges_examined = W;
    st.wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    st.device_ms = ms;
    st.gpu_launches = launches;
    st.device_loop = 1;
    P.h_matrix.assign(1, std::vector<uint64_t>(1, 0));
    P.h_per_iter.assign(S, std::vector<uint64_t>(1, 0));
    P.out_per_iter = r.out;
    P.edges_per_iter = r.edges;
    P.combine_per_iter.assign(S, 0);
    collect_buffer_stats(P);
    g_launches.fetch_add(launches, std::memory_order_relaxed);
    (void)name;
    return r;
  }

 private:
  // every device pointer a captured graph holds; a change (a buffer another
  // primitive regrew) forces a re-capture
  static std::vector<const void*> pointers(const Worker& w) {
    return {w.su32[0].ptr, w.su32[1].ptr, w.su32[2].ptr, w.su32[3].ptr, w.aux[2].ptr,
            w.aux[4].ptr, w.ul_buf[0].ptr, w.ul_buf[1].ptr, w.ul_buf[2].ptr, w.pull_rec.ptr, w.pull_ext.ptr,
            w.off.ptr, w.col.ptr, w.owner.ptr, w.ctr.ptr, w.loop_state.ptr, w.loop_hist.ptr,
            w.loop_front[0].ptr, w.loop_front[1].ptr, w.loop_lb_row.ptr, w.loop_lb_pref.ptr,
            w.loop_lb_bsum.ptr, w.loop_total.ptr, w.loop_tiles.ptr};
  }
  static void ensure_buffers(Worker& w) {
    const uint64_t nw0 = (w.nv + 31) / 32 + 1;
    if (w.su32[0].n < w.nv || !w.su32[0].ptr) w.su32[0].alloc(w.nv ? w.nv : 1);  // labels
    if (w.su32[1].n < w.nv || !w.su32[1].ptr) w.su32[1].alloc(w.nv ? w.nv : 1);  // preds
    if (w.su32[2].n < nw0 || !w.su32[2].ptr) w.su32[2].alloc(nw0);               // visited
    if (w.su32[3].n < nw0 || !w.su32[3].ptr) w.su32[3].alloc(nw0);               // frontier
    if (w.aux[4].n < nw0 || !w.aux[4].ptr) w.aux[4].alloc(nw0);                  // prev
    if (w.aux[2].n < 4 || !w.aux[2].ptr) w.aux[2].alloc(4);
    if (w.loop_state.ptr) return;
    const uint64_t nw = (w.nv + 31) / 32 + 1;
    const uint64_t k = w.n_nonisolated ? w.n_nonisolated : 1;
    w.loop_state.alloc(sizeof(DobfsLoop));
    w.loop_hist.alloc(sizeof(DobfsHist) * kLoopHist);
    MGB_CUDA(cudaMallocHost(&w.loop_host, sizeof(DobfsLoop)));
    MGB_CUDA(cudaMallocHost(&w.loop_hist_host, sizeof(DobfsHist) * kLoopHist));
    for (int i = 0; i < 3; ++i)
      if (w.ul_buf[i].n < k + 1 || !w.ul_buf[i].ptr) w.ul_buf[i].alloc(k + 1);
    w.loop_front[0].alloc(w.nv ? w.nv : 1);
    w.loop_front[1].alloc(w.nv ? w.nv : 1);
    w.loop_lb_row.alloc(w.nv ? w.nv : 1);
    w.loop_lb_pref.alloc(w.nv ? w.nv : 1);
    w.loop_lb_bsum.alloc(w.nv / kLbBlock + 4);
    w.loop_total.alloc(1);
    const uint64_t max_tiles = (2 * w.ne + 1) / kTile + 2 + kMinTiles;
    w.loop_tiles.alloc(max_tiles + 1);
  }

  static DobfsGraph graph(Worker& w, bool mark_preds) {
    const int gi = mark_preds ? 1 : 0;
    const std::vector<const void*> ptrs = pointers(w);
    if (w.loop_exec[gi] && w.loop_ptrs[gi] == ptrs)
      return {w.loop_exec[gi], w.loop_n_pull[gi], w.loop_n_push[gi]};
    if (w.loop_exec[gi]) {  // a captured buffer moved
      cudaGraphExecDestroy(w.loop_exec[gi]);
      w.loop_exec[gi] = nullptr;
    }
    w.loop_ptrs[gi] = ptrs;
    cudaStream_t s = w.stream;
    const uint64_t nw = (w.nv + 31) / 32 + 1;
    DobfsLoop* st = reinterpret_cast<DobfsLoop*>(w.loop_state.ptr);
    DobfsHist* hist = reinterpret_cast<DobfsHist*>(w.loop_hist.ptr);
    Counters* ctr = w.ctr.ptr;
    cudaGraph_t g;
    MGB_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h_while;
    MGB_CUDA(cudaGraphConditionalHandleCreate(&h_while, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = h_while;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    MGB_CUDA(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    // superstep 0 is a push (the defaults, assigned at every launch); the end
    // kernel sets the next superstep's direction
    cudaGraphConditionalHandle h_pull, h_push;
    MGB_CUDA(cudaGraphConditionalHandleCreate(&h_pull, body, 0, cudaGraphCondAssignDefault));
    MGB_CUDA(cudaGraphConditionalHandleCreate(&h_push, body, 1, cudaGraphCondAssignDefault));
    cudaGraph_t tmp;
    // IF pull / IF push
    cudaGraphNode_t ifs[2];
    cudaGraph_t bodies[2];
    cudaGraphConditionalHandle hs[2] = {h_pull, h_push};
    for (int i = 0; i < 2; ++i) {
      cudaGraphNodeParams ip = {};
      ip.type = cudaGraphNodeTypeConditional;
      ip.conditional.handle = hs[i];
      ip.conditional.type = cudaGraphCondTypeIf;
      ip.conditional.size = 1;
      MGB_CUDA(cudaGraphAddNode(&ifs[i], body, nullptr, 0, &ip));
      bodies[i] = ip.conditional.phGraph_out[0];
    }
    GraphView gv = w.graph();
    OwnerView ow{w.owner.ptr, w.l2g.ptr, w.p, w.nlocal, MG_DUP_ALL};
    uint32_t* cnts = w.aux[2].ptr;
    DobfsDyn dyn{st, w.ul_buf[0].ptr, w.ul_buf[1].ptr};
    const int mp = mark_preds ? 1 : 0;
    uint64_t l0 = g_launches.load();
    // pull branch
    MGB_CUDA(cudaStreamBeginCaptureToGraph(s, bodies[0], nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed));
    MGB_LAUNCH(frontier_diff_kernel, grid_for(nw, 256, num_sms() * 8), 256, 0, s, w.su32[2].ptr,
               w.aux[4].ptr, w.su32[3].ptr, (uint32_t)nw, cnts, nullptr, 0ull,
               (const DobfsLoop*)st, &ctr->edges);
    MGB_LAUNCH(dobfs_pull_thread_kernel<false>, num_sms() * kPullCtas, kPullBlock, 0, s, gv, w.pull_rec.ptr,
               w.pull_ext.ptr, nullptr, 0u,
               w.su32[0].ptr, w.su32[1].ptr, w.su32[2].ptr, w.su32[3].ptr, 0u, mp, ow, 0,
               w.loop_front[1].ptr, nullptr, &ctr->misc, w.ul_buf[2].ptr, cnts + 1, ctr,
               (unsigned long long*)nullptr, &ctr->next_deg, dyn);
    uint32_t* gq = w.ul_buf[2].ptr;
    uint32_t* gq_cnt = cnts + 1;
    // the superstep end runs in the last CTA of each branch's last kernel
    DobfsLoopEnd le;
    le.st = st;
    le.hist = hist;
    le.h_while = h_while;
    le.h_pull = h_pull;
    le.h_push = h_push;
    MGB_LAUNCH(dobfs_pull_group_kernel, num_sms() * 8, 256, 0, s, gv, w.pull_rec.ptr,
               gq, gq_cnt, w.su32[0].ptr, w.su32[1].ptr, w.su32[2].ptr,
               w.su32[3].ptr, 0u, mp, ow, 0, w.loop_front[1].ptr, nullptr, &ctr->misc, ctr,
               (unsigned long long*)nullptr, &ctr->next_deg, dyn, le);
    MGB_CUDA(cudaStreamEndCapture(s, &tmp));
    const uint64_t l1 = g_launches.load();
    // push branch: frontier list from the bitmap, prev = vis, edge-balanced advance
    MGB_CUDA(cudaStreamBeginCaptureToGraph(s, bodies[1], nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed));
    MGB_LAUNCH(bitmap_diff_list_kernel, grid_for(nw, 256, num_sms() * 8), 256, 0, s, w.su32[2].ptr,
               w.aux[4].ptr, (uint32_t)nw, w.loop_front[0].ptr, &st->in_count, 1,
               (const DobfsLoop*)st);
    const uint32_t* nin = &st->in_count;
    MGB_LAUNCH(lb_degree_kernel, num_sms() * 8, kLbBlock, 0, s, w.off.ptr, w.loop_front[0].ptr, 0u,
               w.loop_lb_row.ptr, w.loop_lb_pref.ptr, w.loop_lb_bsum.ptr, nin);
    MGB_LAUNCH(lb_scan_kernel, 1, 1024, 0, s, w.loop_lb_bsum.ptr, 0u, w.loop_total.ptr,
               &ctr->edges, nin);
    const uint64_t max_tiles = (2 * w.ne + 1) / kTile + 2 + kMinTiles;
    MGB_LAUNCH(lb_tiles_kernel, num_sms() * 8, 256, 0, s, w.loop_lb_pref.ptr, w.loop_lb_bsum.ptr,
               0u, w.loop_total.ptr, w.loop_tiles.ptr, (uint32_t)max_tiles, nin);
    DobfsDev f{w.su32[0].ptr, w.su32[1].ptr, w.su32[2].ptr, w.su32[3].ptr, ow, 0u, mp, &st->iter};
    // dense pushes (no predecessors): labels and counts from the bitmap diff
    const DensePush dp{w.loop_total.ptr, mark_preds ? 0ull : loop_dense_push_arcs(), w.su32[2].ptr,
                       w.aux[4].ptr, w.su32[0].ptr, (uint32_t)nw};
    f.red_total = dp.total;
    f.red_min = dp.min;
    MGB_LAUNCH((lb_expand_kernel<DobfsDev, true>), (expand_resident<DobfsDev, true>()), kExpBlock, 0, s, f, gv,
               w.loop_front[0].ptr, 0u, w.loop_lb_row.ptr, w.loop_lb_pref.ptr, w.loop_lb_bsum.ptr,
               w.loop_total.ptr, w.loop_tiles.ptr, w.loop_front[1].ptr, &ctr->out_cnt, nin);
    MGB_LAUNCH(dobfs_degsum_end_kernel, num_sms() * MG_LOOP_END_CTAS, 256, 0, s, gv, w.loop_front[1].ptr, ctr,
               le, dp);
    MGB_CUDA(cudaStreamEndCapture(s, &tmp));
    const uint64_t l2 = g_launches.load();
    g_launches.store(l0);  // capture is not execution
    MGB_CUDA(cudaGraphInstantiate(&w.loop_exec[gi], g, 0));
    MGB_CUDA(cudaGraphDestroy(g));
    w.loop_n_pull[gi] = (uint32_t)(l1 - l0);
    w.loop_n_push[gi] = (uint32_t)(l2 - l1);
    return {w.loop_exec[gi], w.loop_n_pull[gi], w.loop_n_push[gi]};
  }
};

// ---------------------------------------------------------------------------
// Device-driven DOBFS across processes (one GPU and one partition per rank,
// the device fabric of engine.cuh).  Every superstep of the enactor —
//   decide   the reference direction rule (primitives.cpp:197-205) on the
//            global quantities, and the exact-cost physical choice on the sums
//            all ranks reported last superstep (u[0], u[1]), in the same double
//            arithmetic as the host path
//   IF pull  frontier_diff, pull thread + cooperative stages (discoveries listed)
//   IF push  prev = visited, edge-balanced advance from the input frontier
//   split + pack (discovery bitmap or records into the peers' inboxes),
//   publish, wait for the peers' publish flags, merge (records + dense),
//   report all-gather through the mailboxes, end (global sums, history,
//   convergence: Σ next frontiers == 0, E:784-820)
// — runs inside ONE graph launch: a WHILE node whose body holds two
// supersteps (even / odd, so the frontier ping-pong buffers and the inbox
// parity are fixed in each); the second one's decide kernel turns all of it
// off once the first converged (conditionals nest two levels deep).  No
// superstep waits for the host; every rank takes the same decisions from the
// same all-gathered reports.  Results and statistics equal the host loop's
// (tests/test_fabric.py::test_dobfs_device_loop_*).
constexpr uint32_t kMpHist = 65536;
constexpr uint32_t kMpMaxRanks = 8;  // history keeps an n x n send matrix per superstep

struct DobfsMpLoop {
  DobfsLoop b;  // first: the pull / frontier kernels read it as a DobfsLoop
  uint32_t n, me, epoch, overflow;
  uint32_t own_next;               // this rank's next frontier (global discoveries)
  uint32_t more;                   // the loop continues after the last end kernel
  unsigned long long own_next_deg;
};
struct DobfsMpHist {
  uint32_t dir, physical;
  unsigned long long out, next, edges, combine;
  uint32_t send[kMpMaxRanks][kMpMaxRanks];  // [src][dst], kDenseFlag kept
};

__global__ void dobfs_mp_init_kernel(DobfsMpLoop* st, uint32_t* labels, uint32_t* vis) {
  (void)labels;
  (void)vis;
  DobfsLoop& b = st->b;
  b.iter = 0;
  b.dir = 0;
  b.switched = 0;
  b.physical = 0;
  b.ul_src = 2;  // every non-isolated record, no list
  b.ul_len = b.n_nonisolated;
  b.visited = 1;
  b.prev_physical = 0;
  st->overflow = 0;
}

// (h_rest: the odd superstep's exchange-and-report IF, 0 for the even one;
// an odd superstep after convergence runs nothing)
__global__ void dobfs_mp_decide_kernel(DobfsMpLoop* st, DobfsMpHist* hist, const Mailbox* mine,
                                       cudaGraphConditionalHandle h_pull,
                                       cudaGraphConditionalHandle h_push,
                                       cudaGraphConditionalHandle h_rest) {
  if (h_rest) {
    cudaGraphSetConditional(h_rest, st->more ? 1u : 0u);
    if (!st->more) {
      cudaGraphSetConditional(h_pull, 0u);
      cudaGraphSetConditional(h_push, 0u);
      return;
    }
  }
  DobfsLoop& b = st->b;
  const uint32_t t = b.iter;
  st->epoch += 1;  // the host loop's ++mp_epoch at the top of a superstep
  if (t >= 1) {    // primitives.cpp:197-205, as DobfsPrim::body
    b.visited += b.in_count;
    const double fv = b.nv > 0 ? (double)b.in_count * b.ne_d / b.nv_d : 0.0;
    const double bv = b.visited > 0 ? (double)((unsigned long long)b.nv - b.visited) * b.nv_d /
                                          (double)b.visited
                                    : 0.0;
    uint32_t next;
    if (b.dir == 0) next = (!b.switched && fv > bv * b.do_a) ? 1u : 0u;
    else next = fv < bv * b.do_b ? 0u : 1u;
    if (next == 1 && b.dir == 0) b.switched = 1;
    b.dir = next;
  }
  uint32_t phys = b.dir == 1;
  if (b.dir == 0 && b.exact && t > 0) {
    // the sums every rank reported last superstep (slot of epoch - 1)
    const uint32_t ps = (st->epoch - 1) & 1u;
    unsigned long long gw = 0, gul = 0;
    for (uint32_t q = 0; q < st->n; ++q) {
      const volatile DevReport* r = &mine->rep[ps][q];
      gw += r->u[1];
      gul += r->u[0];
    }
    phys = (double)gw > b.pull_ratio * (double)gul;
  }
  b.physical = phys;
  hist[t].dir = b.dir;
  hist[t].physical = phys;
  cudaGraphSetConditional(h_pull, phys);
  cudaGraphSetConditional(h_push, phys ? 0u : 1u);
}

// before the report clears the counters: keep what the next superstep needs,
// and share the exact-cost inputs (dobfs_share_kernel)
__global__ void dobfs_mp_pre_report_kernel(DobfsMpLoop* st, Counters* ctr) {
  DobfsLoop& b = st->b;
  st->own_next = ctr->next_cnt;
  st->own_next_deg = ctr->next_deg;
  if (b.exact) {
    ctr->u[0] = b.physical ? ctr->misc : b.ul_len;
    ctr->u[1] = ctr->next_deg;
  }
  if (b.physical) {  // the pull compacted the unvisited list (ping-pong)
    b.ul_len = ctr->misc;
    b.ul_src = b.ul_src == 0 ? 1 : 0;
  }
  b.prev_physical = b.physical;
}

__global__ void dobfs_mp_end_kernel(DobfsMpLoop* st, const Mailbox* mine, DobfsMpHist* hist,
                                    const uint32_t* err, cudaGraphConditionalHandle h_while) {
  DobfsLoop& b = st->b;
  const uint32_t t = b.iter, slot = st->epoch & 1u, n = st->n;
  unsigned long long out = 0, next = 0, edges = 0, comb = 0;
  uint32_t ovf = 0;
  DobfsMpHist& h = hist[t];
  for (uint32_t q = 0; q < n; ++q) {
    const volatile DevReport* r = &mine->rep[slot][q];
    out += r->out_frontier;
    next += r->next_frontier;
    edges += r->edges_delta;
    comb += r->combine_delta;
    ovf |= r->overflow;
    for (uint32_t d = 0; d < kMpMaxRanks; ++d) h.send[q][d] = d < n ? r->send_cnt[d] : 0u;
  }
  h.out = out;
  h.next = next;
  h.edges = edges;
  h.combine = comb;
  b.in_count = st->own_next;
  b.in_degsum = st->own_next_deg;
  b.iter = t + 1;
  st->overflow |= ovf;
  const bool more = next > 0 && t + 1 < b.max_supersteps && t + 1 < kMpHist && !ovf &&
                    !*reinterpret_cast<const volatile uint32_t*>(err);
  st->more = more ? 1u : 0u;
  cudaGraphSetConditional(h_while, more ? 1u : 0u);
}

class DobfsMpGraphRunner {
 public:
  static bool eligible(const Plan& P, const mg_config& c, bool mark_preds) {
    const char* e = getenv("MG_MP_GRAPH_LOOP");
    if ((e && e[0] == '0') || getenv("MG_NO_GRAPH")) return false;
    const bool fused = c.fused == MG_FUSED_ON || (c.fused == MG_FUSED_AUTO &&
                                                  c.policy == MG_POLICY_FUSED);
    return P.n > 1 && P.n <= kMpMaxRanks && P.shm && P.device_fabric &&
           P.local_workers.size() == 1 && P.dup == MG_DUP_ALL && !P.profile && !mark_preds &&
           c.policy == MG_POLICY_MAX && fused && !c.drop_enabled && c.hard_cap_bytes == 0;
  }

  // runs the supersteps of a prepared run (run_primitive's prologue done:
  // inboxes, send tables, init, source seeded into next_input)
  static void run(Plan& P, DobfsPrim& prim, Ctx& c, RunState& rs, const mg_config& cfg,
                  DeviceLoopOut& o) {
    Worker& w = *c.w;
    const uint32_t n = P.n, p = w.p;
    DeviceGuard dg(w.dev);
    // frontier buffers at their superstep bound before capture (next_input
    // keeps the seeded source)
    uint64_t incoming = w.nv;
    for (uint32_t s = 0; s < n; ++s) incoming += (s == p) ? 0 : w.slot_cap[s];
    w.output.ensure(w.nv, w.stream);
    w.next_input.ensure(w.output.cap + incoming, w.stream, rs.next_count[p]);
    w.input.ensure(w.output.cap + incoming, w.stream);
    ensure_buffers(w);
    const DenseView dv = prim.dense_view(c);
    cudaGraphExec_t exec = graph(P, w, c, prim, dv);
    DobfsMpLoop h{};
    DobfsLoop& b = h.b;
    b.nv_d = (double)P.nv;
    b.ne_d = (double)P.ne;
    b.do_a = prim.do_a;
    b.do_b = prim.do_b;
    b.pull_ratio = pull_ratio();
    b.nv = P.nv;
    b.source = prim.source;
    b.max_supersteps = (uint32_t)(cfg.max_supersteps < kMpHist ? cfg.max_supersteps : kMpHist);
    b.exact = prim.exact_cost ? 1u : 0u;
    b.n_nonisolated = w.n_nonisolated;
    b.in_count = rs.next_count[p];
    b.in_degsum = 0;
    h.n = n;
    h.me = P.rank;
    h.epoch = P.mp_epoch;
    DobfsMpLoop* st = reinterpret_cast<DobfsMpLoop*>(w.mp_state.ptr);
    MGB_CUDA(cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, w.stream));
    MGB_LAUNCH(dobfs_mp_init_kernel, 1, 1, 0, w.stream, st, w.su32[0].ptr, w.su32[2].ptr);
    MGB_CUDA(cudaGraphLaunch(exec, w.stream));
    MGB_CUDA(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, w.stream));
    MGB_CUDA(cudaStreamSynchronize(w.stream));
    if (*reinterpret_cast<volatile uint32_t*>(P.host_reports + kMaxMpRanks))
      throw Error(MG_EWORKER, "fabric: a peer rank did not arrive within the timeout");
    if (h.overflow) throw Error(MG_EWORKER, "inbox overflow on a peer worker");
    const uint32_t S = b.iter;
    std::vector<DobfsMpHist> hist(S);
    MGB_CUDA(cudaMemcpy(hist.data(), w.mp_hist.ptr, sizeof(DobfsMpHist) * S,
                        cudaMemcpyDeviceToHost));
    if (S && hist[S - 1].next && S >= kMpHist && cfg.max_supersteps > kMpHist)
      throw Error(MG_EWORKER, "dobfs: the device-driven loop records at most 65536 supersteps "
                              "(MG_MP_GRAPH_LOOP=0 runs the host loop)");
    P.mp_epoch = h.epoch;
    // statistics in the enactor's shapes
    o.supersteps = S;
    o.h_matrix.assign(n, std::vector<uint64_t>(n, 0));
    const uint64_t rec_bytes = 4ull + 4ull * prim.nva + 8ull * prim.nvv;
    const uint64_t dense_bytes = 4ull * (dv.kind ? dv.words : 0);
    uint64_t launches = 2;  // init + graph
    for (uint32_t t = 0; t < S; ++t) {
      const DobfsMpHist& e = hist[t];
      prim.dir_log.push_back((int)e.dir);
      if (e.physical && e.dir == 0) ++prim.physical_pull_steps;
      o.out.push_back(e.out);
      o.next.push_back(e.next);
      o.edges.push_back(e.edges);
      o.combine.push_back(e.combine);
      std::vector<uint64_t> hs(n, 0);
      for (uint32_t q = 0; q < n; ++q)
        for (uint32_t d = 0; d < n; ++d) {
          if (d == q) continue;
          const uint32_t raw = e.send[q][d];
          const uint64_t len = raw & ~kDenseFlag;
          o.h_matrix[q][d] += len;
          hs[q] += len;
          o.wire += len;
          if (q == P.rank) o.xbytes += (raw & kDenseFlag) ? dense_bytes : len * rec_bytes;
        }
      o.h_src.push_back(hs);
      launches += w.mp_n_fixed + (e.physical ? w.mp_n_pull : w.mp_n_push);
    }
    o.stop_reason = (S && hist[S - 1].next == 0) ? MG_STOP_FRONTIERS_EMPTY
                                                 : MG_STOP_MAX_SUPERSTEPS;
    g_launches.fetch_add(launches, std::memory_order_relaxed);
  }

 private:
  static void ensure_buffers(Worker& w) {
    if (!w.mp_state.ptr) w.mp_state.alloc(sizeof(DobfsMpLoop));
    if (!w.mp_hist.ptr) w.mp_hist.alloc(sizeof(DobfsMpHist) * kMpHist);
    const uint64_t nw = (w.nv + 31) / 32 + 1;
    if (w.su32[3].n < nw || !w.su32[3].ptr) w.su32[3].alloc(nw);  // frontier bitmap
    if (w.aux[2].n < 4 || !w.aux[2].ptr) w.aux[2].alloc(4);
    // advance scratch for an input of up to the frontier buffer's capacity
    const uint64_t cap = w.input.cap > 1 ? w.input.cap : 1;
    if (w.loop_lb_row.n < cap) w.loop_lb_row.alloc(cap);
    if (w.loop_lb_pref.n < cap) w.loop_lb_pref.alloc(cap);
    if (w.loop_lb_bsum.n < cap / kLbBlock + 4) w.loop_lb_bsum.alloc(cap / kLbBlock + 4);
    if (!w.loop_total.ptr) w.loop_total.alloc(1);
    const uint64_t tiles = (2 * w.ne + 1) / kTile + 2 + kMinTiles + 1;
    if (w.loop_tiles.n < tiles) w.loop_tiles.alloc(tiles);
  }

  static std::vector<const void*> pointers(const Plan& P, const Worker& w) {
    return {w.su32[0].ptr, w.su32[2].ptr, w.su32[3].ptr, w.aux[2].ptr, w.aux[4].ptr,
            w.ul_buf[0].ptr, w.ul_buf[1].ptr, w.ul_buf[2].ptr, w.pull_rec.ptr, w.pull_ext.ptr,
            w.off.ptr,
            w.col.ptr, w.owner.ptr, w.ctr.ptr, w.mp_state.ptr, w.mp_hist.ptr, w.input.ptr,
            w.next_input.ptr, w.output.ptr, w.send_table.ptr, w.send_cnt_ptr.ptr,
            w.recv_table.ptr, w.inbox_cnt.ptr, w.merge_stamp.ptr, w.loop_lb_row.ptr,
            w.loop_lb_pref.ptr, w.loop_lb_bsum.ptr, w.loop_total.ptr, w.loop_tiles.ptr,
            P.mbox.ptr, P.mbox_ptrs.ptr, P.host_reports_dev,
            reinterpret_cast<const void*>((uintptr_t)P.n)};
  }
  // ... plus the slot capacities (merge grids) and the output capacity (split grid)
  static std::vector<const void*> signature(const Plan& P, const Worker& w) {
    std::vector<const void*> v = pointers(P, w);
    for (uint64_t c : w.slot_cap) v.push_back(reinterpret_cast<const void*>((uintptr_t)c));
    v.push_back(reinterpret_cast<const void*>((uintptr_t)w.output.cap));
    return v;
  }

  // the leaf nodes of an ongoing capture (to hang the next node on)
  static std::vector<cudaGraphNode_t> leaves(cudaStream_t s) {
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    MGB_CUDA(cudaStreamGetCaptureInfo(s, &cs, nullptr, nullptr, &deps, &nd));
    return std::vector<cudaGraphNode_t>(deps, deps + nd);
  }

  // one superstep at a fixed parity into graph g; returns its leaf nodes
  // one superstep at a fixed parity into graph g, after the nodes `deps`
  // (none: the graph's roots); the odd superstep's exchange-and-report part
  // sits in its own IF node, so no conditional nests deeper than two levels
  // (WHILE -> IF).  Returns the superstep's leaf nodes.
  static std::vector<cudaGraphNode_t> substep(Plan& P, Worker& w, Ctx& c, const DenseView& dv,
                                              bool st_exact, cudaGraph_t g, int parity,
                                              const std::vector<cudaGraphNode_t>& deps,
                                              cudaGraphConditionalHandle h_while,
                                              uint64_t& n_pull, uint64_t& n_push,
                                              uint64_t& n_fixed) {
    cudaStream_t s = w.stream;
    const uint32_t n = P.n, p = w.p;
    const uint64_t nw = (w.nv + 31) / 32 + 1;
    DobfsMpLoop* st = reinterpret_cast<DobfsMpLoop*>(w.mp_state.ptr);
    DobfsMpHist* hist = reinterpret_cast<DobfsMpHist*>(w.mp_hist.ptr);
    Mailbox* mine = reinterpret_cast<Mailbox*>(P.mbox.ptr);
    uint32_t* err = reinterpret_cast<uint32_t*>(P.host_reports_dev + kMaxMpRanks);
    Counters* ctr = w.ctr.ptr;
    uint32_t* cnts = w.aux[2].ptr;
    GraphView gv = w.graph();
    OwnerView ow = c.owner_view();
    // even supersteps read input A and fill B, odd ones the reverse
    // (A = the buffer the prologue seeded: next_input)
    uint32_t* in = parity == 0 ? w.next_input.ptr : w.input.ptr;
    uint32_t* nxt = parity == 0 ? w.input.ptr : w.next_input.ptr;
    DobfsDev f{w.su32[0].ptr, w.su32[1].ptr, w.su32[2].ptr, w.su32[3].ptr, ow, 0u, 0,
               &st->b.iter};
    cudaGraphConditionalHandle h_pull, h_push, h_rest = 0;
    MGB_CUDA(cudaGraphConditionalHandleCreate(&h_pull, g, 0, cudaGraphCondAssignDefault));
    MGB_CUDA(cudaGraphConditionalHandleCreate(&h_push, g, 0, cudaGraphCondAssignDefault));
    if (parity == 1)
      MGB_CUDA(cudaGraphConditionalHandleCreate(&h_rest, g, 0, cudaGraphCondAssignDefault));
    cudaGraph_t tmp;
    const uint64_t l0 = g_launches.load();
    // decide
    MGB_CUDA(cudaStreamBeginCaptureToGraph(s, g, deps.data(), nullptr, deps.size(),
                                           cudaStreamCaptureModeRelaxed));
    MGB_LAUNCH(dobfs_mp_decide_kernel, 1, 1, 0, s, st, hist, mine, h_pull, h_push, h_rest);
    std::vector<cudaGraphNode_t> dec = leaves(s);
    MGB_CUDA(cudaStreamEndCapture(s, &tmp));
    cudaGraphNode_t ifs[2];
    cudaGraph_t bodies[2];
    cudaGraphConditionalHandle hs[2] = {h_pull, h_push};
    for (int i = 0; i < 2; ++i) {
      cudaGraphNodeParams ip = {};
      ip.type = cudaGraphNodeTypeConditional;
      ip.conditional.handle = hs[i];
      ip.conditional.type = cudaGraphCondTypeIf;
      ip.conditional.size = 1;
      MGB_CUDA(cudaGraphAddNode(&ifs[i], g, dec.data(), dec.size(), &ip));
      bodies[i] = ip.conditional.phGraph_out[0];
    }
    const uint64_t l1 = g_launches.load();
    // pull branch: discoveries listed into output (several partitions)
    MGB_CUDA(cudaStreamBeginCaptureToGraph(s, bodies[0], nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed));
    DobfsDyn dyn{&st->b, w.ul_buf[0].ptr, w.ul_buf[1].ptr};
    MGB_LAUNCH(frontier_diff_kernel, grid_for(nw, 256, num_sms() * 8), 256, 0, s, w.su32[2].ptr,
               w.aux[4].ptr, w.su32[3].ptr, (uint32_t)nw, cnts, nullptr, 0ull, &st->b,
               &ctr->edges);
    MGB_LAUNCH(dobfs_pull_thread_kernel<true>, num_sms() * kPullCtas, kPullBlock, 0, s, gv,
               w.pull_rec.ptr, w.pull_ext.ptr, nullptr, 0u, w.su32[0].ptr, w.su32[1].ptr, w.su32[2].ptr,
               w.su32[3].ptr, 0u, 0, ow, 1, w.output.ptr, nullptr, &ctr->misc, w.ul_buf[2].ptr,
               cnts + 1, ctr, (unsigned long long*)nullptr, (unsigned long long*)nullptr, dyn);
    MGB_LAUNCH(dobfs_pull_group_kernel, num_sms() * 8, 256, 0, s, gv, w.pull_rec.ptr,
               w.ul_buf[2].ptr, cnts + 1, w.su32[0].ptr, w.su32[1].ptr, w.su32[2].ptr,
               w.su32[3].ptr, 0u, 0, ow, 1, w.output.ptr, nullptr, &ctr->misc, ctr,
               (unsigned long long*)nullptr, (unsigned long long*)nullptr, dyn);
    MGB_CUDA(cudaStreamEndCapture(s, &tmp));
    const uint64_t l2 = g_launches.load();
    // push branch: prev = visited, edge-balanced advance from the input list
    MGB_CUDA(cudaStreamBeginCaptureToGraph(s, bodies[1], nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed));
    MGB_CUDA(cudaMemcpyAsync(w.aux[4].ptr, w.su32[2].ptr, 4 * nw, cudaMemcpyDeviceToDevice, s));
    const uint32_t* nin = &st->b.in_count;
    MGB_LAUNCH(lb_degree_kernel, num_sms() * 8, kLbBlock, 0, s, w.off.ptr, in, 0u,
               w.loop_lb_row.ptr, w.loop_lb_pref.ptr, w.loop_lb_bsum.ptr, nin);
    MGB_LAUNCH(lb_scan_kernel, 1, 1024, 0, s, w.loop_lb_bsum.ptr, 0u, w.loop_total.ptr,
               &ctr->edges, nin);
    const uint64_t max_tiles = (2 * w.ne + 1) / kTile + 2 + kMinTiles;
    MGB_LAUNCH(lb_tiles_kernel, num_sms() * 8, 256, 0, s, w.loop_lb_pref.ptr, w.loop_lb_bsum.ptr,
               0u, w.loop_total.ptr, w.loop_tiles.ptr, (uint32_t)max_tiles, nin);
    MGB_LAUNCH((lb_expand_kernel<DobfsDev, true>), (expand_resident<DobfsDev, true>()), kExpBlock, 0, s, f, gv, in, 0u,
               w.loop_lb_row.ptr, w.loop_lb_pref.ptr, w.loop_lb_bsum.ptr, w.loop_total.ptr,
               w.loop_tiles.ptr, w.output.ptr, &ctr->out_cnt, nin);
    MGB_CUDA(cudaStreamEndCapture(s, &tmp));
    const uint64_t l3 = g_launches.load();
    // exchange + completion, after both branches (the odd superstep: inside IF(rest))
    cudaGraph_t rg = g;
    cudaGraphNode_t rest_node = nullptr;
    if (parity == 1) {
      cudaGraphNodeParams rp = {};
      rp.type = cudaGraphNodeTypeConditional;
      rp.conditional.handle = h_rest;
      rp.conditional.type = cudaGraphCondTypeIf;
      rp.conditional.size = 1;
      MGB_CUDA(cudaGraphAddNode(&rest_node, g, ifs, 2, &rp));
      rg = rp.conditional.phGraph_out[0];
      MGB_CUDA(cudaStreamBeginCaptureToGraph(s, rg, nullptr, nullptr, 0,
                                             cudaStreamCaptureModeRelaxed));
    } else {
      MGB_CUDA(cudaStreamBeginCaptureToGraph(s, g, ifs, nullptr, 2, cudaStreamCaptureModeRelaxed));
    }
    // Σdeg of the next frontier, the exact-cost input (reports_deg, E:845)
    const int want_deg = st_exact ? 1 : 0;
    const uint64_t items = w.output.cap > dv.words ? w.output.cap : dv.words;
    MGB_LAUNCH(split_pack_kernel<DobfsDev>, grid_for(items, 256, num_sms() * 8), 256, 0, s, f, ow,
               gv, w.output.ptr, ctr, nxt, w.send_table.ptr + parity * n, n, 1, 0ull, 0, 0,
               want_deg, dv);
    MGB_LAUNCH(publish_kernel, 1, 64, 0, s, ctr, w.send_cnt_ptr.ptr + parity * n, n, p,
               P.mbox_ptrs.ptr, (uint32_t)parity, 0u, &st->epoch);
    MGB_LAUNCH(mp_wait_pub_kernel, 1, 32, 0, s, mine, (uint32_t)parity, 0u, n, P.rank, err,
               &st->epoch);
    uint64_t maxcap = 0;
    for (uint32_t q = 0; q < n; ++q)
      if (q != p && w.slot_cap[q] > maxcap) maxcap = w.slot_cap[q];
    MGB_LAUNCH(merge_kernel<DobfsDev>, dim3(grid_for(maxcap, 256, num_sms() * 2), n), 256, 0, s,
               f, w.recv_table.ptr + parity * n, w.inbox_cnt.ptr + parity * kMaxWorkers, p, 0u, 0u,
               w.merge_stamp.ptr, nxt, ctr, gv, 0, 0, 1, want_deg, &st->b.iter);
    if (dv.kind)
      MGB_LAUNCH(merge_dense_kernel<DobfsDev>, dim3(grid_for(dv.words, 256, num_sms() * 2), n),
                 256, 0, s, f, dv, w.recv_table.ptr + parity * n,
                 w.inbox_cnt.ptr + parity * kMaxWorkers, p, 0u, 0u, w.merge_stamp.ptr, nxt, ctr,
                 gv, want_deg, &st->b.iter);
    MGB_LAUNCH(dobfs_mp_pre_report_kernel, 1, 1, 0, s, st, ctr);
    MGB_LAUNCH(mp_report_kernel, 1, 128, 0, s, ctr, (Counters*)nullptr, HostReportPart{},
               P.mbox_ptrs.ptr, n, P.rank, 0u, (DevReport*)nullptr, err, &st->epoch);
    MGB_LAUNCH(dobfs_mp_end_kernel, 1, 1, 0, s, st, mine, hist, err, h_while);
    std::vector<cudaGraphNode_t> out = leaves(s);
    MGB_CUDA(cudaStreamEndCapture(s, &tmp));
    if (rest_node) out.assign(1, rest_node);
    const uint64_t l4 = g_launches.load();
    n_pull = l2 - l1;
    n_push = l3 - l2;
    n_fixed = (l1 - l0) + (l4 - l3);
    return out;
  }

  static cudaGraphExec_t graph(Plan& P, Worker& w, Ctx& c, DobfsPrim& prim,
                               const DenseView& dv) {
    std::vector<const void*> ptrs = signature(P, w);
    ptrs.push_back(reinterpret_cast<const void*>((uintptr_t)(prim.exact_cost ? 1 : 0)));
    if (w.mp_exec && w.mp_ptrs == ptrs) return w.mp_exec;
    if (w.mp_exec) {
      cudaGraphExecDestroy(w.mp_exec);
      w.mp_exec = nullptr;
    }
    const uint64_t launches0 = g_launches.load();
    cudaGraph_t g;
    MGB_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h_while;
    MGB_CUDA(cudaGraphConditionalHandleCreate(&h_while, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = h_while;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    MGB_CUDA(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    // even superstep, then the odd one (a no-op once the even one converged)
    uint64_t np, nq, nf;
    std::vector<cudaGraphNode_t> tail =
        substep(P, w, c, dv, prim.exact_cost, body, 0, {}, h_while, np, nq, nf);
    substep(P, w, c, dv, prim.exact_cost, body, 1, tail, h_while, np, nq, nf);
    g_launches.store(launches0);  // capture is not execution
    MGB_CUDA(cudaGraphInstantiate(&w.mp_exec, g, 0));
    MGB_CUDA(cudaGraphDestroy(g));
    w.mp_ptrs = ptrs;
    w.mp_n_pull = (uint32_t)np;
    w.mp_n_push = (uint32_t)nq;
    w.mp_n_fixed = (uint32_t)nf;
    return w.mp_exec;
  }
};

bool DobfsPrim::device_loop(Plan& P, std::vector<Ctx>& ctx, RunState& rs, const mg_config& cfg,
                            DeviceLoopOut& o) {
  if (!DobfsMpGraphRunner::eligible(P, cfg, mark_preds)) return false;
  DobfsMpGraphRunner::run(P, *this, ctx[P.rank], rs, cfg, o);
  return true;
}

// ===========================================================================
// SSSP (primitives.cpp:307-397)

#ifndef MG_SSSP_DENSE_DIV
#define MG_SSSP_DENSE_DIV 256  // RMAT-24 C3: off 11.3 ms, 32: 9.27, 128: 8.25, 512: 8.24, 4096: 8.29, always: 8.41
#endif

// Distances are kept in T = u32 when every finite distance fits (max edge
// weight x |V| < 2^32 - 1: RMAT-24 with w <= 64 needs 1.07e9), else u64 like
// the reference.  The u32 array is half the size (67 MB at |V| = 2^24, inside
// the 126 MB L2), so the random relaxation atomics hit L2; results are widened
// to u64 (u32 inf -> u64 inf) when the run finishes.
template <class T>
struct SsspDev {
  static constexpr T kInf = (T)~(T)0;
  T* dists;
  const T* fdist;
  T* last_sent;
  uint32_t* preds;
  uint32_t* seen;
  const uint32_t* w;
  OwnerView ow;
  uint32_t iter;
  int mark_preds;
  // dense superstep (one partition, no preds): improving arcs issue
  // fire-and-forget atomicMin (RED) and accept nothing; the output frontier is
  // the set of vertices whose distance fell below the superstep's full
  // snapshot, listed by dense_list_kernel<SsspFell> afterwards
  int red = 0;
  // relax from the superstep-frozen source distance (primitives.cpp:340-348)
  __device__ bool visit(uint32_t u, uint32_t v, uint32_t e) const {
    T nd = fdist[u] + (T)w[e];
    if (nd >= __ldcg(&dists[v])) return false;
    T old = atomicMin(&dists[v], nd);
    if (nd < old) {
      if (mark_preds) preds[v] = ow.to_global(u);
      return true;
    }
    return false;
  }
  // once per superstep: a |V|/8-byte bitmap cleared at every superstep (2 MB
  // at 2^24, L2-resident) instead of a 4-byte stamp per vertex, so the random
  // relaxation traffic leaves the L2 to the distances
  __device__ bool keep(uint32_t v) const {
    const uint32_t b = 1u << (v & 31);
    return !(atomicOr(&seen[v >> 5], b) & b);
  }
  __device__ bool prefilter(uint32_t) const { return true; }
  __device__ bool combine(uint32_t v, const uint32_t* va, const double* vv, uint32_t) const {
    T nd = (T)vv[0];
    T old = atomicMin(&dists[v], nd);
    if (nd < old) {
      if (mark_preds) preds[v] = va[0];
      return ow.hosts(v);
    }
    return false;
  }
  __device__ void gather(uint32_t v, uint32_t* va, double* vv) const {
    vv[0] = (double)dists[v];
    if (mark_preds) va[0] = preds[v];
  }
  // pre-send suppression (primitives.cpp:377-383)
  __device__ bool send_filter(uint32_t, uint32_t v) const {
    if (dists[v] < last_sent[v]) {
      last_sent[v] = dists[v];
      return true;
    }
    return false;
  }
  __device__ uint32_t peer_id(uint32_t v, uint32_t, uint32_t) const { return v; }
};

// a dense superstep's relaxations accept nothing (output listed afterwards)
template <class T>
__device__ __forceinline__ bool expand_quiet(const SsspDev<T>& f) { return f.red != 0; }

// batched relaxation: the frozen source distances, weights and current
// destination distances of the whole batch are loaded first (independent
// loads in flight), then the improving arcs issue their atomicMin together
template <int K, class T>
__device__ __forceinline__ void visit_batch(const SsspDev<T>& f, const uint32_t* src,
                                            const uint32_t* nb, const uint32_t* eid,
                                            const bool* pass, bool* acc) {
  T nd[K], cur[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    nd[k] = pass[k] ? __ldg(&f.fdist[src[k]]) + (T)ld_stream(&f.w[eid[k]]) : (T)0;
    cur[k] = pass[k] ? __ldcg(&f.dists[nb[k]]) : (T)0;
  }
  if (f.red) {  // no return value: RED, the thread does not wait for the L2
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (pass[k] && nd[k] < cur[k]) atomicMin(&f.dists[nb[k]], nd[k]);
      acc[k] = false;
    }
    return;
  }
  T old[K];
#pragma unroll
  for (int k = 0; k < K; ++k)
    old[k] = pass[k] && nd[k] < cur[k] ? atomicMin(&f.dists[nb[k]], nd[k]) : (T)0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    acc[k] = pass[k] && nd[k] < cur[k] && nd[k] < old[k];
    if (acc[k] && f.mark_preds) f.preds[nb[k]] = f.ow.to_global(src[k]);
  }
}

template <class T>
__global__ void snapshot_kernel(const uint32_t* __restrict__ in, uint32_t n, const T* dists,
                                T* fdist) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t u = in[i];
    fdist[u] = dists[u];
  }
}

// output frontier of a dense superstep, listed in ID order with one global
// atomic per CTA per round, 4 vertices per thread: P(q) is the 4-bit mask of
// vertices 4q..4q+3 that belong to it
//  * SSSP: the distance fell below the snapshot taken at the superstep's start
//    (= the vertices some arc improved, each once)
//  * BC forward: the vertex was labelled in this superstep
struct SsspFell {
  const uint32_t* d;
  const uint32_t* snap;
  __device__ uint32_t operator()(uint32_t q) const {
    const uint4 a = __ldcs(reinterpret_cast<const uint4*>(d) + q);
    const uint4 b = __ldcs(reinterpret_cast<const uint4*>(snap) + q);
    return (a.x < b.x) | (a.y < b.y) << 1 | (a.z < b.z) << 2 | (a.w < b.w) << 3;
  }
  __device__ bool one(uint32_t v) const { return d[v] < snap[v]; }
};
struct LabelIs {
  const uint32_t* labels;
  uint32_t level;
  __device__ uint32_t operator()(uint32_t q) const {
    const uint4 a = __ldcs(reinterpret_cast<const uint4*>(labels) + q);
    return (a.x == level) | (a.y == level) << 1 | (a.z == level) << 2 | (a.w == level) << 3;
  }
  __device__ bool one(uint32_t v) const { return labels[v] == level; }
};

template <class Pred>
__global__ void __launch_bounds__(256)
    dense_list_kernel(Pred pred, uint32_t nv, uint32_t* out, uint32_t* cnt) {
  __shared__ uint32_t s_warp[8];
  __shared__ uint32_t s_base;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t nq = (nv + 3) / 4;
  for (uint32_t base = blockIdx.x * 256; base < nq; base += gridDim.x * 256) {
    const uint32_t q = base + threadIdx.x;
    uint32_t m = 0;
    if (q < nq) {
      if (4 * q + 3 < nv) {
        m = pred(q);
      } else {
        for (uint32_t k = 0; 4 * q + k < nv; ++k) m |= (uint32_t)pred.one(4 * q + k) << k;
      }
    }
    const uint32_t c = __popc(m);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t run = 0;
      for (int k = 0; k < 8; ++k) {
        const uint32_t t = s_warp[k];
        s_warp[k] = run;
        run += t;
      }
      s_base = run ? atomicAdd(cnt, run) : 0u;
    }
    __syncthreads();
    uint32_t o = s_base + s_warp[warp] + x - c;
    while (m) {
      out[o++] = 4 * q + (__ffs(m) - 1);
      m &= m - 1;
    }
    __syncthreads();
  }
}

__global__ void widen_dist_kernel(const uint32_t* __restrict__ d32, uint32_t n,
                                  unsigned long long* d64) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t d = d32[i];
    d64[i] = d == kInfLabel ? ~0ull : (unsigned long long)d;
  }
}

struct SsspPrim : PrimBase {
  uint32_t source;
  bool mark_preds;
  bool narrow = false;  // u32 distances (decided per run from the plan's max weight)
  SsspPrim(uint32_t s, bool m) : source(s), mark_preds(m) {
    name = "sssp";
    nva = m ? 1 : 0;
    nvv = 1;
    allow_comm_override = true;
  }
  void init(Ctx& c) {  // primitives.cpp:323-332
    Worker& w = *c.w;
    narrow = (uint64_t)c.P->max_weight * ((uint64_t)c.P->nv + 1) < 0xFFFFFFFFull;
    if (narrow) {
      fill(w.su32[0], w.nv, 0xFF, w.stream);  // dists
      fill(w.su32[3], w.nv, 0xFF, w.stream);  // frontier_dist
      fill(w.aux[5], w.nv, 0xFF, w.stream);   // last_sent
      MGB_LAUNCH(set_one_kernel<uint32_t>, 1, 1, 0, w.stream, w.su32[0].ptr, source, 0u);
    } else {
      fill(w.su64[0], w.nv, 0xFF, w.stream);  // dists
      fill(w.su64[1], w.nv, 0xFF, w.stream);  // frontier_dist
      fill(w.su64[2], w.nv, 0xFF, w.stream);  // last_sent
      MGB_LAUNCH(set_one_kernel<unsigned long long>, 1, 1, 0, w.stream, w.su64[0].ptr, source,
                 0ull);
    }
    fill(w.su32[2], w.nv / 32 + 1, 0, w.stream);  // output dedup bitmap (cleared per superstep)
    if (mark_preds) fill(w.su32[1], w.nv, 0xFF, w.stream);
    if (c.P->owner_host[source] == w.p) c.push_initial({source});
  }
  SsspDev<uint32_t> dev32(Ctx& c) {
    Worker& w = *c.w;
    return {w.su32[0].ptr, w.su32[3].ptr, w.aux[5].ptr, w.su32[1].ptr, w.su32[2].ptr,
            w.w.ptr, c.owner_view(), (uint32_t)c.iter, mark_preds ? 1 : 0};
  }
  SsspDev<unsigned long long> dev64(Ctx& c) {
    Worker& w = *c.w;
    return {w.su64[0].ptr, w.su64[1].ptr, w.su64[2].ptr, w.su32[1].ptr, w.su32[2].ptr,
            w.w.ptr, c.owner_view(), (uint32_t)c.iter, mark_preds ? 1 : 0};
  }
  // a superstep whose frontier holds at least nv / kSsspDenseDiv vertices runs
  // dense (SsspDev::red) when there is one partition, no predecessor output and
  // the fused policy (its output buffer is sized for the superstep's bound)
  static constexpr uint32_t kSsspDenseDiv = MG_SSSP_DENSE_DIV;
  void body(Ctx& c) {
    Worker& w = *c.w;
    if (narrow && c.fused && c.num_workers() == 1 && !mark_preds && kSsspDenseDiv &&
        (uint64_t)c.in_count * kSsspDenseDiv >= w.nv) {
      // full snapshot (it is the frozen source distance of every frontier vertex)
      MGB_CUDA(cudaMemcpyAsync(w.su32[3].ptr, w.su32[0].ptr, 4ull * w.nv,
                               cudaMemcpyDeviceToDevice, w.stream));
      SsspDev<uint32_t> f = dev32(c);
      f.red = 1;
      c.pipeline(f, w.nv);
      MGB_LAUNCH(dense_list_kernel<SsspFell>, grid_for((w.nv + 3) / 4, 256, num_sms() * 8), 256,
                 0, w.stream, SsspFell{w.su32[0].ptr, w.su32[3].ptr}, w.nv, w.output.ptr,
                 &c.ctr()->out_cnt);
      return;
    }
    if (c.iter > 0)
      MGB_CUDA(cudaMemsetAsync(w.su32[2].ptr, 0, 4ull * (w.nv / 32 + 1), w.stream));
    if (narrow) {
      if (c.in_count)
        MGB_LAUNCH(snapshot_kernel<uint32_t>, grid_for(c.in_count, 256), 256, 0, w.stream,
                   w.input.ptr, c.in_count, w.su32[0].ptr, w.su32[3].ptr);
      c.pipeline(dev32(c), w.nv);
    } else {
      if (c.in_count)
        MGB_LAUNCH(snapshot_kernel<unsigned long long>, grid_for(c.in_count, 256), 256, 0,
                   w.stream, w.input.ptr, c.in_count, w.su64[0].ptr, w.su64[1].ptr);
      c.pipeline(dev64(c), w.nv);
    }
  }
  void finalize(Ctx& c, const GlobalView&) {
    Worker& w = *c.w;
    if (!narrow) return;
    if (w.su64[0].n < w.nv || !w.su64[0].ptr) w.su64[0].alloc(w.nv ? w.nv : 1);
    if (w.nv)
      MGB_LAUNCH(widen_dist_kernel, grid_for(w.nv, 256, num_sms() * 8), 256, 0, w.stream,
                 w.su32[0].ptr, w.nv, w.su64[0].ptr);
  }
};

// ===========================================================================
// CC (primitives.cpp:416-495)

struct CcDev {
  uint32_t* comp;
  uint32_t* snapshot;
  __device__ bool visit(uint32_t, uint32_t, uint32_t) const { return false; }
  __device__ bool keep(uint32_t) const { return true; }
  __device__ bool prefilter(uint32_t) const { return true; }
  __device__ bool combine(uint32_t v, const uint32_t* va, const double*, uint32_t) const {
    uint32_t c = va[0];
    if (c >= __ldcg(&comp[v])) return false;  // comp only falls: no atomic for a no-op
    uint32_t old = atomicMin(&comp[v], c);
    if (c < old) {
      atomicMin(&snapshot[v], c);  // the sender already broadcast it to everyone
      return true;
    }
    return false;
  }
  __device__ void gather(uint32_t v, uint32_t* va, double*) const { va[0] = comp[v]; }
  __device__ bool send_filter(uint32_t, uint32_t) const { return true; }
  __device__ uint32_t peer_id(uint32_t v, uint32_t, uint32_t) const { return v; }
};

__device__ __forceinline__ uint32_t cc_root(const uint32_t* comp, uint32_t x) {
  uint32_t y = comp[x];
  while (y != x) {
    x = y;
    y = comp[x];
  }
  return x;
}

// hook the larger root under the smaller over every hosted arc (primitives.cpp:443-455)
__global__ void __launch_bounds__(256)
    cc_hook_kernel(GraphView g, const uint32_t* __restrict__ hosted, uint32_t nh, uint32_t* comp,
                   uint32_t* hooked) {
  // one warp per hosted vertex: lanes stride its arcs
  const uint32_t warps = gridDim.x * blockDim.x / 32;
  uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  bool any = false;
  for (uint32_t i = wid; i < nh; i += warps) {
    uint32_t u = hosted[i];
    uint32_t b = g.off[u], e = g.off[u + 1];
    for (uint32_t k = b + lane_id(); k < e; k += 32) {
      uint32_t v = g.col[k];
      uint32_t ru = cc_root(comp, u), rv = cc_root(comp, v);
      if (ru == rv) continue;
      uint32_t hi = ru > rv ? ru : rv, lo = ru < rv ? ru : rv;
      atomicMin(&comp[hi], lo);
      any = true;
    }
  }
  if (__any_sync(__activemask(), any) && lane_id() == 0) *hooked = 1;
}

// full pointer jumping over every local vertex (primitives.cpp:456-457)
__global__ void cc_jump_kernel(uint32_t* comp, uint32_t nv) {
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nv; w += gridDim.x * blockDim.x)
    comp[w] = cc_root(comp, w);
}

// delta encoding: emit local vertices whose value changed since the snapshot
// (CTA-aggregated appends: one global atomic per CTA round; with
// write_list == 0 the changed vertices are only counted)
__global__ void __launch_bounds__(256)
    cc_delta_kernel(uint32_t* comp, uint32_t* snapshot, uint32_t nv, uint32_t* out,
                    Counters* ctr, int write_list) {
  using Scan = cub::BlockScan<uint32_t, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint32_t s_base;
  for (uint32_t base = blockIdx.x * blockDim.x; base < nv; base += gridDim.x * blockDim.x) {
    uint32_t w = base + threadIdx.x;
    uint32_t ch = 0;
    if (w < nv) {
      uint32_t c = comp[w];
      ch = c != snapshot[w];
      if (ch) snapshot[w] = c;
    }
    uint32_t excl, total;
    Scan(tmp).ExclusiveSum(ch, excl, total);
    if (threadIdx.x == 0) s_base = total ? atomicAdd(&ctr->out_cnt, total) : 0u;
    __syncthreads();
    if (ch && write_list) out[s_base + excl] = w;
    __syncthreads();
  }
}

// A single Duplicate-All partition may keep its gather-heavy state (PageRank,
// CC) in the FIFO-BFS locality order of bfs_locality_order; the transpose
// built for it (rows = vertices in that order, arcs = in-neighbours) is shared.
bool ordered_layout(const Plan& P) { return P.n == 1 && P.dup == MG_DUP_ALL; }
void ensure_transpose(Plan& P, Worker& w);  // defined with the PageRank kernels

__global__ void iperm_kernel(const uint32_t* __restrict__ perm, uint32_t n, uint32_t* iperm) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    iperm[perm[v]] = v;
}

// hook over the ordered arcs (the arc set is the sub-graph's, so the union is
// the same): 8 lanes per row, same larger-root-under-smaller rule
constexpr int kCcGroup = 8;
__global__ void __launch_bounds__(256)
    cc_hook_rows_kernel(const uint32_t* __restrict__ toff, const uint32_t* __restrict__ tcol,
                        uint32_t nv, uint32_t* comp, uint32_t* hooked) {
  const unsigned sub = threadIdx.x & (kCcGroup - 1);
  const uint32_t groups = gridDim.x * (blockDim.x / kCcGroup);
  bool any = false;
  for (uint32_t u = blockIdx.x * (blockDim.x / kCcGroup) + threadIdx.x / kCcGroup; u < nv;
       u += groups) {
    const uint32_t b = toff[u], e = toff[u + 1];
    for (uint32_t k = b + sub; k < e; k += kCcGroup) {
      const uint32_t v = __ldg(&tcol[k]);
      uint32_t ru = cc_root(comp, u), rv = cc_root(comp, v);
      if (ru == rv) continue;
      uint32_t hi = ru > rv ? ru : rv, lo = ru < rv ? ru : rv;
      atomicMin(&comp[hi], lo);
      any = true;
    }
  }
  if (__any_sync(0xffffffffu, any) && lane_id() == 0) *hooked = 1;
}

// --- sampled hooking (Afforest-style) for a symmetric single partition -----
// 1. link every vertex to its first kCcLink neighbours, compress;
// 2. sample roots, the most frequent one is the giant component's;
// 3. hook sweeps over the arcs of the vertices NOT in the giant (after step 1)
//    until no hook.  On a symmetric graph every arc between the giant and
//    another tree is also an arc of the other tree's vertex, so skipping the
//    giant's rows loses no union; the fixpoint (every set's minimum) is the
//    same as the reference's full sweeps, so labels are identical.
constexpr uint32_t kCcLink = 2;
constexpr uint32_t kCcSamples = 1024;

__global__ void __launch_bounds__(256)
    cc_link_kernel(const uint32_t* __restrict__ toff, const uint32_t* __restrict__ tcol,
                   uint32_t nv, uint32_t* comp) {
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < nv; u += gridDim.x * blockDim.x) {
    const uint32_t b = toff[u], e = toff[u + 1];
    for (uint32_t k = b; k < e && k < b + kCcLink; ++k) {
      uint32_t ru = cc_root(comp, u), rv = cc_root(comp, __ldg(&tcol[k]));
      if (ru == rv) continue;
      atomicMin(&comp[ru > rv ? ru : rv], ru < rv ? ru : rv);
    }
  }
}

__global__ void cc_sample_kernel(const uint32_t* comp, uint32_t nv, uint32_t* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < kCcSamples) out[i] = comp[(uint32_t)(((uint64_t)i * 2654435761ull) % nv)];
}

__global__ void __launch_bounds__(256)
    cc_hook_rest_kernel(const uint32_t* __restrict__ toff, const uint32_t* __restrict__ tcol,
                        uint32_t nv, const uint32_t* __restrict__ comp0, uint32_t giant,
                        uint32_t* comp, uint32_t* hooked, unsigned long long* scanned_out) {
  const unsigned sub = threadIdx.x & (kCcGroup - 1);
  const uint32_t groups = gridDim.x * (blockDim.x / kCcGroup);
  bool any = false;
  uint32_t scanned = 0;
  for (uint32_t u = blockIdx.x * (blockDim.x / kCcGroup) + threadIdx.x / kCcGroup; u < nv;
       u += groups) {
    if (comp0[u] == giant) continue;
    const uint32_t b = toff[u], e = toff[u + 1];
    if (sub == 0) scanned += e - b;
    for (uint32_t k = b + sub; k < e; k += kCcGroup) {
      uint32_t ru = cc_root(comp, u), rv = cc_root(comp, __ldg(&tcol[k]));
      if (ru == rv) continue;
      atomicMin(&comp[ru > rv ? ru : rv], ru < rv ? ru : rv);
      any = true;
    }
  }
  if (__any_sync(0xffffffffu, any) && lane_id() == 0) *hooked = 1;
  if (scanned_out) warp_add_u64(scanned_out, scanned);
}

// is the (ordered) transpose symmetric?  every arc (u <- v) needs (v <- u):
// a binary search in v's sorted row; any miss clears *sym
__global__ void __launch_bounds__(256)
    cc_symmetric_kernel(const uint32_t* __restrict__ toff, const uint32_t* __restrict__ tcol,
                        uint32_t nv, uint32_t* sym) {
  const uint32_t warps = gridDim.x * blockDim.x / 32;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) / 32; u < nv; u += warps) {
    for (uint32_t k = toff[u] + lane_id(); k < toff[u + 1]; k += 32) {
      const uint32_t v = tcol[k];
      uint32_t lo = toff[v], hi = toff[v + 1];
      while (lo < hi) {
        const uint32_t m = (lo + hi) >> 1;
        if (tcol[m] < u) lo = m + 1;
        else hi = m;
      }
      if (lo == toff[v + 1] || tcol[lo] != u) *sym = 0u;
    }
  }
}

// labels back in vertex IDs: the component label is its smallest vertex ID.
// Each CTA walks a contiguous range of ordered positions; runs of equal roots
// are min-reduced by shuffles, the CTA's first root in shared memory, so the
// giant component's root sees one global atomic per CTA, not one per vertex.
__global__ void __launch_bounds__(256)
    cc_min_id_kernel(const uint32_t* __restrict__ comp_p, const uint32_t* __restrict__ iperm,
                     uint32_t n, uint32_t* minid) {
  __shared__ uint32_t s_root, s_min;
  const uint32_t per = (n + gridDim.x - 1) / gridDim.x;
  const uint32_t lo = blockIdx.x * per, hi = lo + per < n ? lo + per : n;
  if (lo >= hi) return;
  if (threadIdx.x == 0) {
    s_root = comp_p[lo];
    s_min = 0xFFFFFFFFu;
  }
  __syncthreads();
  const unsigned lane = lane_id();
  for (uint32_t base = lo; base < hi; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const bool ok = i < hi;
    const uint32_t r = ok ? comp_p[i] : 0xFFFFFFFFu;
    uint32_t m = ok ? iperm[i] : 0xFFFFFFFFu;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t om = __shfl_down_sync(0xffffffffu, m, o);
      const uint32_t orr = __shfl_down_sync(0xffffffffu, r, o);
      if (lane + o < 32 && orr == r) m = om < m ? om : m;
    }
    const uint32_t pr = __shfl_up_sync(0xffffffffu, r, 1);
    if (ok && (lane == 0 || pr != r)) {
      if (r == s_root) atomicMin(&s_min, m);
      else atomicMin(&minid[r], m);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMin(&minid[s_root], s_min);
}
// gather form: coalesced writes in vertex order, random reads of comp_p
__global__ void cc_labels_kernel(const uint32_t* __restrict__ comp_p,
                                 const uint32_t* __restrict__ perm,
                                 const uint32_t* __restrict__ minid, uint32_t n, uint32_t* comp) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    comp[v] = minid[comp_p[perm[v]]];
}

struct CcPrim : PrimBase {
  DevArray<uint32_t>* flag = nullptr;
  CcPrim() {
    name = "cc";
    nva = 1;
    communication = MG_COMM_BROADCAST;
  }
  // single partition: components computed in the locality order (comp_p in
  // aux[5], snapshot in su32[1]); labels mapped back to vertex IDs at the end
  bool ordered = false;
  uint32_t* comp_arr(Worker& w) { return ordered ? w.aux[5].ptr : w.su32[0].ptr; }
  void init(Ctx& c) {  // primitives.cpp:425-434
    Worker& w = *c.w;
    ordered = ordered_layout(*c.P) && w.nv > 0;
    if (ordered) ensure_transpose(*c.P, w);  // plan lifetime
    if (w.su32[0].n < w.nv || !w.su32[0].ptr) w.su32[0].alloc(w.nv ? w.nv : 1);
    if (w.su32[1].n < w.nv || !w.su32[1].ptr) w.su32[1].alloc(w.nv ? w.nv : 1);
    if (ordered && (w.aux[5].n < w.nv || !w.aux[5].ptr)) w.aux[5].alloc(w.nv);
    if (!w.su32[3].ptr) w.su32[3].alloc(1);
    if (w.nv) {
      MGB_LAUNCH(iota_kernel, grid_for(w.nv, 256), 256, 0, w.stream, comp_arr(w), w.nv);
      MGB_CUDA(cudaMemcpyAsync(w.su32[1].ptr, comp_arr(w), 4ull * w.nv,
                               cudaMemcpyDeviceToDevice, w.stream));
    }
    // a non-empty initial frontier keeps superstep 0 alive
    uint32_t nh = (uint32_t)w.hosted_host.size();
    uint32_t& nc = c.run->next_count[w.p];
    w.next_input.ensure(nh, w.stream);
    if (nh)
      MGB_CUDA(cudaMemcpyAsync(w.next_input.ptr, w.hosted.ptr, 4ull * nh,
                               cudaMemcpyDeviceToDevice, w.stream));
    nc = nh;
  }
  CcDev dev(Ctx& c) { return {c.w->su32[0].ptr, c.w->su32[1].ptr}; }
  // several partitions: a delta of more than half the vertices goes to the
  // peers as the whole comp[] array (4 B/vertex instead of 8 B/record); the
  // receivers' min-combine turns the exchange into an all-gather + MIN
  // reduction (engine.cuh DenseView)
  DenseView dense_view(Ctx& c) const {
    if (ordered) return {};
    DenseView d;
    d.kind = 2;
    d.cur = c.w->su32[0].ptr;
    d.words = c.w->nv;
    d.threshold = c.w->nv / 2 + 1;
    return d;
  }
  void body(Ctx& c) {  // primitives.cpp:436-472: local fixpoint, then delta
    Worker& w = *c.w;
    uint32_t nh = (uint32_t)w.hosted_host.size();
    uint32_t* hooked = w.su32[3].ptr;
    uint32_t h = 1;
    uint64_t scanned = 0;
    const uint64_t local_edges = w.ne;  // every hosted arc once per hook pass
    uint32_t* comp = comp_arr(w);
    if (ordered && c.P->n == 1) {
      // one partition receives nothing, so superstep 0's fixpoint is final.
      // W keeps the reference's unit, |E_i| per hook sweep (primitives.cpp:
      // 441-457): the sampled fixpoint counts its link pass plus its rest
      // sweeps; a later superstep counts the one confirming sweep the
      // reference runs on its own output (it can hook nothing, so it is not run)
      if (c.iter == 0) {
        if (symmetric(w)) {
          scanned = sampled_fixpoint(c, comp) * local_edges;
          h = 0;
        }
      } else {
        scanned = local_edges;
        h = 0;
      }
    }
    while (h) {
      MGB_CUDA(cudaMemsetAsync(hooked, 0, 4, w.stream));
      if (ordered)
        MGB_LAUNCH(cc_hook_rows_kernel, grid_for((uint64_t)w.nv * kCcGroup, 256, num_sms() * 16),
                   256, 0, w.stream, w.toff.ptr, w.tcol.ptr, w.nv, comp, hooked);
      else if (nh)
        MGB_LAUNCH(cc_hook_kernel, grid_for((uint64_t)nh * 32, 256, num_sms() * 16), 256, 0,
                   w.stream, w.graph(), w.hosted.ptr, nh, comp, hooked);
      if (w.nv)
        MGB_LAUNCH(cc_jump_kernel, grid_for(w.nv, 256, num_sms() * 16), 256, 0, w.stream, comp,
                   w.nv);
      MGB_CUDA(cudaMemcpyAsync(&h, hooked, 4, cudaMemcpyDeviceToHost, w.stream));
      MGB_CUDA(cudaStreamSynchronize(w.stream));
      scanned += local_edges;
    }
    c.ensure_output(w.nv);
    if (w.nv)
      MGB_LAUNCH(cc_delta_kernel, grid_for(w.nv, 256, num_sms() * 8), 256, 0, w.stream, comp,
                 w.su32[1].ptr, w.nv, w.output.ptr, c.ctr(),
                 (c.P->n > 1 || c.want_deg) ? 1 : 0);  // one partition: only the count is read
    add_edges(c, scanned);
  }
  void finalize(Ctx& c, const GlobalView&) {
    Worker& w = *c.w;
    if (!ordered) return;
    MGB_CUDA(cudaMemsetAsync(w.su32[1].ptr, 0xFF, 4ull * w.nv, w.stream));  // min vertex ID
    MGB_LAUNCH(cc_min_id_kernel, grid_for(w.nv, 256, num_sms() * 4), 256, 0, w.stream,
               w.aux[5].ptr, w.pr_iperm.ptr, w.nv, w.su32[1].ptr);
    MGB_LAUNCH(cc_labels_kernel, grid_for(w.nv, 256, num_sms() * 8), 256, 0, w.stream,
               w.aux[5].ptr, w.pr_perm.ptr, w.su32[1].ptr, w.nv, w.su32[0].ptr);
  }
  static void add_edges(Ctx& c, uint64_t k);
  // plan lifetime: is the ordered transpose symmetric (sampled hooking valid)?
  static bool symmetric(Worker& w) {
    if (w.cc_symmetric < 0) {
      DevArray<uint32_t> f;
      f.alloc(1);
      uint32_t one = 1;
      MGB_CUDA(cudaMemcpy(f.ptr, &one, 4, cudaMemcpyHostToDevice));
      MGB_LAUNCH(cc_symmetric_kernel, grid_for((uint64_t)w.nv * 32, 256, num_sms() * 16), 256, 0,
                 w.stream, w.toff.ptr, w.tcol.ptr, w.nv, f.ptr);
      MGB_CUDA(cudaMemcpyAsync(&one, f.ptr, 4, cudaMemcpyDeviceToHost, w.stream));
      MGB_CUDA(cudaStreamSynchronize(w.stream));
      w.cc_symmetric = one ? 1 : 0;
    }
    return w.cc_symmetric == 1;
  }
  // returns the number of sweeps (link pass + rest sweeps, the last finding no hook)
  uint64_t sampled_fixpoint(Ctx& c, uint32_t* comp) {
    Worker& w = *c.w;
    const unsigned g = grid_for(w.nv, 256, num_sms() * 16);
    MGB_LAUNCH(cc_link_kernel, g, 256, 0, w.stream, w.toff.ptr, w.tcol.ptr, w.nv, comp);
    MGB_LAUNCH(cc_jump_kernel, g, 256, 0, w.stream, comp, w.nv);
    if (w.aux[4].n < w.nv || !w.aux[4].ptr) w.aux[4].alloc(w.nv);  // roots after linking
    if (w.aux[3].n < kCcSamples || !w.aux[3].ptr) w.aux[3].alloc(kCcSamples);
    MGB_CUDA(cudaMemcpyAsync(w.aux[4].ptr, comp, 4ull * w.nv, cudaMemcpyDeviceToDevice,
                             w.stream));
    MGB_LAUNCH(cc_sample_kernel, kCcSamples / 256, 256, 0, w.stream, comp, w.nv, w.aux[3].ptr);
    std::vector<uint32_t> smp(kCcSamples);
    MGB_CUDA(cudaMemcpyAsync(smp.data(), w.aux[3].ptr, 4ull * kCcSamples,
                             cudaMemcpyDeviceToHost, w.stream));
    MGB_CUDA(cudaStreamSynchronize(w.stream));
    std::sort(smp.begin(), smp.end());
    uint32_t giant = smp[0], best = 0;
    for (size_t i = 0; i < smp.size();) {
      size_t j = i;
      while (j < smp.size() && smp[j] == smp[i]) ++j;
      if (j - i > best) {
        best = (uint32_t)(j - i);
        giant = smp[i];
      }
      i = j;
    }
    uint32_t* hooked = w.su32[3].ptr;
    uint64_t sweeps = 1;  // the link pass
    for (uint32_t h = 1; h; ++sweeps) {
      MGB_CUDA(cudaMemsetAsync(hooked, 0, 4, w.stream));
      MGB_LAUNCH(cc_hook_rest_kernel, grid_for((uint64_t)w.nv * kCcGroup, 256, num_sms() * 16),
                 256, 0, w.stream, w.toff.ptr, w.tcol.ptr, w.nv, w.aux[4].ptr, giant, comp,
                 hooked, (unsigned long long*)nullptr);
      MGB_LAUNCH(cc_jump_kernel, g, 256, 0, w.stream, comp, w.nv);
      MGB_CUDA(cudaMemcpyAsync(&h, hooked, 4, cudaMemcpyDeviceToHost, w.stream));
      MGB_CUDA(cudaStreamSynchronize(w.stream));
    }
    return sweeps;
  }
};

__global__ void add_u64_kernel(unsigned long long* dst, unsigned long long v) { *dst += v; }

void CcPrim::add_edges(Ctx& c, uint64_t k) {
  if (k) MGB_LAUNCH(add_u64_kernel, 1, 1, 0, c.w->stream, &c.ctr()->edges, k);
}

// ===========================================================================
// BC (primitives.cpp:518-680)

enum : uint64_t { kFwd = 0, kBwd = 1, kDone = 2 };

struct BcDev {
  uint32_t* labels;
  double* sigma;
  double* delta;
  uint32_t* bstamp;
  double* coef;
  OwnerView ow;
  uint32_t iter;
  int phase;
  // dense forward superstep (one partition): a vertex not labelled before
  // this superstep gets a plain store of the level (every writer stores the
  // same value) and the sigma addition, nothing is accepted; the output is
  // listed by dense_list_kernel<LabelIs> afterwards
  int red = 0;
  // forward visit (primitives.cpp:559-567): sigma counts are integers, so the
  // order of the atomic additions does not change the result
  __device__ bool visit(uint32_t u, uint32_t v, uint32_t) const {
    uint32_t cand = iter + 1;
    uint32_t old = labels[v];
    if (old == kInfLabel) old = atomicCAS(&labels[v], kInfLabel, cand);
    if (old == kInfLabel || old == cand) atomicAdd(&sigma[v], sigma[u]);
    return old == kInfLabel;
  }
  // the claiming CAS accepts each vertex exactly once per superstep, so the
  // output needs no second dedup (the per-vertex stamp cost an atomic and 4
  // bytes of random L2 traffic per discovery)
  __device__ bool keep(uint32_t) const { return true; }
  __device__ bool prefilter(uint32_t) const { return true; }
  __device__ bool combine(uint32_t v, const uint32_t*, const double* vv, uint32_t it) const {
    if (phase == kFwd) {  // primitives.cpp:639-648
      uint32_t cand = it + 1;
      uint32_t old = atomicMin(&labels[v], cand);
      if (old >= cand) atomicAdd(&sigma[v], vv[0]);  // label was inf => sigma was 0
      return old > cand && ow.hosts(v);
    }
    sigma[v] = vv[0];  // dependency phase (primitives.cpp:650-653)
    delta[v] = vv[1];
    bstamp[v] = it + 1;
    coef[v] = (1.0 + vv[1]) / vv[0];  // the proxy's successor coefficient
    return false;
  }
  __device__ void gather(uint32_t v, uint32_t*, double* vv) const {
    vv[0] = sigma[v];
    if (phase == kFwd) {
      vv[1] = 0.0;
      sigma[v] = 0.0;  // partial shipped; reset the proxy accumulator
    } else {
      vv[1] = delta[v];
    }
  }
  __device__ bool send_filter(uint32_t, uint32_t) const { return true; }
  __device__ uint32_t peer_id(uint32_t v, uint32_t, uint32_t) const { return v; }
};

// a dense forward superstep accepts nothing (output listed afterwards)
__device__ __forceinline__ bool expand_quiet(const BcDev& f) { return f.red != 0; }
}  // namespace
#ifndef MG_BC_LONG_ROWS
#define MG_BC_LONG_ROWS 0
#endif
template <>
struct expand_long_rows<BcDev> {
  static constexpr bool value = MG_BC_LONG_ROWS;
};
namespace {

// batched forward visit: label loads, then the claiming CASes, then the sigma
// additions of the whole batch, each group in flight together
template <int K>
__device__ __forceinline__ void visit_batch(const BcDev& f, const uint32_t* src,
                                            const uint32_t* nb, const uint32_t*,
                                            const bool* pass, bool* acc) {
  const uint32_t cand = f.iter + 1;
  uint32_t old[K];
  double su[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    old[k] = pass[k] ? __ldcg(&f.labels[nb[k]]) : 0u;
    su[k] = pass[k] ? f.sigma[src[k]] : 0.0;
  }
  if (f.red) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (pass[k] && (old[k] == kInfLabel || old[k] == cand)) {
        if (old[k] == kInfLabel) __stcg(&f.labels[nb[k]], cand);
        atomicAdd(&f.sigma[nb[k]], su[k]);
      }
      acc[k] = false;
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (pass[k] && old[k] == kInfLabel) old[k] = atomicCAS(&f.labels[nb[k]], kInfLabel, cand);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (pass[k] && (old[k] == kInfLabel || old[k] == cand)) atomicAdd(&f.sigma[nb[k]], su[k]);
    acc[k] = pass[k] && old[k] == kInfLabel;
  }
}

__global__ void max_hosted_label_kernel(const uint32_t* labels, const uint32_t* hosted,
                                        uint32_t nh, Counters* ctr) {
  uint32_t m = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nh; i += gridDim.x * blockDim.x) {
    uint32_t l = labels[hosted[i]];
    if (l != kInfLabel && l > m) m = l;
  }
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane_id() == 0 && m) atomicMax(&ctr->u[0], (unsigned long long)m);
}

// backward level step (primitives.cpp:592-617), in two kernels:
//   select: hosted vertices of the level -> the level list (also the output
//           broadcast of the superstep) split by degree;
//   accumulate: rows below kBcWarpDeg by one thread walking its arcs in order,
//           longer rows by a warp (lane-strided partial sums, fixed xor-tree
//           reduction: deterministic).
// Successor coefficients: once a vertex's dependency is final its coefficient
// coef[w] = (1 + delta[w]) / sigma[w] is stored — by the select pass of the
// NEXT (shallower) level for hosted vertices, on receipt of the owner's
// broadcast for proxies — so
//   delta[v] = sigma[v] * sum over arcs (v,w) of coef[w]
// needs ONE random 8-byte load per arc.  No mask is needed: while level L is
// processed only levels > L carry coefficients (levels finish from the
// deepest up, and level L's own are written only after its pass), and an arc
// from level L never reaches past L+1 (BFS levels), so every non-zero
// coefficient on a row of level L belongs to a successor — the reference's
// "label == L+1 / stamped by the last broadcast" test (primitives.cpp:600-610).  The factored sum differs from the
// reference's per-term sigma_v/sigma_w*(1+delta_w) by rounding only (~1e-16
// relative; the bar is 1e-5).
constexpr uint32_t kBcWarpDeg = 32;

__global__ void __launch_bounds__(256)
    bc_level_select_kernel(const uint32_t* __restrict__ hosted, uint32_t nh,
                           const uint32_t* __restrict__ labels, const uint32_t* __restrict__ off,
                           uint32_t level, uint32_t* out, Counters* ctr, uint32_t* small,
                           uint32_t* nsmall, uint32_t* big, uint32_t* nbig, int deepest,
                           const double* __restrict__ sigma, const double* __restrict__ delta,
                           double* coef) {
  for (uint32_t base = blockIdx.x * blockDim.x; base < nh; base += gridDim.x * blockDim.x) {
    uint32_t i = base + threadIdx.x;
    bool in = false, is_big = false;
    uint32_t v = 0;
    if (i < nh) {
      v = hosted[i];
      const uint32_t lv = labels[v];
      in = lv == level;
      if (in) is_big = off[v + 1] - off[v] >= kBcWarpDeg;
      if (in && deepest) coef[v] = 1.0 / sigma[v];  // delta = 0 on the deepest level
      else if (lv == level + 1 && !deepest) coef[v] = (1.0 + delta[v]) / sigma[v];
    }
    uint32_t s = warp_append(&ctr->out_cnt, in);
    if (in) out[s] = v;
    if (deepest) continue;
    s = warp_append(nsmall, in && !is_big);
    if (in && !is_big) small[s] = v;
    s = warp_append(nbig, in && is_big);
    if (in && is_big) big[s] = v;
  }
}

__device__ __forceinline__ void bc_finish(uint32_t v, uint32_t source, double sv, double acc,
                                          double* delta, double* bc) {
  const double dv = sv * acc;
  delta[v] = dv;
  if (v != source) bc[v] += dv;
}

__global__ void __launch_bounds__(256)
    bc_backward_thread_kernel(GraphView g, const uint32_t* __restrict__ list, const uint32_t* nlist,
                              uint32_t nfix, const double* __restrict__ sigma, double* delta,
                              double* bc, const double* __restrict__ coef, uint32_t source,
                              Counters* ctr) {
  const uint32_t n = nlist ? *nlist : nfix;
  unsigned long long scanned = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t v = list[i];
    const uint32_t b = g.off[v], e = g.off[v + 1];
    double acc = 0.0;
    uint32_t k = b;
    for (; k + 1 < e; k += 2) {  // two gathers in flight
      const double c0 = __ldg(&coef[__ldg(&g.col[k])]);
      const double c1 = __ldg(&coef[__ldg(&g.col[k + 1])]);
      acc += c0;
      acc += c1;
    }
    if (k < e) acc += __ldg(&coef[__ldg(&g.col[k])]);
    scanned += e - b;
    bc_finish(v, source, sigma[v], acc, delta, bc);
  }
  warp_add_u64(&ctr->edges, scanned);
}

__global__ void __launch_bounds__(256)
    bc_backward_warp_kernel(GraphView g, const uint32_t* __restrict__ list, const uint32_t* nlist,
                            uint32_t nfix, const double* __restrict__ sigma, double* delta,
                            double* bc, const double* __restrict__ coef, uint32_t source,
                            Counters* ctr) {
  const uint32_t n = nlist ? *nlist : nfix;
  const uint32_t warps = gridDim.x * blockDim.x / 32;
  unsigned long long scanned = 0;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / 32; i < n; i += warps) {
    const uint32_t v = list[i];
    const uint32_t b = g.off[v], e = g.off[v + 1];
    double acc = 0.0;
    for (uint32_t k = b + lane_id(); k < e; k += 32) acc += __ldg(&coef[__ldg(&g.col[k])]);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane_id() == 0) {
      scanned += e - b;
      bc_finish(v, source, sigma[v], acc, delta, bc);
    }
  }
  warp_add_u64(&ctr->edges, scanned);
}

// Level buckets for the backward phase: the hosted vertices are counting-
// sorted once by (label, long row) — bucket 2L: short rows of level L, 2L+1:
// long rows — so every backward superstep works on a contiguous slice
// instead of rescanning all hosted vertices per level.  Per-CTA shared
// histograms, one small scan (bucket-major), a scatter with shared cursors.
constexpr uint32_t kBcBuckets = 2048;  // kBcClasses * (max_level + 1) must fit
// row classes inside a level: thread rows, warp rows, and huge rows that are
// cut into kBcChunk-arc chunks over many CTAs (a hub row of 1e6 arcs on one
// warp left the GPU at 3.5% SM throughput for 2.7 ms)
constexpr uint32_t kBcClasses = 3;
constexpr uint32_t kBcHugeDeg = 8192;
constexpr uint32_t kBcChunk = 4096;
__device__ __forceinline__ uint32_t bc_row_class(uint32_t deg) {
  return deg < kBcWarpDeg ? 0u : (deg < kBcHugeDeg ? 1u : 2u);
}

// huge rows of a level: chunk prefix (one CTA; few rows), chunked sums with
// one f64 atomic per chunk, then the per-row finish
__global__ void __launch_bounds__(1024)
    bc_huge_prefix_kernel(const uint32_t* __restrict__ rows, uint32_t n,
                          const uint32_t* __restrict__ off, uint32_t* chunk_start,
                          double* acc) {
  using Scan = cub::BlockScan<uint32_t, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < n; base += 1024) {
    const uint32_t i = base + threadIdx.x;
    uint32_t c = 0;
    if (i < n) {
      const uint32_t v = rows[i];
      c = (off[v + 1] - off[v] + kBcChunk - 1) / kBcChunk;
      acc[i] = 0.0;
    }
    uint32_t excl, total;
    Scan(tmp).ExclusiveSum(c, excl, total);
    if (i < n) chunk_start[i] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) chunk_start[n] = carry;
}

__global__ void __launch_bounds__(256)
    bc_huge_chunks_kernel(GraphView g, const uint32_t* __restrict__ rows, uint32_t n,
                          const uint32_t* __restrict__ chunk_start,
                          const double* __restrict__ coef, double* acc) {
  using Reduce = cub::BlockReduce<double, 256>;
  __shared__ typename Reduce::TempStorage tmp;
  const uint32_t total = chunk_start[n];
  for (uint32_t c = blockIdx.x; c < total; c += gridDim.x) {
    uint32_t lo = 0, hi = n - 1;  // last row with chunk_start <= c
    while (lo < hi) {
      const uint32_t m = (lo + hi + 1) >> 1;
      if (chunk_start[m] <= c) lo = m;
      else hi = m - 1;
    }
    const uint32_t v = rows[lo];
    const uint32_t b = g.off[v] + (c - chunk_start[lo]) * kBcChunk;
    const uint32_t e = b + kBcChunk < g.off[v + 1] ? b + kBcChunk : g.off[v + 1];
    double sum = 0.0;
    for (uint32_t k = b + threadIdx.x; k < e; k += 256) sum += __ldg(&coef[ld_stream(&g.col[k])]);
    sum = Reduce(tmp).Sum(sum);
    if (threadIdx.x == 0) atomicAdd(&acc[lo], sum);
    __syncthreads();
  }
}

__global__ void bc_huge_finish_kernel(GraphView g, const uint32_t* __restrict__ rows, uint32_t n,
                                      const double* __restrict__ acc, const double* sigma,
                                      double* delta, double* bc, uint32_t source, Counters* ctr) {
  unsigned long long scanned = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t v = rows[i];
    const double dv = sigma[v] * acc[i];
    delta[v] = dv;
    if (v != source) bc[v] += dv;
    scanned += g.off[v + 1] - g.off[v];
  }
  warp_add_u64(&ctr->edges, scanned);
}
constexpr uint32_t kBcBucketCtas = kB200SMs * 4;

__global__ void __launch_bounds__(256)
    bc_bucket_count_kernel(const uint32_t* __restrict__ hosted, uint32_t nh,
                           const uint32_t* __restrict__ labels, const uint32_t* __restrict__ off,
                           uint32_t max_level, uint32_t nb, uint32_t* cta_hist) {
  __shared__ uint32_t h[kBcBuckets];
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const uint32_t per = (nh + gridDim.x - 1) / gridDim.x;
  const uint32_t lo = blockIdx.x * per, hi = lo + per < nh ? lo + per : nh;
  for (uint32_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint32_t v = hosted[i], l = labels[v];
    if (l <= max_level) atomicAdd(&h[kBcClasses * l + bc_row_class(off[v + 1] - off[v])], 1u);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) cta_hist[b * gridDim.x + blockIdx.x] = h[b];
}

// exclusive scan of the bucket-major CTA histogram in one CTA; bucket b starts
// at the scanned entry of (b, CTA 0), the total closes the table
__global__ void __launch_bounds__(1024)
    bc_bucket_scan_kernel(uint32_t* cta_hist, uint32_t nb, uint32_t nctas, uint32_t* start) {
  using Scan = cub::BlockScan<uint32_t, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint32_t carry;
  const uint32_t n = nb * nctas;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < n; base += 1024) {
    const uint32_t i = base + threadIdx.x;
    uint32_t d = i < n ? cta_hist[i] : 0u, excl, total;
    Scan(tmp).ExclusiveSum(d, excl, total);
    if (i < n) {
      cta_hist[i] = carry + excl;
      if (i % nctas == 0) start[i / nctas] = carry + excl;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) start[nb] = carry;
}

__global__ void __launch_bounds__(256)
    bc_bucket_scatter_kernel(const uint32_t* __restrict__ hosted, uint32_t nh,
                             const uint32_t* __restrict__ labels, const uint32_t* __restrict__ off,
                             uint32_t max_level, uint32_t nb, const uint32_t* __restrict__ cta_off,
                             uint32_t* out) {
  __shared__ uint32_t cur[kBcBuckets];
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) cur[b] = cta_off[b * gridDim.x + blockIdx.x];
  __syncthreads();
  const uint32_t per = (nh + gridDim.x - 1) / gridDim.x;
  const uint32_t lo = blockIdx.x * per, hi = lo + per < nh ? lo + per : nh;
  for (uint32_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint32_t v = hosted[i], l = labels[v];
    if (l <= max_level)
      out[atomicAdd(&cur[kBcClasses * l + bc_row_class(off[v + 1] - off[v])], 1u)] = v;
  }
}

// per backward superstep: the level's slice becomes the output (the broadcast
// of the superstep), the deepest level gets coef = 1/sigma, and the level
// below the current one (finished last superstep) gets its coefficients
__global__ void bc_level_prep_kernel(const uint32_t* __restrict__ list, uint32_t l0, uint32_t l1,
                                     uint32_t c0, uint32_t c1, int deepest,
                                     const double* __restrict__ sigma,
                                     const double* __restrict__ delta, double* coef, uint32_t* out,
                                     Counters* ctr) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = l0 + blockIdx.x * blockDim.x + threadIdx.x; i < l1; i += stride) {
    const uint32_t v = list[i];
    out[i - l0] = v;
    if (deepest) coef[v] = 1.0 / sigma[v];  // delta = 0 on the deepest level
  }
  for (uint32_t i = c0 + blockIdx.x * blockDim.x + threadIdx.x; i < c1; i += stride) {
    const uint32_t v = list[i];
    coef[v] = (1.0 + delta[v]) / sigma[v];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->out_cnt = l1 - l0;
}

#ifndef MG_BC_DENSE_DIV
#define MG_BC_DENSE_DIV 512  // RMAT-24 C5: off 7.24 ms, 32: 7.20, 512: 7.12, always: 7.14
#endif
// a forward superstep whose frontier holds at least |V| / kBcDenseDiv vertices
// runs dense (BcDev::red) on one partition under the fused policy
constexpr uint32_t kBcDenseDiv = MG_BC_DENSE_DIV;

struct BcPrim : PrimBase {
  uint32_t source;
  int phase = kFwd;
  uint32_t max_level = 0;
  uint64_t backward_from = 0;
  // per worker: level buckets built for this run, host copy of the bucket table
  std::vector<char> bucketed = std::vector<char>(kMaxWorkers, 0);
  std::vector<std::vector<uint32_t>> bucket_starts =
      std::vector<std::vector<uint32_t>>(kMaxWorkers);
  BcPrim(uint32_t s) : source(s) {
    name = "bc";
    nvv = 2;
    has_stop_condition = true;
  }
  uint64_t inbox_bound(Plan& P, uint32_t src, uint32_t dst, int) const {
    // forward: selective (|B|); backward: broadcast of one level of hosted vertices
    uint64_t a = P.pair_border[src][dst], b = P.nlocal[src];
    return a > b ? a : b;
  }
  void init(Ctx& c) {  // primitives.cpp:528-541
    Worker& w = *c.w;
    fill(w.su32[0], w.nv, 0xFF, w.stream);  // labels
    fill(w.su32[3], w.nv, 0, w.stream);     // bstamp
    fill(w.sf64[0], w.nv, 0, w.stream);     // sigma
    fill(w.sf64[1], w.nv, 0, w.stream);     // delta
    fill(w.sf64[2], w.nv, 0, w.stream);     // bc
    fill(w.sf64[3], w.nv, 0, w.stream);     // successor coefficients
    MGB_LAUNCH(set_one_kernel<uint32_t>, 1, 1, 0, w.stream, w.su32[0].ptr, source, 0u);
    if (c.P->owner_host[source] == w.p) {
      MGB_LAUNCH(set_one_kernel<double>, 1, 1, 0, w.stream, w.sf64[0].ptr, source, 1.0);
      c.push_initial({source});
    }
  }
  BcDev dev(Ctx& c) {
    Worker& w = *c.w;
    return {w.su32[0].ptr, w.sf64[0].ptr, w.sf64[1].ptr, w.su32[3].ptr, w.sf64[3].ptr,
            c.owner_view(), (uint32_t)c.iter, phase};
  }
  int phase_at_body = kFwd;
  void body(Ctx& c) {  // primitives.cpp:543-625
    Worker& w = *c.w;
    const bool first = c.worker() == c.P->local_workers.front();
    if (first && phase == kFwd && c.prev && c.prev->total_next == 0 &&
        c.prev->inflight_records == 0) {
      phase = kBwd;
      backward_from = c.iter;
      // one partition: the deepest label is the last superstep that found
      // anything (superstep t labels t+1; superstep c.iter-1 found nothing)
      max_level = c.P->n == 1 ? (uint32_t)c.iter - 1 : (uint32_t)c.prev->max_u(0);
      std::fill(bucketed.begin(), bucketed.end(), 0);
    }
    if (first && phase == kBwd && c.iter - backward_from >= max_level) phase = kDone;
    uint32_t nh = (uint32_t)w.hosted_host.size();
    if (phase == kFwd) {
      if (c.fused && c.P->n == 1 && kBcDenseDiv &&
          (uint64_t)c.in_count * kBcDenseDiv >= w.nv) {
        BcDev f = dev(c);
        f.red = 1;
        c.pipeline(f, w.nv);
        MGB_LAUNCH(dense_list_kernel<LabelIs>, grid_for((w.nv + 3) / 4, 256, num_sms() * 8),
                   256, 0, w.stream, LabelIs{w.su32[0].ptr, (uint32_t)c.iter + 1}, w.nv,
                   w.output.ptr, &c.ctr()->out_cnt);
      } else {
        c.pipeline(dev(c), w.nv);
      }
      if (nh && c.P->n > 1)  // the global max hosted label; n = 1 derives it
        MGB_LAUNCH(max_hosted_label_kernel, grid_for(nh, 256, num_sms() * 4), 256, 0, w.stream,
                   w.su32[0].ptr, w.hosted.ptr, nh, c.ctr());
      c.report.u[1] = kFwd;
      c.report.u[0] = 0;  // filled from the device counter
      return;
    }
    if (phase == kBwd && (uint64_t)kBcClasses * (max_level + 1) <= kBcBuckets) {
      const uint32_t level = max_level - (uint32_t)(c.iter - backward_from);
      const uint32_t nb = kBcClasses * (max_level + 1);
      c.ensure_output(nh);
      std::vector<uint32_t>& bucket_start = bucket_starts[w.p];
      if (!bucketed[w.p]) {  // once per run: counting sort of the hosted vertices by level
        bucketed[w.p] = 1;
        if (w.aux[0].n < nh + 1ull) w.aux[0].alloc(nh + 1ull);
        if (w.aux[1].n < (uint64_t)nb * kBcBucketCtas) w.aux[1].alloc((uint64_t)nb * kBcBucketCtas);
        if (w.aux[2].n < nb + 1ull) w.aux[2].alloc(nb + 1ull);
        MGB_LAUNCH(bc_bucket_count_kernel, kBcBucketCtas, 256, 0, w.stream, w.hosted.ptr, nh,
                   w.su32[0].ptr, w.off.ptr, max_level, nb, w.aux[1].ptr);
        MGB_LAUNCH(bc_bucket_scan_kernel, 1, 1024, 0, w.stream, w.aux[1].ptr, nb, kBcBucketCtas,
                   w.aux[2].ptr);
        MGB_LAUNCH(bc_bucket_scatter_kernel, kBcBucketCtas, 256, 0, w.stream, w.hosted.ptr, nh,
                   w.su32[0].ptr, w.off.ptr, max_level, nb, w.aux[1].ptr, w.aux[0].ptr);
        bucket_start.assign(nb + 1, 0);
        MGB_CUDA(cudaMemcpyAsync(bucket_start.data(), w.aux[2].ptr, 4ull * (nb + 1),
                                 cudaMemcpyDeviceToHost, w.stream));
        MGB_CUDA(cudaStreamSynchronize(w.stream));
      }
      const uint32_t* list = w.aux[0].ptr;
      const uint32_t K = kBcClasses;
      const uint32_t s0 = bucket_start[K * level], s1 = bucket_start[K * level + 1],
                     s2 = bucket_start[K * level + 2], s3 = bucket_start[K * level + 3];
      const bool deepest = level == max_level;
      const uint32_t c0 = deepest ? 0 : bucket_start[K * (level + 1)];
      const uint32_t c1 = deepest ? 0 : bucket_start[K * (level + 2)];
      const uint32_t work = (s3 - s0) > (c1 - c0) ? (s3 - s0) : (c1 - c0);
      MGB_LAUNCH(bc_level_prep_kernel, grid_for(work, 256, num_sms() * 8), 256, 0, w.stream, list,
                 s0, s3, c0, c1, deepest ? 1 : 0, w.sf64[0].ptr, w.sf64[1].ptr, w.sf64[3].ptr,
                 w.output.ptr, c.ctr());
      if (!deepest) {  // the deepest level only broadcasts
        if (s1 > s0)
          MGB_LAUNCH(bc_backward_thread_kernel, grid_for(s1 - s0, 256, num_sms() * 8), 256, 0,
                     w.stream, w.graph(), list + s0, nullptr, s1 - s0, w.sf64[0].ptr,
                     w.sf64[1].ptr, w.sf64[2].ptr, w.sf64[3].ptr, source, c.ctr());
        if (s2 > s1)
          MGB_LAUNCH(bc_backward_warp_kernel, grid_for((uint64_t)(s2 - s1) * 32, 256, num_sms() * 8),
                     256, 0, w.stream, w.graph(), list + s1, nullptr, s2 - s1, w.sf64[0].ptr,
                     w.sf64[1].ptr, w.sf64[2].ptr, w.sf64[3].ptr, source, c.ctr());
        if (s3 > s2) {  // huge rows: chunks over many CTAs
          const uint32_t nh_ = s3 - s2;
          if (w.aux[3].n < nh_ + 1ull) w.aux[3].alloc(nh_ + 1ull);
          if (w.bc_acc.n < nh_) w.bc_acc.alloc(nh_);
          MGB_LAUNCH(bc_huge_prefix_kernel, 1, 1024, 0, w.stream, list + s2, nh_, w.off.ptr,
                     w.aux[3].ptr, w.bc_acc.ptr);
          MGB_LAUNCH(bc_huge_chunks_kernel, num_sms() * 8, 256, 0, w.stream, w.graph(), list + s2,
                     nh_, w.aux[3].ptr, w.sf64[3].ptr, w.bc_acc.ptr);
          MGB_LAUNCH(bc_huge_finish_kernel, grid_for(nh_, 256, num_sms()), 256, 0, w.stream,
                     w.graph(), list + s2, nh_, w.bc_acc.ptr, w.sf64[0].ptr, w.sf64[1].ptr,
                     w.sf64[2].ptr, source, c.ctr());
        }
      }
      c.report.u[0] = max_level;
      c.report.u[1] = kBwd;
      return;
    }
    if (phase == kBwd) {  // very deep BFS trees: one selection pass per level
      uint32_t level = max_level - (uint32_t)(c.iter - backward_from);
      c.ensure_output(nh);
      if (w.aux[0].n < nh + 1ull) w.aux[0].alloc(nh + 1ull);  // short rows of the level
      if (w.aux[1].n < nh + 1ull) w.aux[1].alloc(nh + 1ull);  // long rows of the level
      if (w.aux[2].n < 2) w.aux[2].alloc(2);
      uint32_t* cnts = w.aux[2].ptr;
      MGB_CUDA(cudaMemsetAsync(cnts, 0, 8, w.stream));
      if (nh) {
        MGB_LAUNCH(bc_level_select_kernel, grid_for(nh, 256, num_sms() * 16), 256, 0, w.stream,
                   w.hosted.ptr, nh, w.su32[0].ptr, w.off.ptr, level, w.output.ptr, c.ctr(),
                   w.aux[0].ptr, cnts, w.aux[1].ptr, cnts + 1, level == max_level ? 1 : 0,
                   w.sf64[0].ptr, w.sf64[1].ptr, w.sf64[3].ptr);
        if (level < max_level) {  // the deepest level only broadcasts
          MGB_LAUNCH(bc_backward_thread_kernel, num_sms() * 8, 256, 0, w.stream, w.graph(),
                     w.aux[0].ptr, cnts, 0u, w.sf64[0].ptr, w.sf64[1].ptr, w.sf64[2].ptr,
                     w.sf64[3].ptr, source, c.ctr());
          MGB_LAUNCH(bc_backward_warp_kernel, num_sms() * 8, 256, 0, w.stream, w.graph(),
                     w.aux[1].ptr, cnts + 1, 0u, w.sf64[0].ptr, w.sf64[1].ptr, w.sf64[2].ptr,
                     w.sf64[3].ptr, source, c.ctr());
        }
      }
      c.report.u[0] = max_level;
      c.report.u[1] = kBwd;
      return;
    }
    c.report.u[0] = max_level;
    c.report.u[1] = kDone;
  }
  int comm_selector(Ctx&, int) {
    return phase == kFwd ? MG_COMM_SELECTIVE : MG_COMM_BROADCAST;
  }
  bool stop_condition(const GlobalView& v) {  // primitives.cpp:632-635
    return v.all_u_equal(1, kDone) && v.total_next == 0 && v.inflight_records == 0;
  }
};

// ===========================================================================
// PageRank (primitives.cpp:697-827)

struct PrDev {
  double* accum;
  const uint32_t* border_dst;
  __device__ bool visit(uint32_t, uint32_t, uint32_t) const { return false; }
  __device__ bool keep(uint32_t) const { return true; }
  __device__ bool prefilter(uint32_t) const { return true; }
  __device__ bool combine(uint32_t v, const uint32_t*, const double* vv, uint32_t) const {
    atomicAdd(&accum[v], vv[0]);
    return false;  // ranks are combined, never enqueued
  }
  __device__ void gather(uint32_t v, uint32_t*, double* vv) const {
    vv[0] = accum[v];
    accum[v] = 0.0;  // partial shipped
  }
  __device__ bool send_filter(uint32_t, uint32_t) const { return true; }
  // the output is the static border list: entry i's destination-local ID
  __device__ uint32_t peer_id(uint32_t, uint32_t, uint32_t i) const { return border_dst[i]; }
};

// --- pull-form accumulation ------------------------------------------------
// accum[v] = sum over hosted in-neighbours u of rank[u]/deg(u) is the same sum
// the reference's push loop forms (primitives.cpp:766-776), gathered per
// destination in a fixed order instead of scattered with f64 atomics.  The
// transpose of the worker's sub-graph is built once per plan.

__global__ void transpose_keys_kernel(GraphView g, const uint32_t* __restrict__ hosted,
                                      uint32_t nh, unsigned long long* keys) {
  const uint32_t warps = gridDim.x * blockDim.x / 32;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / 32; i < nh; i += warps) {
    uint32_t u = hosted[i];
    for (uint32_t e = g.off[u] + lane_id(); e < g.off[u + 1]; e += 32)
      keys[e] = ((unsigned long long)g.col[e] << 32) | u;
  }
}

__global__ void transpose_csr_kernel(const unsigned long long* __restrict__ keys, uint64_t ne,
                                     uint32_t nv, uint32_t* toff, uint32_t* tcol) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ne; i += stride)
    tcol[i] = (uint32_t)keys[i];
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= nv; v += stride) {
    unsigned long long target = v << 32;
    uint64_t lo = 0, hi = ne;
    while (lo < hi) {
      uint64_t m = (lo + hi) >> 1;
      if (keys[m] < target) lo = m + 1;
      else hi = m;
    }
    toff[v] = (uint32_t)lo;
  }
}

constexpr uint32_t kPullLong = 64;  // rows at least this long get a warp

__global__ void select_long_rows_kernel(const uint32_t* __restrict__ toff, uint32_t nv,
                                        uint32_t* out, uint32_t* cnt) {
  for (uint32_t base = blockIdx.x * blockDim.x; base < nv; base += gridDim.x * blockDim.x) {
    uint32_t v = base + threadIdx.x;
    bool lng = v < nv && toff[v + 1] - toff[v] >= kPullLong;
    uint32_t s = warp_append(cnt, lng);
    if (lng) out[s] = v;
  }
}

// contrib[u] = rank[u]/deg(u) for hosted u; dangling mass aside
__global__ void pr_contrib_kernel(GraphView g, const uint32_t* __restrict__ hosted, uint32_t nh,
                                  const double* __restrict__ rank, double* contrib,
                                  Counters* ctr) {
  double dangling = 0.0;
  unsigned long long scanned = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nh; i += gridDim.x * blockDim.x) {
    uint32_t u = hosted[i];
    uint32_t d = g.off[u + 1] - g.off[u];
    if (d == 0) {
      dangling += rank[u];
      contrib[u] = 0.0;
    } else {
      contrib[u] = rank[u] / (double)d;
      scanned += d;
    }
  }
  for (int o = 16; o > 0; o >>= 1) dangling += __shfl_xor_sync(0xffffffffu, dangling, o);
  warp_add_u64(&ctr->edges, scanned);
  if (lane_id() == 0 && dangling != 0.0) atomicAdd(&ctr->f[0], dangling);
}

// rows shorter than kPullLong: one thread per row, four gathers in flight.
// In the locality order neighbouring threads own neighbouring rows whose
// in-neighbours overlap, so the contribution gathers mostly hit L1/L2.
__global__ void __launch_bounds__(256)
    pr_pull_kernel(const uint32_t* __restrict__ toff, const uint32_t* __restrict__ tcol,
                   uint32_t nv, const double* __restrict__ contrib, double* accum) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    const uint32_t b = __ldg(&toff[v]), e = __ldg(&toff[v + 1]);
    if (e - b >= kPullLong) continue;  // warp kernel
    double s0 = 0.0, s1 = 0.0;
    uint32_t k = b;
    for (; k + 3 < e; k += 4) {
      const uint32_t u0 = __ldg(&tcol[k]), u1 = __ldg(&tcol[k + 1]);
      const uint32_t u2 = __ldg(&tcol[k + 2]), u3 = __ldg(&tcol[k + 3]);
      const double c0 = __ldg(&contrib[u0]), c1 = __ldg(&contrib[u1]);
      const double c2 = __ldg(&contrib[u2]), c3 = __ldg(&contrib[u3]);
      s0 += c0;
      s1 += c1;
      s0 += c2;
      s1 += c3;
    }
    for (; k < e; ++k) s0 += __ldg(&contrib[__ldg(&tcol[k])]);
    accum[v] = s0 + s1;
  }
}

__global__ void __launch_bounds__(256)
    pr_pull_warp_kernel(const uint32_t* __restrict__ toff, const uint32_t* __restrict__ tcol,
                        const uint32_t* __restrict__ rows, uint32_t nrows,
                        const double* __restrict__ contrib, double* accum) {
  const uint32_t warps = gridDim.x * blockDim.x / 32;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / 32; i < nrows; i += warps) {
    uint32_t v = rows[i];
    double s = 0.0;
    for (uint32_t k = toff[v] + lane_id(); k < toff[v + 1]; k += 32)
      s += __ldg(&contrib[__ldg(&tcol[k])]);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane_id() == 0) accum[v] = s;
  }
}

// --- locality-ordered single-partition form --------------------------------
// With one partition every vertex is hosted, so the rank / accumulator /
// contribution arrays can live in a vertex order chosen for locality (the
// FIFO-BFS order of bfs_locality_order): the pull's gathers then fall inside
// a narrow band of the contribution array instead of all of it.  The
// transpose, the out-degrees and the rank arrays are kept in that order; the
// ranks are mapped back to vertex IDs when the run ends.

__global__ void transpose_keys_perm_kernel(GraphView g, const uint32_t* __restrict__ perm,
                                           unsigned long long* keys, uint32_t* pdeg) {
  const uint32_t warps = gridDim.x * blockDim.x / 32;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) / 32; u < g.nv; u += warps) {
    const uint32_t pu = perm[u], b = g.off[u], e = g.off[u + 1];
    if (lane_id() == 0) pdeg[pu] = e - b;
    for (uint32_t k = b + lane_id(); k < e; k += 32)
      keys[k] = ((unsigned long long)perm[g.col[k]] << 32) | pu;
  }
}

// pr_update (primitives.cpp:697-711) fused with the next contribution
// rank/deg (primitives.cpp:766-771): one streaming pass in the locality order
__global__ void __launch_bounds__(256)
    pr_update_contrib_kernel(uint32_t nv, const uint32_t* __restrict__ pdeg, double* rank,
                             const double* __restrict__ accum, double* contrib, double base,
                             double damping, double dangling_n, int update, Counters* ctr) {
  double dmax = 0.0, sum = 0.0, dangling = 0.0;
  unsigned long long scanned = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
    double r = rank[i];
    if (update) {
      double nr = base + damping * (accum[i] + dangling_n);
      double rel = fabs(nr - r) / fmax(nr, 1e-300);
      dmax = fmax(dmax, rel);
      rank[i] = nr;
      sum += nr;
      r = nr;
    }
    const uint32_t d = pdeg[i];
    if (d == 0) {
      dangling += r;
      contrib[i] = 0.0;
    } else {
      contrib[i] = r / (double)d;
      scanned += d;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    dangling += __shfl_xor_sync(0xffffffffu, dangling, o);
  }
  warp_add_u64(&ctr->edges, scanned);
  if (lane_id() == 0) {
    if (update) {
      atomic_max_pos_f64(&ctr->f[1], dmax);
      atomicAdd(&ctr->f[2], sum);
    }
    if (dangling != 0.0) atomicAdd(&ctr->f[0], dangling);
  }
}

// Fused superstep (locality-ordered single partition): pull this superstep's
// accumulator from contrib_cur and immediately apply the NEXT pr_update
// (primitives.cpp:697-711) and contribution rank/deg — the update of
// superstep t+1 needs only accum_t and dangling_t, both final here — so one
// pass per superstep replaces pull + update/contrib.  Next-superstep scalars
// go to u[1] (max relative delta, ordered bits), u[2] (rank sum), u[3]
// (dangling mass) as doubles; contributions are double-buffered.
struct PrFuse {
  const uint32_t* __restrict__ pdeg;
  double* rank;
  double* contrib_next;
  double base, damping, dangling_n;
  const double* dangling_ptr;  // superstep 0: dangling_0 on the device
  double nv;
  int count_edges;             // superstep 0's arcs were counted by its contribution pass
};

__device__ __forceinline__ void pr_fuse_finish(const PrFuse& f, uint32_t v, double s, double dn,
                                               double& dmax, double& sum, double& dangl,
                                               uint32_t& scanned) {
  const double nr = f.base + f.damping * (s + dn);
  const double rel = fabs(nr - f.rank[v]) / fmax(nr, 1e-300);
  dmax = fmax(dmax, rel);
  f.rank[v] = nr;
  sum += nr;
  const uint32_t d = f.pdeg[v];
  if (d == 0) {
    dangl += nr;
    f.contrib_next[v] = 0.0;
  } else {
    f.contrib_next[v] = nr / (double)d;
    scanned += d;
  }
}

__device__ __forceinline__ void pr_fuse_reduce(Counters* ctr, double dmax, double sum,
                                               double dangl, uint32_t scanned) {
  for (int o = 16; o > 0; o >>= 1) {
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    dangl += __shfl_xor_sync(0xffffffffu, dangl, o);
  }
  if (scanned) warp_add_u64(&ctr->edges, scanned);
  if (lane_id() == 0) {
    atomicMax(&ctr->u[1], (unsigned long long)__double_as_longlong(dmax));
    atomicAdd(reinterpret_cast<double*>(&ctr->u[2]), sum);
    if (dangl != 0.0) atomicAdd(reinterpret_cast<double*>(&ctr->u[3]), dangl);
  }
}

__global__ void __launch_bounds__(256)
    pr_pull_update_kernel(const uint32_t* __restrict__ toff, const uint32_t* __restrict__ tcol,
                          uint32_t nv, const double* __restrict__ contrib, PrFuse f,
                          Counters* ctr) {
  const double dn = f.dangling_ptr ? *f.dangling_ptr / f.nv : f.dangling_n;
  double dmax = 0.0, sum = 0.0, dangl = 0.0;
  uint32_t scanned = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    const uint32_t b = __ldg(&toff[v]), e = __ldg(&toff[v + 1]);
    if (e - b >= kPullLong) continue;  // warp kernel
    double s0 = 0.0, s1 = 0.0;
    uint32_t k = b;
    for (; k + 3 < e; k += 4) {
      const uint32_t u0 = __ldg(&tcol[k]), u1 = __ldg(&tcol[k + 1]);
      const uint32_t u2 = __ldg(&tcol[k + 2]), u3 = __ldg(&tcol[k + 3]);
      const double c0 = __ldg(&contrib[u0]), c1 = __ldg(&contrib[u1]);
      const double c2 = __ldg(&contrib[u2]), c3 = __ldg(&contrib[u3]);
      s0 += c0;
      s1 += c1;
      s0 += c2;
      s1 += c3;
    }
    for (; k < e; ++k) s0 += __ldg(&contrib[__ldg(&tcol[k])]);
    pr_fuse_finish(f, v, s0 + s1, dn, dmax, sum, dangl, scanned);
  }
  pr_fuse_reduce(ctr, dmax, sum, dangl, f.count_edges ? scanned : 0u);
}

__global__ void __launch_bounds__(256)
    pr_pull_update_warp_kernel(const uint32_t* __restrict__ toff,
                               const uint32_t* __restrict__ tcol,
                               const uint32_t* __restrict__ rows, uint32_t nrows,
                               const double* __restrict__ contrib, PrFuse f, Counters* ctr) {
  const double dn = f.dangling_ptr ? *f.dangling_ptr / f.nv : f.dangling_n;
  double dmax = 0.0, sum = 0.0, dangl = 0.0;
  uint32_t scanned = 0;
  const uint32_t warps = gridDim.x * blockDim.x / 32;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / 32; i < nrows; i += warps) {
    const uint32_t v = rows[i];
    double s = 0.0;
    for (uint32_t k = toff[v] + lane_id(); k < toff[v + 1]; k += 32)
      s += __ldg(&contrib[__ldg(&tcol[k])]);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane_id() == 0) pr_fuse_finish(f, v, s, dn, dmax, sum, dangl, scanned);
  }
  pr_fuse_reduce(ctr, dmax, sum, dangl, f.count_edges ? scanned : 0u);
}

__global__ void unpermute_f64_kernel(const double* __restrict__ src, const uint32_t* __restrict__ perm,
                                     uint32_t n, double* dst) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    dst[v] = src[perm[v]];
}

// pr_update (primitives.cpp:697-711) fused with zeroing the hosted accumulators
__global__ void pr_update_kernel(const uint32_t* __restrict__ hosted, uint32_t nh, double* rank,
                                 double* accum, double base, double damping, double dangling_n,
                                 int update, Counters* ctr) {
  double dmax = 0.0, sum = 0.0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nh; i += gridDim.x * blockDim.x) {
    uint32_t v = hosted[i];
    if (update) {
      double nr = base + damping * (accum[v] + dangling_n);
      double rel = fabs(nr - rank[v]) / fmax(nr, 1e-300);
      dmax = fmax(dmax, rel);
      rank[v] = nr;
      sum += nr;
    }
    accum[v] = 0.0;
  }
  if (!update) return;
  for (int o = 16; o > 0; o >>= 1) {
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
  }
  if (lane_id() == 0) {
    atomic_max_pos_f64(&ctr->f[1], dmax);
    atomicAdd(&ctr->f[2], sum);
  }
}

// push rank/outdegree into every out-neighbour; dangling mass aside
// (primitives.cpp:762-778).  One warp per hosted vertex, lanes over its arcs.
__global__ void __launch_bounds__(256)
    pr_push_kernel(GraphView g, const uint32_t* __restrict__ hosted, uint32_t nh,
                   const double* rank, double* accum, Counters* ctr) {
  const uint32_t warps = gridDim.x * blockDim.x / 32;
  uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  double dangling = 0.0;
  unsigned long long scanned = 0;
  for (uint32_t i = wid; i < nh; i += warps) {
    uint32_t v = hosted[i];
    uint32_t b = g.off[v], e = g.off[v + 1];
    if (e == b) {
      if (lane_id() == 0) dangling += rank[v];
      continue;
    }
    double contrib = rank[v] / (double)(e - b);
    for (uint32_t k = b + lane_id(); k < e; k += 32) atomicAdd(&accum[g.col[k]], contrib);
    if (lane_id() == 0) scanned += e - b;
  }
  for (int o = 16; o > 0; o >>= 1) dangling += __shfl_xor_sync(0xffffffffu, dangling, o);
  if (lane_id() == 0) {
    if (dangling != 0.0) atomicAdd(&ctr->f[0], dangling);
    if (scanned) atomicAdd(&ctr->edges, scanned);
  }
}

__global__ void copy_border_kernel(const uint32_t* border, uint32_t n, uint32_t* out,
                                   Counters* ctr) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = border[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->out_cnt = n;
}

// plan-lifetime transpose of the worker's sub-graph (rows sorted by source);
// for a single Duplicate-All partition it is built in the locality order
void ensure_transpose(Plan& P, Worker& w) {
  if (w.transpose_ready) return;
  const uint64_t ne = w.ne;
  const uint32_t nh = (uint32_t)w.hosted_host.size();
  w.toff.alloc(w.nv + 1ull);
  w.tcol.alloc(ne ? ne : 1);
  DevArray<unsigned long long> k0, k1;
  k0.alloc(ne ? ne : 1);
  k1.alloc(ne ? ne : 1);
  w.pr_reordered = ordered_layout(P) && w.nv > 0;
  if (w.pr_reordered) {
    std::vector<uint32_t> off(w.nv + 1ull), col(ne);
    MGB_CUDA(cudaMemcpy(off.data(), w.off.ptr, 4ull * (w.nv + 1ull), cudaMemcpyDeviceToHost));
    if (ne) MGB_CUDA(cudaMemcpy(col.data(), w.col.ptr, 4ull * ne, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> perm = bfs_locality_order(off.data(), col.data(), w.nv);
    w.pr_perm.upload(perm.data(), w.nv, w.stream);
    w.pr_pdeg.alloc(w.nv);
  w.pr_iperm.alloc(w.nv);
  MGB_LAUNCH(iperm_kernel, grid_for(w.nv, 256, num_sms() * 8), 256, 0, w.stream, w.pr_perm.ptr,
             w.nv, w.pr_iperm.ptr);
    MGB_LAUNCH(transpose_keys_perm_kernel, grid_for((uint64_t)w.nv * 32, 256, num_sms() * 16),
               256, 0, w.stream, w.graph(), w.pr_perm.ptr, k0.ptr, w.pr_pdeg.ptr);
    MGB_CUDA(cudaStreamSynchronize(w.stream));
  } else if (nh && ne) {
    MGB_LAUNCH(transpose_keys_kernel, grid_for((uint64_t)nh * 32, 256, num_sms() * 16), 256, 0,
               w.stream, w.graph(), w.hosted.ptr, nh, k0.ptr);
  }
  cub::DoubleBuffer<unsigned long long> db(k0.ptr, k1.ptr);
  size_t tb = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int64_t)ne, 0, 64, w.stream);
  void* tmp = nullptr;
  MGB_CUDA(cudaMalloc(&tmp, tb + 16));
  cub::DeviceRadixSort::SortKeys(tmp, tb, db, (int64_t)ne, 0, 64, w.stream);
  MGB_LAUNCH(transpose_csr_kernel, num_sms() * 16, 256, 0, w.stream, db.Current(), ne, w.nv,
             w.toff.ptr, w.tcol.ptr);
  DevArray<uint32_t> cnt;
  cnt.alloc(1);
  MGB_CUDA(cudaMemsetAsync(cnt.ptr, 0, 4, w.stream));
  w.tlong.alloc(w.nv ? w.nv : 1);
  if (w.nv)
    MGB_LAUNCH(select_long_rows_kernel, grid_for(w.nv, 256, num_sms() * 8), 256, 0, w.stream,
               w.toff.ptr, w.nv, w.tlong.ptr, cnt.ptr);
  MGB_CUDA(cudaMemcpyAsync(&w.n_tlong, cnt.ptr, 4, cudaMemcpyDeviceToHost, w.stream));
  MGB_CUDA(cudaStreamSynchronize(w.stream));
  cudaFree(tmp);
  k0.free_();
  k1.free_();
  cnt.free_();
  w.transpose_ready = true;
}

struct PrPrim : PrimBase {
  double damping, epsilon;
  uint64_t max_iter;
  uint64_t updates = 0;
  std::vector<double> rank_sums;
  PrPrim(double d, double e, uint64_t m) : damping(d), epsilon(e), max_iter(m) {
    name = "pr";
    nvv = 1;
    dup_required = -1;  // duplicate-all or duplicate-1-hop
    has_stop_condition = true;
  }
  uint64_t inbox_bound(Plan& P, uint32_t src, uint32_t dst, int) const {
    return P.pair_border[src][dst];
  }
  void init(Ctx& c) {  // primitives.cpp:728-745
    Worker& w = *c.w;
    ensure_transpose(*c.P, w);  // plan lifetime
    if (w.pr_reordered) {
      for (int k : {0, 1, 2, 3})
        if (w.sf64[k].n < w.nv || !w.sf64[k].ptr) w.sf64[k].alloc(w.nv);
      MGB_LAUNCH(fill_f64_kernel, grid_for(w.nv, 256, num_sms() * 8), 256, 0, w.stream,
                 w.sf64[3].ptr, w.nv, 1.0 / (double)c.P->nv);
      return;
    }
    fill(w.sf64[0], w.nv, 0, w.stream);  // rank
    fill(w.sf64[1], w.nv, 0, w.stream);  // accum
    uint32_t nh = (uint32_t)w.hosted_host.size();
    if (nh)
      MGB_LAUNCH(fill_hosted_f64_kernel, grid_for(nh, 256), 256, 0, w.stream, w.sf64[0].ptr,
                 w.hosted.ptr, nh, 1.0 / (double)c.P->nv);
  }
  PrDev dev(Ctx& c) { return {c.w->sf64[1].ptr, c.w->border_dst.ptr}; }
  void update(Ctx& c, double dangling_prev, bool do_update) {
    Worker& w = *c.w;
    const double n = (double)c.P->nv;
    uint32_t nh = (uint32_t)w.hosted_host.size();
    if (nh)
      MGB_LAUNCH(pr_update_kernel, grid_for(nh, 256, num_sms() * 8), 256, 0, w.stream, w.hosted.ptr,
                 nh, w.sf64[0].ptr, w.sf64[1].ptr, (1.0 - damping) / n, damping,
                 dangling_prev / n, do_update ? 1 : 0, c.ctr());
  }
  static void ensure_transpose(Plan& P, Worker& w) { mgb::ensure_transpose(P, w); }
  // locality-ordered single partition: rank in sf64[3] (ordered), accum
  // sf64[1], contributions sf64[2]; ranks mapped back into sf64[0] at the end
  void update_contrib(Ctx& c, double dangling_prev, bool do_update) {
    Worker& w = *c.w;
    const double n = (double)c.P->nv;
    MGB_LAUNCH(pr_update_contrib_kernel, grid_for(w.nv, 256, num_sms() * 8), 256, 0, w.stream,
               w.nv, w.pr_pdeg.ptr, w.sf64[3].ptr, w.sf64[1].ptr, w.sf64[2].ptr,
               (1.0 - damping) / n, damping, dangling_prev / n, do_update ? 1 : 0, c.ctr());
  }
  void pull(Worker& w) {
    if (w.nv)
      MGB_LAUNCH(pr_pull_kernel, grid_for(w.nv, 256, num_sms() * 16), 256, 0, w.stream,
                 w.toff.ptr, w.tcol.ptr, w.nv, w.sf64[2].ptr, w.sf64[1].ptr);
    if (w.n_tlong)
      MGB_LAUNCH(pr_pull_warp_kernel, grid_for((uint64_t)w.n_tlong * 32, 256, num_sms() * 8), 256,
                 0, w.stream, w.toff.ptr, w.tcol.ptr, w.tlong.ptr, w.n_tlong, w.sf64[2].ptr,
                 w.sf64[1].ptr);
  }
  // Fused ordered form.  Superstep t reports the reference's values of its own
  // update (delta_t, sum_t, dangling_t), which the fused pass of superstep t-1
  // already produced, and runs the fused pass for t+1 unless delta_t < eps
  // stops the run here (then rank already holds rank_t, the reference's
  // result).  On a max-iteration stop the pass of the last superstep is the
  // reference's finalize update (primitives.cpp:801-810).
  double next_delta = 0, next_sum = 0, next_dangling = 0;
  uint64_t edges_per_step = 0;
  void body_ordered(Ctx& c) {
    Worker& w = *c.w;
    const bool first = c.worker() == c.P->local_workers.front();
    const double n = (double)c.P->nv;
    bool run_pass = true;
    if (c.iter >= 1) {
      const WorkerReport& pr = c.prev->reports[w.p];
      if (c.iter == 1) edges_per_step = pr.edges_delta;
      std::memcpy(&next_delta, &pr.u[1], 8);
      std::memcpy(&next_sum, &pr.u[2], 8);
      std::memcpy(&next_dangling, &pr.u[3], 8);
      c.report.f[0] = next_dangling;  // pushed mass of rank_t
      c.report.f[1] = next_delta;     // pr_update of superstep t
      c.report.f[2] = next_sum;
      if (first) ++updates;
      run_pass = !(next_delta < epsilon);
      if (!run_pass && edges_per_step)  // the push of rank_t still counts (E:66)
        MGB_LAUNCH(add_u64_kernel, 1, 1, 0, w.stream, &c.ctr()->edges,
                   (unsigned long long)edges_per_step);
    } else {
      update_contrib(c, 0.0, false);  // contrib_0, dangling_0 -> f[0], W
      c.report.f[1] = INFINITY;
    }
    if (first && c.prev && c.iter >= 2) rank_sums.push_back(c.prev->sum_f(2));
    if (!run_pass) return;
    double* cur = (c.iter & 1) ? w.sf64[0].ptr : w.sf64[2].ptr;
    double* nxt = (c.iter & 1) ? w.sf64[2].ptr : w.sf64[0].ptr;
    PrFuse f{w.pr_pdeg.ptr, w.sf64[3].ptr, nxt, (1.0 - damping) / n, damping,
             next_dangling / n, c.iter == 0 ? &c.ctr()->f[0] : nullptr, n, c.iter == 0 ? 0 : 1};
    if (w.nv)
      MGB_LAUNCH(pr_pull_update_kernel, grid_for(w.nv, 256, num_sms() * 16), 256, 0, w.stream,
                 w.toff.ptr, w.tcol.ptr, w.nv, cur, f, c.ctr());
    if (w.n_tlong)
      MGB_LAUNCH(pr_pull_update_warp_kernel, grid_for((uint64_t)w.n_tlong * 32, 256, num_sms() * 8),
                 256, 0, w.stream, w.toff.ptr, w.tcol.ptr, w.tlong.ptr, w.n_tlong, cur, f, c.ctr());
  }
  void body(Ctx& c) {  // primitives.cpp:747-782
    Worker& w = *c.w;
    ensure_transpose(*c.P, w);
    if (w.pr_reordered) return body_ordered(c);
    const bool first = c.worker() == c.P->local_workers.front();
    if (c.iter >= 1) {
      update(c, c.prev->sum_f(0), true);
      if (first) ++updates;
    } else {
      update(c, 0.0, false);  // zero hosted accum only
      c.report.f[1] = INFINITY;
    }
    if (first && c.worker() == 0 && c.prev && c.iter >= 2) rank_sums.push_back(c.prev->sum_f(2));
    uint32_t nh = (uint32_t)w.hosted_host.size();
    // accum[v] = sum of rank[u]/deg(u) over hosted in-neighbours u,
    // gathered per destination (pull) in a fixed order
    if (w.sf64[2].n < w.nv || !w.sf64[2].ptr) w.sf64[2].alloc(w.nv ? w.nv : 1);
    if (nh)
      MGB_LAUNCH(pr_contrib_kernel, grid_for(nh, 256, num_sms() * 8), 256, 0, w.stream, w.graph(),
                 w.hosted.ptr, nh, w.sf64[0].ptr, w.sf64[2].ptr, c.ctr());
    if (w.nv)
      MGB_LAUNCH(pr_pull_kernel, grid_for(w.nv, 256, num_sms() * 16), 256, 0, w.stream,
                 w.toff.ptr, w.tcol.ptr, w.nv, w.sf64[2].ptr, w.sf64[1].ptr);
    if (w.n_tlong)
      MGB_LAUNCH(pr_pull_warp_kernel, grid_for((uint64_t)w.n_tlong * 32, 256, num_sms() * 8), 256,
                 0, w.stream, w.toff.ptr, w.tcol.ptr, w.tlong.ptr, w.n_tlong, w.sf64[2].ptr,
                 w.sf64[1].ptr);
    uint32_t nb = (uint32_t)w.border.n;
    c.ensure_output(nb);
    if (nb)
      MGB_LAUNCH(copy_border_kernel, grid_for(nb, 256), 256, 0, w.stream, w.border.ptr, nb,
                 w.output.ptr, c.ctr());
  }
  bool stop_condition(const GlobalView& v) {  // primitives.cpp:796-799
    if (v.iteration + 1 >= max_iter) return true;
    return v.iteration >= 1 && v.max_f(1) < epsilon;
  }
  void finalize(Ctx& c, const GlobalView& last) {  // primitives.cpp:801-810
    bool delta_stopped = last.iteration >= 1 && last.max_f(1) < epsilon;
    const bool first = c.worker() == c.P->local_workers.front();
    if (first && c.worker() == 0 && last.iteration >= 1) rank_sums.push_back(last.sum_f(2));
    Worker& w = *c.w;
    if (!delta_stopped) {
      // ordered form: the last superstep's fused pass already applied it
      if (!w.pr_reordered) {
        MGB_CUDA(cudaMemsetAsync(c.ctr(), 0, sizeof(Counters), w.stream));
        update(c, last.sum_f(0), true);
      }
      if (first) ++updates;
    }
    if (w.pr_reordered && w.nv)  // ranks back to vertex IDs
      MGB_LAUNCH(unpermute_f64_kernel, grid_for(w.nv, 256, num_sms() * 8), 256, 0, w.stream,
                 w.sf64[3].ptr, w.pr_perm.ptr, w.nv, w.sf64[0].ptr);
  }
};

// ---------------------------------------------------------------------------
// C-ABI plumbing

thread_local std::string t_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return MG_OK;
  } catch (const Error& e) {
    t_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    t_err = "host allocation failed";
    return MG_ECAPACITY;
  } catch (const std::exception& e) {
    t_err = e.what();
    return MG_EWORKER;
  }
}

void check_source(Plan& P, uint32_t s, const char* prim) {  // primitives.cpp:27-30
  if (s >= P.nv) throw Error(MG_EINVAL, std::string(prim) + ": source out of range");
}

mg_config cfg_or_default(const mg_config* c) {
  mg_config d;
  mg_config_default(&d);
  return c ? *c : d;
}

void finish_stats(Plan& P, mg_stats* st) {
  if (st) *st = P.last;
}

template <class T, size_t N>
std::vector<const T*> pw(Plan& P, DevArray<T> (Worker::*arr)[N], int idx) {
  std::vector<const T*> v(P.n, nullptr);
  for (uint32_t p : P.local_workers) v[p] = (P.workers[p].get()->*arr)[idx].ptr;
  return v;
}

}  // namespace

void set_error(const std::string& msg) { t_err = msg; }
const char* last_error() { return t_err.c_str(); }
int run_guarded(const std::function<void()>& f) { return guarded(f); }

}  // namespace mgb

using namespace mgb;

extern "C" {

void mg_config_default(mg_config* cfg) {
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->policy = MG_POLICY_JUST;
  cfg->fused = MG_FUSED_AUTO;
  cfg->comm_override = MG_COMM_DEFAULT;
  cfg->h_inflation = 1;
  cfg->max_supersteps = 1000000;
}

int mg_bfs(mg_plan* plan, uint32_t source, int mark_preds, const mg_config* cfg, uint32_t* labels,
           uint32_t* preds, mg_stats* stats) {
  return guarded([&] {
    Plan& P = *reinterpret_cast<Plan*>(plan);
    P.last_d2h_bytes = 0;
    check_source(P, source, "bfs");
    mg_config c = cfg_or_default(cfg);
    P.last = mg_stats{};
    bool done = false;
    if (c.dobfs_exact_cost && DobfsGraphRunner::eligible(P, c))
      done = DobfsGraphRunner::run(P, source, INFINITY, 0.1, mark_preds != 0, c, "bfs",
                                   MG_COMM_SELECTIVE)
                 .complete;
    if (done) {
    } else if (c.dobfs_exact_cost && P.n == 1) {
      // extension: the BFS schedule (every superstep logically forward: a
      // direction rule that never switches) on the DOBFS machinery, heavy
      // supersteps run physically as pulls; labels, S and W are BFS's
      DobfsPrim prim(source, INFINITY, 0.1, mark_preds != 0, true, 1);
      prim.name = "bfs";
      prim.communication = MG_COMM_SELECTIVE;
      run_primitive(P, prim, c);
      for (uint32_t p : P.local_workers) P.workers[p]->dobfs_labels_ok = true;
    } else {
      BfsPrim prim(source, mark_preds != 0);
      run_primitive(P, prim, c);
    }
    P.last_result_kind = 0;
    // BFS levels: the largest label is S - 1 (CLI:339-346)
    gather_labels_u32(P, pw(P, &Worker::su32, 0), labels, P.last.supersteps);
    if (mark_preds) gather_u32(P, pw(P, &Worker::su32, 1), preds);
    finish_stats(P, stats);
  });
}

void mg_make_direction_state(int current, uint64_t q, uint64_t u, uint64_t p, uint64_t edges,
                             uint64_t vertices, double do_a, double do_b, int switched_once,
                             mg_direction_state* s) {
  std::memset(s, 0, sizeof(*s));
  s->current = current;
  s->q_size = q;
  s->u_size = u;
  s->p_size = p;
  s->do_a = do_a;
  s->do_b = do_b;
  s->switched_to_backward_once = switched_once;
  if (vertices > 0) s->fv = (double)q * (double)edges / (double)vertices;
  if (p > 0) s->bv = (double)u * (double)vertices / (double)p;
}

int mg_direction_decide(const mg_direction_state* s) {
  if (s->current == 0) return (!s->switched_to_backward_once && s->fv > s->bv * s->do_a) ? 1 : 0;
  return s->fv < s->bv * s->do_b ? 0 : 1;
}

int mg_dobfs(mg_plan* plan, uint32_t source, double do_a, double do_b, int mark_preds,
             const mg_config* cfg, uint32_t* labels, uint32_t* preds, int32_t* direction_log,
             uint64_t cap, uint64_t* len, uint64_t* forward_edges, uint64_t* backward_edges,
             mg_stats* stats) {
  return guarded([&] {
    Plan& P = *reinterpret_cast<Plan*>(plan);
    P.last_d2h_bytes = 0;
    check_source(P, source, "dobfs");
    mg_config c = cfg_or_default(cfg);
    std::vector<int> dir_log;
    bool done = false;
    if (DobfsGraphRunner::eligible(P, c)) {  // device-driven supersteps (one graph launch)
      DobfsGraphRun r = DobfsGraphRunner::run(P, source, do_a, do_b, mark_preds != 0, c, "dobfs",
                                              MG_COMM_BROADCAST);
      if (r.complete) {
        dir_log = r.dir_log;
        done = true;
      }
    }
    if (!done) {
      DobfsPrim prim(source, do_a, do_b, mark_preds != 0, c.dobfs_exact_cost != 0, P.n);
      P.last = mg_stats{};
      run_primitive(P, prim, c);
      for (uint32_t p : P.local_workers) P.workers[p]->dobfs_labels_ok = true;
      dir_log = prim.dir_log;
    }
    P.last_result_kind = 0;
    gather_labels_u32(P, pw(P, &Worker::su32, 0), labels, P.last.supersteps);
    if (mark_preds) gather_u32(P, pw(P, &Worker::su32, 1), preds);
    P.last_dir_log = dir_log;  // full log (mg_plan_last_array) when `cap` is short
    if (len) *len = dir_log.size();
    for (uint64_t i = 0; direction_log && i < dir_log.size() && i < cap; ++i)
      direction_log[i] = dir_log[i];
    uint64_t f = 0, b = 0;
    for (size_t i = 0; i < dir_log.size() && i < P.edges_per_iter.size(); ++i)
      (dir_log[i] ? b : f) += P.edges_per_iter[i];
    if (forward_edges) *forward_edges = f;
    if (backward_edges) *backward_edges = b;
    finish_stats(P, stats);
  });
}

int mg_sssp(mg_plan* plan, uint32_t source, int mark_preds, const mg_config* cfg, uint64_t* dists,
            uint32_t* preds, mg_stats* stats) {
  return guarded([&] {
    Plan& P = *reinterpret_cast<Plan*>(plan);
    P.last_d2h_bytes = 0;
    check_source(P, source, "sssp");
    if (!P.weighted && P.ne > 0) throw Error(MG_EINVAL, "sssp: graph has no edge weights");
    mg_config c = cfg_or_default(cfg);
    SsspPrim prim(source, mark_preds != 0);
    P.last = mg_stats{};
    run_primitive(P, prim, c);
    P.last_result_kind = 2;
    gather_u64(P, pw(P, &Worker::su64, 0), dists);
    if (mark_preds) gather_u32(P, pw(P, &Worker::su32, 1), preds);
    finish_stats(P, stats);
  });
}

int mg_cc(mg_plan* plan, const mg_config* cfg, uint32_t* components, mg_stats* stats) {
  return guarded([&] {
    Plan& P = *reinterpret_cast<Plan*>(plan);
    P.last_d2h_bytes = 0;
    mg_config c = cfg_or_default(cfg);
    CcPrim prim;
    P.last = mg_stats{};
    run_primitive(P, prim, c);
    P.last_result_kind = 3;
    gather_u32(P, pw(P, &Worker::su32, 0), components);
    finish_stats(P, stats);
  });
}

int mg_bc(mg_plan* plan, uint32_t source, const mg_config* cfg, double* bc, double* sigma,
          uint32_t* labels, mg_stats* stats) {
  return guarded([&] {
    Plan& P = *reinterpret_cast<Plan*>(plan);
    P.last_d2h_bytes = 0;
    check_source(P, source, "bc");
    mg_config c = cfg_or_default(cfg);
    BcPrim prim(source);
    P.last = mg_stats{};
    run_primitive(P, prim, c);
    P.last_result_kind = 4;
    gather_f64(P, pw(P, &Worker::sf64, 2), bc);
    gather_f64(P, pw(P, &Worker::sf64, 0), sigma);
    gather_u32(P, pw(P, &Worker::su32, 0), labels);
    finish_stats(P, stats);
  });
}

int mg_pagerank(mg_plan* plan, double damping, double epsilon, uint64_t max_iter,
                const mg_config* cfg, double* ranks, uint64_t* iterations, double* rank_sums,
                uint64_t cap, uint64_t* len, mg_stats* stats) {
  return guarded([&] {
    Plan& P = *reinterpret_cast<Plan*>(plan);
    P.last_d2h_bytes = 0;
    if (!(damping > 0.0 && damping < 1.0))
      throw Error(MG_EINVAL, "pagerank: damping must lie in (0,1)");
    if (!(epsilon > 0.0)) throw Error(MG_EINVAL, "pagerank: epsilon must be positive");
    if (max_iter < 1) throw Error(MG_EINVAL, "pagerank: max_iter must be >= 1");
    mg_config c = cfg_or_default(cfg);
    PrPrim prim(damping, epsilon, max_iter);
    P.last = mg_stats{};
    run_primitive(P, prim, c);
    P.last_result_kind = 6;
    std::vector<double> host(ranks ? 0 : P.nv);
    double* out = ranks ? ranks : host.data();
    gather_f64(P, pw(P, &Worker::sf64, 0), out);
    std::vector<double> sums = prim.rank_sums;
    bool finalized = prim.updates > P.last.supersteps - 1;  // primitives.cpp:820-825
    if (finalized) {
      double s = 0.0;
      for (uint32_t v = 0; v < P.nv; ++v) s += out[v];
      sums.push_back(s);
    }
    if (iterations) *iterations = prim.updates;
    if (len) *len = sums.size();
    for (uint64_t i = 0; rank_sums && i < sums.size() && i < cap; ++i) rank_sums[i] = sums[i];
    finish_stats(P, stats);
  });
}

int mg_plan_fetch(mg_plan* plan, int which, void* host_out) {
  return guarded([&] {
    Plan& P = *reinterpret_cast<Plan*>(plan);
    P.last_d2h_bytes = 0;
    switch (which) {
      case MG_RES_LABELS: gather_u32(P, pw(P, &Worker::su32, 0), (uint32_t*)host_out); break;
      case MG_RES_PREDS: gather_u32(P, pw(P, &Worker::su32, 1), (uint32_t*)host_out); break;
      case MG_RES_DISTS: gather_u64(P, pw(P, &Worker::su64, 0), (uint64_t*)host_out); break;
      case MG_RES_COMPONENTS: gather_u32(P, pw(P, &Worker::su32, 0), (uint32_t*)host_out); break;
      case MG_RES_BC: gather_f64(P, pw(P, &Worker::sf64, 2), (double*)host_out); break;
      case MG_RES_SIGMA: gather_f64(P, pw(P, &Worker::sf64, 0), (double*)host_out); break;
      case MG_RES_RANKS: gather_f64(P, pw(P, &Worker::sf64, 0), (double*)host_out); break;
      default: throw Error(MG_EINVAL, "mg_plan_fetch: unknown result kind");
    }
  });
}

}  // extern "C"
