// operators.cuh — the traversal operators as sm_100a kernels, templated on the
// primitive's device functors (the reference's advance/filter/fused operators,
// engine.hpp:54-99, and the functor hooks of PrimitiveSpec, engine.hpp:587-626).
//
// advance = edge-balanced ("merge-path") expansion in three kernels:
//   lb_degree_kernel   one pass over the frontier: row start + out-degree per
//                      vertex, CTA-local exclusive scan of the degrees, CTA sums
//   lb_scan_kernel     one CTA scans the CTA sums (global offsets + total W)
//   lb_expand_kernel   persistent CTAs walk tiles of the concatenated
//                      adjacency (kTile = 8192 arcs, smaller for small advances
//                      so at least kMinTiles = 2 x 148 tiles exist): one binary
//                      search per tile over the global degree prefix, the
//                      tile's vertex range staged in shared memory in chunks of
//                      kStage vertices, then every lane expands kItems
//                      lane-strided arcs (one smem search + a short walk), so a
//                      1e6-arc hub is spread over every SM and consecutive
//                      lanes read consecutive col_indices.
// The edge count W (reference E:66) is the scan total.
// filter = order-free compaction by keep(v) with warp-aggregated appends.
#pragma once

#include <cub/block/block_scan.cuh>

#include "plan.cuh"

namespace mgb {

constexpr int kLbBlock = 256;     // degree pass: one vertex per thread
constexpr int kExpBlock = 256;    // expansion CTA
constexpr int kItems = 8;         // arcs per thread per batch (lane-strided)
constexpr uint32_t kTile = 8192;  // arcs per tile for large advances
#ifndef MG_WARPQ
#define MG_WARPQ 384
#endif
#ifndef MG_EXPAND_MIN_CTAS
#define MG_EXPAND_MIN_CTAS 4
#endif
#ifndef MG_KSTAGE
#define MG_KSTAGE 1536
#endif
constexpr int kWarpQ = MG_WARPQ;   // warp-private output staging entries
constexpr int kStage = MG_KSTAGE;  // max tile vertices staged in shared memory

// lb 1: row starts + CTA-local exclusive prefix of degrees
// (n_in_ptr: the frontier length read on the device — graph-captured
// supersteps; the CTAs then walk the virtual blocks of 256 entries)
static __global__ void __launch_bounds__(kLbBlock)
    lb_degree_kernel(const uint32_t* __restrict__ off, const uint32_t* __restrict__ in,
                     uint32_t n_in, uint32_t* __restrict__ rowstart,
                     unsigned long long* __restrict__ prefix, unsigned long long* block_sum,
                     const uint32_t* n_in_ptr = nullptr) {
  using Scan = cub::BlockScan<unsigned long long, kLbBlock>;
  __shared__ typename Scan::TempStorage tmp;
  if (n_in_ptr) n_in = *n_in_ptr;
  const uint32_t nb = (n_in + kLbBlock - 1) / kLbBlock;
  for (uint32_t vb = blockIdx.x; vb < nb; vb += gridDim.x) {
    uint32_t i = vb * kLbBlock + threadIdx.x;
    unsigned long long d = 0;
    if (i < n_in) {
      uint32_t u = in[i];
      uint32_t rs = off[u];
      d = off[u + 1] - rs;
      rowstart[i] = rs;
    }
    unsigned long long excl, total;
    Scan(tmp).ExclusiveSum(d, excl, total);
    if (i < n_in) prefix[i] = excl;
    if (threadIdx.x == 0) block_sum[vb] = total;
    __syncthreads();
  }
}

// lb 2: scan the CTA sums in one CTA; block_sum becomes exclusive offsets,
// block_sum[nb] the total (= edges examined)
static __global__ void __launch_bounds__(1024)
    lb_scan_kernel(unsigned long long* block_sum, uint32_t nb, unsigned long long* total_out,
                   unsigned long long* edges, const uint32_t* n_in_ptr = nullptr) {
  using Scan = cub::BlockScan<unsigned long long, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long carry;
  if (n_in_ptr) nb = (*n_in_ptr + kLbBlock - 1) / kLbBlock;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < nb; base += 1024) {
    uint32_t i = base + threadIdx.x;
    unsigned long long d = i < nb ? block_sum[i] : 0ull;
    unsigned long long excl, total;
    Scan(tmp).ExclusiveSum(d, excl, total);
    if (i < nb) block_sum[i] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    block_sum[nb] = carry;
    *total_out = carry;
    atomicAdd(edges, carry);
  }
}

// Arcs per expansion tile: kTile for large advances; small advances are cut
// into at least kMinTiles tiles (multiples of 256 arcs) so every SM gets work.
constexpr uint32_t kMinTiles = 2 * kB200SMs;
__host__ __device__ __forceinline__ unsigned long long lb_tile_size(unsigned long long total) {
  if (total >= (unsigned long long)kTile * kMinTiles) return kTile;
  unsigned long long t = (total + kMinTiles - 1) / kMinTiles;
  t = (t + 255) / 256 * 256;
  return t < 256 ? 256 : t;
}

// global prefix of frontier entry i
__device__ __forceinline__ unsigned long long lb_pref(const unsigned long long* prefix,
                                                      const unsigned long long* block_off,
                                                      uint32_t i) {
  return block_off[i / kLbBlock] + prefix[i];
}

// last frontier index j in [0,n) with pref(j) <= k
__device__ __forceinline__ uint32_t lb_search(const unsigned long long* prefix,
                                              const unsigned long long* block_off, uint32_t n,
                                              unsigned long long k) {
  uint32_t lo = 0, hi = n - 1;
  while (lo < hi) {
    uint32_t mid = (lo + hi + 1) >> 1;
    if (lb_pref(prefix, block_off, mid) <= k) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Visit a batch of pre-tested arcs.  The generic form calls visit() per arc; a
// functor may provide an overload (found by argument-dependent lookup) that
// issues its atomics for the whole batch before consuming any result, so a
// thread keeps several atomics in flight.
template <int K, class F>
__device__ __forceinline__ void visit_batch(const F& f, const uint32_t* src, const uint32_t* nb,
                                            const uint32_t* eid, const bool* pass, bool* acc) {
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = pass[k] && f.visit(src[k], nb[k], eid[k]);
}

// lb 3a: first frontier entry of every tile (one binary search per tile, all
// tiles in parallel) so the expansion never waits on a serial search
static __global__ void lb_tiles_kernel(const unsigned long long* __restrict__ prefix,
                                       const unsigned long long* __restrict__ block_off,
                                       uint32_t n_in, const unsigned long long* total_ptr,
                                       uint32_t* tile_lo, uint32_t max_tiles,
                                       const uint32_t* n_in_ptr = nullptr) {
  if (n_in_ptr) n_in = *n_in_ptr;
  const unsigned long long total = *total_ptr;
  const unsigned long long ts = lb_tile_size(total);
  const unsigned long long ntiles = (total + ts - 1) / ts;
  for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       t <= ntiles && t <= max_tiles; t += (unsigned long long)gridDim.x * blockDim.x)
    tile_lo[t] = t == ntiles ? n_in - 1 : lb_search(prefix, block_off, n_in, t * ts);
}

// A functor whose visits never read the arc's source vertex (e.g. a dense
// DOBFS push without predecessors) lets the locate phase skip the staged
// source loads.  Found by argument-dependent lookup, like expand_quiet.
template <class F>
__device__ __forceinline__ bool expand_needs_src(const F&) {
  return true;
}
// Minimum resident CTAs per SM the expansion is compiled for (register cap);
// a primitive may specialise it for its functor.
template <class F>
struct expand_min_ctas {
  static constexpr int value = MG_EXPAND_MIN_CTAS;
};
// Locate a lane's whole batch with one test when it lies inside one row (the
// hub rows of a DOBFS push).  Off by default: the extra code path costs SSSP
// more than it saves (RMAT-24 C3 6.76 -> 7.1 ms with it, same box).
template <class F>
struct expand_long_rows {
  static constexpr bool value = false;
};

// A functor may declare an expansion "quiet" (nothing is ever accepted, e.g.
// a dense DOBFS push that only sets visited bits): the kernel then skips the
// per-batch queue ballots and flushes.  Found by argument-dependent lookup.
template <class F>
__device__ __forceinline__ bool expand_quiet(const F&) {
  return false;
}

// lb 3b: edge-balanced expansion (visit [+ keep when fused]).  Per tile the
// vertex range is staged in shared memory (chunks of kStage vertices); batches
// of 32*kItems arcs go round-robin to the warps, lane l taking arcs l, l+32,
// ... of its batch (coalesced col_indices).
// The kItems arcs of a lane go through four batched phases — locate, load the
// neighbour IDs, pre-test them (prefilter, e.g. the visited bitmap in L2),
// then visit the survivors — so each thread keeps kItems independent loads in
// flight instead of one dependent chain per arc.
// Arc positions are 32-bit offsets from the tile start (a tile holds at most
// kTile arcs): the staged row starts are clamped to [0, tile arcs] and each
// row keeps the col index its offset 0 maps to (mod 2^32), so locating an arc
// is 32-bit work; a lane finds its batch's row by galloping forward from the
// row of its previous batch (one probe on long rows) instead of a binary
// search over the whole chunk.
template <class F, bool kFused>
__global__ void __launch_bounds__(kExpBlock, expand_min_ctas<F>::value)
    lb_expand_kernel(F f, GraphView g, const uint32_t* __restrict__ in, uint32_t n_in,
                     const uint32_t* __restrict__ rowstart,
                     const unsigned long long* __restrict__ prefix,
                     const unsigned long long* __restrict__ block_off,
                     const unsigned long long* total_ptr, const uint32_t* __restrict__ tile_lo,
                     uint32_t* __restrict__ out, uint32_t* out_cnt,
                     const uint32_t* n_in_ptr = nullptr) {
  if (n_in_ptr) n_in = *n_in_ptr;
  __shared__ uint32_t s_pref[kStage + 1];  // row start - tile start, clamped to [0, tn]
  __shared__ uint32_t s_base[kStage];      // col index of tile offset 0 seen from the row
  __shared__ uint32_t s_src[kStage];
  __shared__ uint32_t s_q[kExpBlock / 32][kWarpQ];
  const unsigned long long total = *total_ptr;
  const unsigned long long ts = lb_tile_size(total);
  const unsigned long long ntiles = (total + ts - 1) / ts;
  const unsigned warp = threadIdx.x >> 5, lane = lane_id();
  const bool quiet = expand_quiet(f);
  const bool need_src = expand_needs_src(f);
  constexpr bool kLongRows = expand_long_rows<F>::value;
  WarpQueue<kWarpQ, kWarpQ - 32 * kItems> q;
  q.init(s_q[warp]);
  for (unsigned long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const unsigned long long t0 = tile * ts;
    const unsigned long long t1 = t0 + ts < total ? t0 + ts : total;
    const uint32_t tn = (uint32_t)(t1 - t0);
    const uint32_t lo = tile_lo[tile];
    const uint32_t hi = tile + 1 < ntiles ? tile_lo[tile + 1] : n_in - 1;
    const uint32_t R = hi - lo + 1;
    // The tile's vertex range is staged in chunks of at most kStage vertices, so
    // a tile of many low-degree rows (R up to kTile) still locates every arc in
    // shared memory; hub-heavy tiles need one chunk.
    for (uint32_t c0 = 0; c0 < R; c0 += kStage) {
    const uint32_t cR = R - c0 < (uint32_t)kStage ? R - c0 : (uint32_t)kStage;
    const uint32_t clo = lo + c0;
    __syncthreads();  // previous chunk done with the stage
    for (uint32_t j = threadIdx.x; j < cR; j += kExpBlock) {
      const unsigned long long p = lb_pref(prefix, block_off, clo + j);
      s_pref[j] = p <= t0 ? 0u : (p >= t1 ? tn : (uint32_t)(p - t0));
      s_base[j] = (uint32_t)((unsigned long long)rowstart[clo + j] + t0 - p);
      s_src[j] = in[clo + j];
    }
    if (threadIdx.x == 0) {
      const unsigned long long p = (clo + cR < n_in) ? lb_pref(prefix, block_off, clo + cR) : total;
      s_pref[cR] = p <= t0 ? 0u : (p >= t1 ? tn : (uint32_t)(p - t0));
    }
    __syncthreads();
    // arcs of this chunk inside the tile (tile offsets)
    const uint32_t a0 = s_pref[0], a1 = s_pref[cR];
    uint32_t j = 0;  // this lane's row: monotone over its batches
    // batches of 32*kItems arcs round-robin over the warps; lane l takes arcs
    // l, l+32, ... of its batch (coalesced col_indices)
    for (uint32_t e0 = a0 + warp * 32 * kItems + lane; e0 - lane < a1;
         e0 += (kExpBlock / 32) * 32 * kItems) {
      {
        // last row with s_pref <= key, galloping forward from j (s_pref[j] <= key)
        const uint32_t key = e0 < a1 ? e0 : a1 - 1;
        uint32_t step = 1;
        while (j + step < cR && s_pref[j + step] <= key) {
          j += step;
          step <<= 1;
        }
        uint32_t b = j + step < cR ? j + step - 1 : cR - 1;  // s_pref[b + 1] > key
        while (j < b) {
          const uint32_t m = (j + b + 1) >> 1;
          if (s_pref[m] <= key) j = m;
          else b = m - 1;
        }
      }
      uint32_t jnext = s_pref[j + 1];
      uint32_t eid[kItems], src[kItems], nb[kItems];
      const uint32_t elast = e0 + 32u * (kItems - 1);
      if (kLongRows && elast < jnext && elast < a1) {  // the lane's whole batch in row j
        const uint32_t b0 = s_base[j] + e0;
        const uint32_t s0 = need_src ? s_src[j] : 0u;
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          eid[k] = b0 + 32u * k;
          src[k] = s0;
        }
      } else {
#pragma unroll
        for (int k = 0; k < kItems; ++k) {  // locate: a short walk in shared memory
          const uint32_t e = e0 + 32u * k;
          eid[k] = 0xFFFFFFFFu;
          src[k] = 0u;
          if (e < a1) {
            while (e >= jnext) jnext = s_pref[++j + 1];
            eid[k] = s_base[j] + e;
            if (need_src) src[k] = s_src[j];
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kItems; ++k)  // neighbour IDs: independent, coalesced loads
        nb[k] = eid[k] != 0xFFFFFFFFu ? ld_stream(&g.col[eid[k]]) : 0u;
      bool pass[kItems];
#pragma unroll
      for (int k = 0; k < kItems; ++k)  // pre-tests: independent loads
        pass[k] = eid[k] != 0xFFFFFFFFu && f.prefilter(nb[k]);
      bool acc[kItems];
      visit_batch<kItems>(f, src, nb, eid, pass, acc);
      if (!quiet) {
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          bool a = acc[k];
          if (kFused && a) a = f.keep(nb[k]);
          q.push(a, nb[k]);
        }
        q.flush(out_cnt, out, false);
      }
    }
    }
  }
  q.flush(out_cnt, out, true);
}

// Persistent expansion grid: the CTAs that are resident at once (registers
// and shared memory of this instantiation, asked of the runtime once), so no
// second wave of CTAs starts late on a grid-stride share of the tiles.
template <class F, bool kFused>
inline unsigned expand_resident() {
  static unsigned per_sm = 0;
  if (!per_sm) {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, lb_expand_kernel<F, kFused>, kExpBlock, 0);
    per_sm = b > 0 ? static_cast<unsigned>(b) : 4u;
    if (const char* e = getenv("MG_EXPAND_CTAS_PER_SM")) per_sm = (unsigned)atoi(e);  // A/B
  }
  return num_sms() * per_sm;
}

// filter (engine.hpp:71-79): compaction by keep(v); input length read on device
template <class F>
__global__ void __launch_bounds__(256)
    filter_kernel(F f, const uint32_t* __restrict__ in, const uint32_t* in_cnt,
                  uint32_t* __restrict__ out, uint32_t* out_cnt) {
  uint32_t n = *in_cnt;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    uint32_t i = base + threadIdx.x;
    bool acc = false;
    uint32_t v = 0;
    if (i < n) {
      v = in[i];
      acc = f.keep(v);
    }
    uint32_t slot = warp_append(out_cnt, acc);
    if (acc) out[slot] = v;
  }
}

}  // namespace mgb
