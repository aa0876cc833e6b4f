// operators.cuh — the traversal operators as sm_100a kernels, templated on the
// primitive's device functors (the reference's advance/filter/fused operators,
// engine.hpp:54-99, and the functor hooks of PrimitiveSpec, engine.hpp:587-626).
//
// advance (load balanced):  each CTA takes a chunk of 256 frontier vertices,
//   block-scans their degrees in shared memory and expands the chunk's arcs
//   edge-parallel (merge-path style: thread i of the expansion finds its source
//   vertex by binary search over the 256-entry prefix), so consecutive lanes
//   read consecutive col_indices (coalesced).  Vertices with degree above
//   kBigDegree are deferred to a grid-wide pass over a global degree prefix, so
//   one hub (RMAT source: ~1e6 arcs) is spread over every SM.
// filter:  order-free compaction by keep(v) with warp-aggregated appends.
// Both count W (edges examined) exactly as the reference (= sum of degrees).
#pragma once

#include <cub/block/block_scan.cuh>

#include "plan.cuh"

namespace mgb {

constexpr int kAdvBlock = 256;
constexpr uint32_t kBigDegree = 2048;

// stage 1: chunked expansion of small/medium-degree vertices; big ones deferred
template <class F, bool kFused>
__global__ void __launch_bounds__(kAdvBlock)
    advance_chunk_kernel(F f, GraphView g, const uint32_t* __restrict__ in, uint32_t n_in,
                         uint32_t* __restrict__ out, uint32_t* out_cnt, uint32_t* big,
                         uint32_t* big_cnt, unsigned long long* edges) {
  using Scan = cub::BlockScan<uint32_t, kAdvBlock>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ uint32_t s_pref[kAdvBlock + 1];
  __shared__ uint32_t s_row[kAdvBlock];
  __shared__ uint32_t s_src[kAdvBlock];
  unsigned long long my_edges = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * kAdvBlock; base < n_in;
       base += (uint64_t)gridDim.x * kAdvBlock) {
    uint64_t i = base + threadIdx.x;
    uint32_t u = 0, deg = 0, row = 0;
    if (i < n_in) {
      u = in[i];
      row = g.off[u];
      deg = g.off[u + 1] - row;
      my_edges += deg;
      if (deg > kBigDegree) {
        uint32_t slot = atomicAdd(big_cnt, 1u);
        big[slot] = (uint32_t)i;
        deg = 0;
      }
    }
    uint32_t excl, total;
    Scan(scan_tmp).ExclusiveSum(deg, excl, total);
    s_pref[threadIdx.x] = excl;
    s_row[threadIdx.x] = row;
    s_src[threadIdx.x] = u;
    if (threadIdx.x == 0) s_pref[kAdvBlock] = total;
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < ((total + 31u) & ~31u); k += kAdvBlock) {
      bool acc = false;
      uint32_t v = 0;
      if (k < total) {
        // largest j with s_pref[j] <= k (degree-0 entries share prefixes)
        int lo = 0, hi = kAdvBlock - 1;
        while (lo < hi) {
          int mid = (lo + hi + 1) >> 1;
          if (s_pref[mid] <= k) lo = mid;
          else hi = mid - 1;
        }
        uint32_t e = s_row[lo] + (k - s_pref[lo]);
        v = g.col[e];
        acc = f.visit(s_src[lo], v, e);
        if (kFused && acc) acc = f.keep(v);
      }
      uint32_t slot = warp_append(out_cnt, acc);
      if (acc) out[slot] = v;
    }
    __syncthreads();
  }
  warp_add_u64(edges, my_edges);
}

// stage 2a: exclusive prefix of the deferred big vertices' degrees (one CTA)
static __global__ void __launch_bounds__(1024)
    big_prefix_kernel(GraphView g, const uint32_t* __restrict__ in, const uint32_t* big,
                      const uint32_t* big_cnt, unsigned long long* prefix) {
  using Scan = cub::BlockScan<unsigned long long, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  uint32_t nb = *big_cnt;
  for (uint32_t base = 0; base < nb; base += 1024) {
    uint32_t i = base + threadIdx.x;
    unsigned long long d = 0;
    if (i < nb) {
      uint32_t u = in[big[i]];
      d = g.off[u + 1] - g.off[u];
    }
    unsigned long long excl, total;
    Scan(tmp).ExclusiveSum(d, excl, total);
    if (i < nb) prefix[i] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) prefix[nb] = carry;
}

// stage 2b: edge-parallel expansion of the big vertices over the whole grid
template <class F, bool kFused>
__global__ void __launch_bounds__(kAdvBlock)
    advance_big_kernel(F f, GraphView g, const uint32_t* __restrict__ in, const uint32_t* big,
                       const uint32_t* big_cnt, const unsigned long long* __restrict__ prefix,
                       uint32_t* __restrict__ out, uint32_t* out_cnt) {
  uint32_t nb = *big_cnt;
  if (nb == 0) return;
  unsigned long long total = prefix[nb];
  const unsigned long long stride = (unsigned long long)gridDim.x * kAdvBlock;
  for (unsigned long long base = (unsigned long long)blockIdx.x * kAdvBlock; base < total;
       base += stride) {
    unsigned long long k = base + threadIdx.x;
    bool acc = false;
    uint32_t v = 0;
    if (k < total) {
      uint32_t lo = 0, hi = nb - 1;
      while (lo < hi) {
        uint32_t mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= k) lo = mid;
        else hi = mid - 1;
      }
      uint32_t u = in[big[lo]];
      uint32_t e = g.off[u] + (uint32_t)(k - prefix[lo]);
      v = g.col[e];
      acc = f.visit(u, v, e);
      if (kFused && acc) acc = f.keep(v);
    }
    uint32_t slot = warp_append(out_cnt, acc);
    if (acc) out[slot] = v;
  }
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
