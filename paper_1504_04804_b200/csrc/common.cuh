// common.cuh — CUDA plumbing shared by every translation unit of the engine:
// error handling (status codes of include/mgraph_b200.h), launch accounting,
// warp-aggregated queue appends and the policy-aware device buffer that
// re-states the reference's CapVector/MemoryBudget (frontier.hpp:63-187).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "host_graph.hpp"
#include "mgraph_b200.h"

namespace mgb {

constexpr uint32_t kInfLabel = 0xFFFFFFFFu;
constexpr uint64_t kInfDist = 0xFFFFFFFFFFFFFFFFull;
constexpr int kMaxWorkers = 64;
constexpr int kMaxAssoc = 8;  // vertex / value associates per record (engine.hpp:645-646)
// B200 (sm_100a) has 148 SMs.  Device-side tiling heuristics use this design
// constant (kMinTiles, the BC bucket CTA count: layout, not correctness);
// host-side launch sizing asks the device (num_sms()), so grids stay
// multiples of the SM count on any part the library runs on.
constexpr int kB200SMs = 148;

extern std::atomic<uint64_t> g_launches;

#define MGB_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      throw ::mgb::Error(MG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e));   \
  } while (0)

// every kernel launch goes through here so gpu_launches is an exact count
#define MGB_LAUNCH(kernel, grid, block, smem, stream, ...)                               \
  do {                                                                                    \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                           \
    ::mgb::g_launches.fetch_add(1, std::memory_order_relaxed);                            \
    MGB_CUDA(cudaGetLastError());                                                         \
  } while (0)

// SM count of the current device (cached per ordinal)
inline unsigned num_sms() {
  static unsigned cache[64] = {};
  int d = 0;
  cudaGetDevice(&d);
  if (d < 0 || d >= 64) return kB200SMs;
  if (!cache[d]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    cache[d] = v > 0 ? static_cast<unsigned>(v) : kB200SMs;
  }
  return cache[d];
}

inline unsigned grid_for(uint64_t items, unsigned per_block, unsigned cap = 0) {
  if (!cap) cap = num_sms() * 8;
  uint64_t g = (items + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// ---------------------------------------------------------------------------
// device helpers

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Loads of arrays streamed once per superstep (col_indices, weights) are
// issued evict-first (ld.global.cs) so they do not push the randomly probed
// state arrays (labels, distances, bitmaps) out of L2 (measured: SSSP RMAT-24
// 12.4 -> 11.8 ms).
template <class T>
__device__ __forceinline__ T ld_stream(const T* p) {
  return __ldcs(p);
}

// Warp-aggregated append: every active lane with `pred` gets a slot in the
// queue; one atomicAdd per warp.  Returns the slot or 0xFFFFFFFF.
__device__ __forceinline__ uint32_t warp_append(uint32_t* counter, bool pred) {
  unsigned active = __activemask();
  unsigned mask = __ballot_sync(active, pred);
  if (!pred) return 0xFFFFFFFFu;
  unsigned leader = __ffs(mask) - 1;
  uint32_t base = 0;
  if (lane_id() == leader) base = atomicAdd(counter, (uint32_t)__popc(mask));
  base = __shfl_sync(mask, base, leader);
  return base + __popc(mask & ((1u << lane_id()) - 1u));
}

// CTA-aggregated queue append: items are staged in shared memory and the CTA
// reserves its output range with ONE global atomic per flush.  A single global
// counter hit by every warp serialises at its L2 slice (~1 op/ns); at 1e7+
// appends per superstep that, not HBM, would bound the kernel.
template <int kCap>
struct BlockQueue {
  uint32_t n, base;
  uint32_t buf[kCap];
  __device__ __forceinline__ void reset() {
    if (threadIdx.x == 0) n = 0;
  }
  // all threads of the warp that reach this call participate
  __device__ __forceinline__ void push(bool pred, uint32_t v) {
    unsigned active = __activemask();
    unsigned mask = __ballot_sync(active, pred);
    if (!mask) return;
    unsigned leader = __ffs(mask) - 1;
    uint32_t b = 0;
    if (lane_id() == leader) b = atomicAdd(&n, (uint32_t)__popc(mask));
    b = __shfl_sync(active, b, leader);
    if (pred) buf[b + __popc(mask & ((1u << lane_id()) - 1u))] = v;
  }
  // CTA-wide: requires __syncthreads() before (all pushes done) — performed here
  __device__ __forceinline__ void flush(uint32_t* counter, uint32_t* out) {
    __syncthreads();
    if (threadIdx.x == 0) base = n ? atomicAdd(counter, n) : 0u;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) out[base + i] = buf[i];
    __syncthreads();
    if (threadIdx.x == 0) n = 0;
    __syncthreads();
  }
};

// Warp-private staging queue in shared memory: no CTA barrier is involved;
// the warp reserves global space with one atomic per >= kFlush items, so the
// shared output counter sees ~items/kFlush atomics in total.
template <int kCap, int kFlush>
struct WarpQueue {
  uint32_t* buf;  // this warp's kCap-entry region of shared memory
  uint32_t n;     // warp-uniform fill level
  __device__ __forceinline__ void init(uint32_t* region) {
    buf = region;
    n = 0;
  }
  // every lane of the (full) warp must call push
  __device__ __forceinline__ void push(bool pred, uint32_t v) {
    unsigned mask = __ballot_sync(0xffffffffu, pred);
    if (pred) buf[n + __popc(mask & ((1u << lane_id()) - 1u))] = v;
    n += __popc(mask);
  }
  __device__ __forceinline__ void flush(uint32_t* counter, uint32_t* out, bool force) {
    if (n == 0 || (!force && n < (uint32_t)kFlush)) return;
    __syncwarp();
    uint32_t base = 0;
    if (lane_id() == 0) base = atomicAdd(counter, n);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (uint32_t i = lane_id(); i < n; i += 32) out[base + i] = buf[i];
    __syncwarp();
    n = 0;
  }
};

// Sums are skipped when zero: a kernel that found no work must not end with
// one same-address atomic per warp (~10^4 of them serialise at one L2 slice
// for ~15 us — measured on the empty DOBFS long-row stage).
__device__ __forceinline__ void warp_add_u64(unsigned long long* counter, uint64_t v) {
  unsigned active = __activemask();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(active, v, o);
  // lanes outside `active` contributed nothing; the lowest active lane adds
  if (v && lane_id() == (unsigned)(__ffs(active) - 1)) atomicAdd(counter, (unsigned long long)v);
}

// CTA-wide sums of N counters with ONE atomic per counter per CTA (zero sums
// and null counters skipped), for the totals a kernel reports at its end.
// Every thread of the CTA must call it, once per kernel.
template <int N>
__device__ __forceinline__ void block_add_u64(unsigned long long* const (&dst)[N],
                                              const uint64_t (&v)[N]) {
  __shared__ unsigned long long s_part[32][N];
  const unsigned warp = threadIdx.x >> 5, lane = lane_id(), nwarps = (blockDim.x + 31) >> 5;
  uint64_t x[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    x[i] = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x[i] += __shfl_xor_sync(0xffffffffu, x[i], o);
    if (lane == 0) s_part[warp][i] = x[i];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      uint64_t y = lane < nwarps ? s_part[lane][i] : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
      if (lane == 0 && y && dst[i]) atomicAdd(dst[i], (unsigned long long)y);
    }
  }
}

// ---------------------------------------------------------------------------
// policy-aware device buffer (CapVector + BufferStats + MemoryBudget)

struct BufferStats {  // frontier.hpp:71-81
  uint64_t realloc_count = 0, peak_items = 0, peak_bytes = 0;
  void merge(const BufferStats& o) {
    realloc_count += o.realloc_count;
    peak_items = peak_items > o.peak_items ? peak_items : o.peak_items;
    peak_bytes = peak_bytes > o.peak_bytes ? peak_bytes : o.peak_bytes;
  }
};

struct MemoryBudget {  // frontier.hpp:86-104
  uint64_t allocated = 0, peak = 0, hard_cap = 0;
  void charge(uint64_t add, uint64_t release) {
    allocated = allocated + add - release;
    if (allocated > peak) peak = allocated;
    if (hard_cap && allocated > hard_cap)
      throw Error(MG_ECAPACITY, "worker memory cap exceeded: need " + std::to_string(allocated) +
                                    " bytes, cap " + std::to_string(hard_cap) +
                                    " (graph does not fit under this budget)");
  }
};

// Device array with exact ("just-enough") growth: capacity extends to exactly
// the requested size, never speculatively; prealloc() is the policy's up-front
// sizing and is not counted as a reallocation (frontier.hpp:109-187).
// The LOGICAL capacity (`cap`, what the policy and the stats see) restarts at 0
// every run, while the physical allocation (`phys`) is kept across runs of the
// same plan, so a warm plan pays no cudaMalloc inside the timed region.
template <class T>
struct DevBuf {
  T* ptr = nullptr;
  uint64_t cap = 0;   // logical capacity (policy semantics)
  uint64_t phys = 0;  // allocated items
  BufferStats* stats = nullptr;
  MemoryBudget* budget = nullptr;

  void attach(BufferStats* s, MemoryBudget* b) {
    stats = s;
    budget = b;
  }
  // start of a run: logical capacity back to 0, memory kept
  void reset() {
    if (budget && cap) budget->allocated -= cap * sizeof(T);
    cap = 0;
  }
  void release() {
    reset();
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    phys = 0;
  }
  // grow to exactly `items`; contents up to `keep` items are preserved
  void grow(uint64_t items, bool counted, uint64_t keep, cudaStream_t s) {
    if (budget) budget->charge(items * sizeof(T), cap * sizeof(T));
    if (items > phys) {
      T* np = nullptr;
      MGB_CUDA(cudaMalloc(&np, items * sizeof(T) + 16));
      if (ptr) {
        if (keep)
          MGB_CUDA(cudaMemcpyAsync(np, ptr, keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
        MGB_CUDA(cudaStreamSynchronize(s));
        cudaFree(ptr);
      }
      ptr = np;
      phys = items;
    }
    cap = items;
    if (stats) {
      if (counted) ++stats->realloc_count;
      if (cap > stats->peak_items) stats->peak_items = cap;
      if (cap * sizeof(T) > stats->peak_bytes) stats->peak_bytes = cap * sizeof(T);
    }
  }
  void prealloc(uint64_t items, cudaStream_t s) {
    if (items > cap) grow(items, false, 0, s);
  }
  void ensure(uint64_t items, cudaStream_t s, uint64_t keep = 0) {
    if (items > cap) grow(items, true, keep, s);
  }
};

// plain owned device array (graph data, per-run state): no policy accounting
template <class T>
struct DevArray {
  T* ptr = nullptr;
  uint64_t n = 0;
  void alloc(uint64_t count) {
    free_();
    n = count;
    if (count) MGB_CUDA(cudaMalloc(&ptr, count * sizeof(T) + 16));
  }
  void free_() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    n = 0;
  }
  void upload(const T* h, uint64_t count, cudaStream_t s) {
    alloc(count);
    if (count) MGB_CUDA(cudaMemcpyAsync(ptr, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

void set_error(const std::string& msg);

}  // namespace mgb
