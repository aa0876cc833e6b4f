// rmat_hash.hpp — counter-based R-MAT edge draw shared by the host generator
// (host_graph.cpp) and the device generator (gen.cu), so both produce the same
// edge list bit for bit.  The reference generator (generate.cpp:25-62) draws one
// mt19937_64 uniform per bit per edge sequentially, which cannot be generated in
// parallel; this variant keeps its quadrant probabilities (a,b,c,d) =
// (0.57,0.19,0.19,0.05) and its exact edge count 2^scale * edge_factor, with
// draw (i,k) = 32-bit half of mix64(mix64(seed) + 64*i + k/2).
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define MGB_HD __host__ __device__ __forceinline__
#else
#define MGB_HD inline
#endif

namespace mgb {

MGB_HD uint64_t mix64_hd(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// thresholds for a, a+b, a+b+c in 32-bit fixed point
constexpr uint32_t kRmatA = 2448131358u;    // floor(0.57 * 2^32)
constexpr uint32_t kRmatAB = 3264175144u;   // floor(0.76 * 2^32)
constexpr uint32_t kRmatABC = 4080218931u;  // floor(0.95 * 2^32)

MGB_HD void rmat_hashed_edge(uint64_t seed_mixed, uint64_t i, int scale, uint32_t* u,
                             uint32_t* v) {
  uint32_t uu = 0, vv = 0;
  for (int k = 0; k < scale; k += 2) {
    uint64_t x = mix64_hd(seed_mixed + 64ull * i + (uint64_t)(k >> 1));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (k + h >= scale) break;
      uint32_t r = h ? (uint32_t)x : (uint32_t)(x >> 32);
      uint32_t bu = r >= kRmatAB ? 1u : 0u;                  // quadrants c, d
      uint32_t bv = (r >= kRmatA && r < kRmatAB) || r >= kRmatABC ? 1u : 0u;  // b, d
      uu = (uu << 1) | bu;
      vv = (vv << 1) | bv;
    }
  }
  *u = uu;
  *v = vv;
}

}  // namespace mgb
