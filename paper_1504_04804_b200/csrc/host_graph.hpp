// host_graph.hpp — host-side graph preparation and partition planning.
//
// These are the pieces the north star says are KEPT from the reference: CSR
// construction (csr.cpp:27-108), the generators (generate.cpp:25-97) and the
// random / border-minimising partitioners + plan builder (partition.cpp:31-209).
// They are re-stated here (no reference source is compiled into the product)
// and produce bit-identical outputs for the same seeds because they drive the
// same libstdc++ engines (std::mt19937_64, uniform_*_distribution, shuffle)
// in the same call order.  tests/test_host.py checks that equality against the
// reference built in oracle/_ref.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace mgb {

constexpr uint32_t kInvalid = 0xFFFFFFFFu;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// reference Csr (csr.hpp:38-52): u32 offsets, u32 columns, optional u32 weights
struct HostCsr {
  uint32_t nv = 0;
  std::vector<uint32_t> off;  // nv + 1
  std::vector<uint32_t> col;
  std::vector<uint32_t> w;    // empty or ne

  uint64_t ne() const { return off.empty() ? 0 : off.back(); }
  bool weighted() const { return !w.empty(); }
  uint32_t deg(uint32_t v) const { return off[v + 1] - off[v]; }
};

struct Arc {
  uint32_t src, dst, w;
};

inline uint64_t mix64(uint64_t x) {  // splitmix64 finaliser (types.hpp:53-58)
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

HostCsr csr_from_arcs(const std::vector<Arc>& arcs, uint32_t nv, bool weighted);
HostCsr symmetrize_dedup(const HostCsr& g, int threads = 0);
HostCsr assign_weights(const HostCsr& g, uint32_t lo, uint32_t hi, uint64_t seed);
void validate(const HostCsr& g);
std::vector<Arc> rmat_arcs(int scale, int ef, double a, double b, double c, double d,
                           uint64_t seed);
std::vector<Arc> grid_arcs(uint32_t rows, uint32_t cols);
std::vector<Arc> path_arcs(uint32_t n);

// counter-based R-MAT (host twin of the device generator in gen.cu)
HostCsr rmat_hashed(int scale, int ef, uint64_t seed, int threads);

std::vector<uint32_t> partition_random(uint32_t nv, uint32_t n, uint64_t seed);
std::vector<uint32_t> partition_biased(const HostCsr& g, uint32_t n, uint64_t seed, double bias);

// build_partition_plan (partition.cpp:121-209)
struct HostPlan {
  uint32_t n = 1;
  int dup = 0;  // 0 All, 1 OneHop
  uint32_t nv = 0;
  uint64_t ne = 0;
  std::vector<uint32_t> owner;
  std::vector<std::vector<uint32_t>> locals;               // hosted global IDs, sorted
  std::vector<std::vector<std::vector<uint32_t>>> borders;  // [i][j] sorted global IDs
  std::vector<HostCsr> sub;                                 // per-partition sub-graph
  std::vector<std::vector<uint32_t>> l2g, g2l;              // OneHop only
};

HostPlan build_plan(const HostCsr& g, const std::vector<uint32_t>& owner, uint32_t n, int dup);

// u8 levels (255 = unreached) -> u32 labels (split label download, plan.cu)
void widen_labels_u8(const uint8_t* src, uint32_t* dst, size_t n);
void widen_labels_u4(const uint8_t* src, uint32_t* dst, size_t lo, size_t hi);

// FIFO-BFS (Cuthill-McKee order without degree sort) vertex order: perm[old] = new
std::vector<uint32_t> bfs_locality_order(const uint32_t* off, const uint32_t* col, uint32_t nv);

// counter-based R-MAT draw shared by host and device: edge i, bit k
struct RmatThresholds {
  uint32_t a, ab, abc;
};
inline RmatThresholds rmat_thresholds() {
  // a=0.57, b=c=0.19, d=0.05 (generate.hpp:30) as 32-bit fixed point
  return {uint32_t(0.57 * 4294967296.0), uint32_t(0.76 * 4294967296.0),
          uint32_t(0.95 * 4294967296.0)};
}

}  // namespace mgb
