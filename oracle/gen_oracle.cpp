// oracle/gen_oracle.cpp — TEST INFRASTRUCTURE ONLY (linked into oracle/_ref/libmgraph_ref.so,
// never into the product).
//
// Input synthesis for the reference side of the parity tests and of
// `bench.py --impl reference`, so that the reference arm never maps the
// product library:
//
//   ref_rmat_hashed_edges   the raw counter-based R-MAT draws (the benchmark
//                           generator of DESIGN.md §9; restated here from its
//                           definition: draw k of edge i is a 32-bit half of
//                           mix64(mix64(seed) + 64 i + k/2), quadrant
//                           thresholds floor({.57,.76,.95} * 2^32)).  At small
//                           scales the tests feed these edges through the
//                           reference's own build_csr + symmetrize_dedup
//                           (csr.cpp:27-108) to pin the parallel builder below.
//   ref_graph_rmat_hashed   the same draws, symmetrized and deduplicated with
//                           the reference's semantics (self-loops dropped, one
//                           arc per ordered pair, rows sorted by neighbour,
//                           csr.cpp:82-108) by a multi-threaded count / scatter /
//                           per-row sort+unique, straight into a reference
//                           mgraph::Csr.  RMAT-26 takes ~1 min on 16 threads
//                           where the reference's sequential symmetrize_dedup
//                           needs ~10 min and ~50 GB.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "mgraph/csr.hpp"
#include "mgraph_b200.h"

using namespace mgraph;

namespace {

thread_local std::string g_gen_err;

constexpr uint32_t kA = 2448131358u;    // floor(0.57 * 2^32)
constexpr uint32_t kAB = 3264175144u;   // floor(0.76 * 2^32)
constexpr uint32_t kABC = 4080218931u;  // floor(0.95 * 2^32)

inline void draw_edge(uint64_t sm, uint64_t i, int scale, uint32_t* u, uint32_t* v) {
  uint32_t uu = 0, vv = 0;
  uint64_t x = 0;
  for (int k = 0; k < scale; ++k) {
    if (!(k & 1)) x = mix64(sm + 64ull * i + static_cast<uint64_t>(k >> 1));
    const uint32_t r = (k & 1) ? static_cast<uint32_t>(x) : static_cast<uint32_t>(x >> 32);
    uu = (uu << 1) | (r >= kAB ? 1u : 0u);
    vv = (vv << 1) | (((r >= kA && r < kAB) || r >= kABC) ? 1u : 0u);
  }
  *u = uu;
  *v = vv;
}

template <class F>
void par(uint64_t n, unsigned threads, F&& f) {
  if (threads <= 1 || n < 4096) {
    f(0, n, 0u);
    return;
  }
  std::vector<std::thread> ts;
  for (unsigned t = 0; t < threads; ++t) {
    const uint64_t lo = n * t / threads, hi = n * (t + 1) / threads;
    ts.emplace_back([&f, lo, hi, t] { f(lo, hi, t); });
  }
  for (auto& t : ts) t.join();
}

// MG_GEN_TRACE=1: phase times on stderr
struct Phase {
  bool on = getenv("MG_GEN_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void operator()(const char* what) {
    if (!on) return;
    auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "[gen] %-10s %.2f s\n", what, std::chrono::duration<double>(n - t).count());
    t = n;
  }
};

unsigned pick_threads(int threads) {
  if (threads > 0) return static_cast<unsigned>(threads);
  unsigned h = std::thread::hardware_concurrency();
  return h ? h : 1u;
}

}  // namespace

extern "C" {

const char* ref_gen_last_error(void) { return g_gen_err.c_str(); }

// raw draws i in [0, 2^scale * ef): src[i], dst[i]
int ref_rmat_hashed_edges(int scale, int ef, uint64_t seed, uint32_t* src, uint32_t* dst) {
  if (scale < 1 || scale > 31 || ef < 1) {
    g_gen_err = "ref_rmat_hashed_edges: bad scale / edge factor";
    return MG_EINVAL;
  }
  const uint64_t m = (uint64_t{1} << scale) * static_cast<uint64_t>(ef);
  const uint64_t sm = mix64(seed);
  par(m, pick_threads(0), [&](uint64_t lo, uint64_t hi, unsigned) {
    for (uint64_t i = lo; i < hi; ++i) draw_edge(sm, i, scale, &src[i], &dst[i]);
  });
  return MG_OK;
}

int ref_graph_rmat_hashed(int scale, int ef, uint64_t seed, int threads, void** out) {
  try {
    if (scale < 1 || scale > 31 || ef < 1) throw std::invalid_argument("bad scale / edge factor");
    const unsigned T = pick_threads(threads);
    const uint32_t nv = uint32_t{1} << scale;
    const uint64_t m = uint64_t{nv} * static_cast<uint64_t>(ef);
    if (2 * m >= (uint64_t{1} << 32)) throw std::invalid_argument("arcs exceed 32-bit EdgeId");
    const uint64_t sm = mix64(seed);
    Phase ph;
    // 1. both arcs of every non-loop draw, counted per row.  R-MAT piles its
    //    arcs onto low IDs, so rows below `hot` are counted per thread (no
    //    shared-counter contention) and get a per-thread block of their row;
    //    the long tail of cold rows uses relaxed atomics.
    const uint32_t hot = nv < (1u << 18) ? nv : (1u << 18);
    std::vector<uint32_t> cnt(nv, 0);
    std::vector<std::vector<uint32_t>> hcnt(T, std::vector<uint32_t>(hot, 0));
    auto each_arc = [&](uint64_t lo, uint64_t hi, auto&& f) {
      for (uint64_t i = lo; i < hi; ++i) {
        uint32_t u, v;
        draw_edge(sm, i, scale, &u, &v);
        if (u == v) continue;  // self-loops removed (csr.cpp:90)
        f(u, v);
        f(v, u);
      }
    };
    par(m, T, [&](uint64_t lo, uint64_t hi, unsigned t) {
      uint32_t* hc = hcnt[t].data();
      each_arc(lo, hi, [&](uint32_t a, uint32_t) {
        if (a < hot) ++hc[a];
        else __atomic_fetch_add(&cnt[a], 1u, __ATOMIC_RELAXED);
      });
    });
    for (uint32_t v = 0; v < hot; ++v)
      for (unsigned t = 0; t < T; ++t) cnt[v] += hcnt[t][v];
    ph("count");
    std::vector<uint32_t> start(static_cast<size_t>(nv) + 1, 0);
    for (uint32_t v = 0; v < nv; ++v) start[v + 1] = start[v] + cnt[v];
    const uint64_t total = start[nv];
    // 2. scatter (regenerating the draws instead of storing them)
    std::vector<uint32_t> tmp(total);
    for (uint32_t v = 0; v < nv; ++v) cnt[v] = start[v];
    for (uint32_t v = 0; v < hot; ++v) {  // per-thread cursors of the hot rows
      uint32_t c = start[v];
      for (unsigned t = 0; t < T; ++t) {
        const uint32_t k = hcnt[t][v];
        hcnt[t][v] = c;
        c += k;
      }
    }
    par(m, T, [&](uint64_t lo, uint64_t hi, unsigned t) {
      uint32_t* hc = hcnt[t].data();
      each_arc(lo, hi, [&](uint32_t a, uint32_t b) {
        if (a < hot) tmp[hc[a]++] = b;
        else tmp[__atomic_fetch_add(&cnt[a], 1u, __ATOMIC_RELAXED)] = b;
      });
    });
    ph("scatter");
    // 3. per row: sort + unique (one arc per (src, dst), csr.cpp:100-105);
    //    rows split over threads by arc count
    std::vector<uint32_t> bounds(T + 1, nv);
    bounds[0] = 0;
    for (unsigned t = 1; t < T; ++t)
      bounds[t] = static_cast<uint32_t>(
          std::upper_bound(start.begin(), start.end(), total * t / T) - start.begin() - 1);
    std::vector<std::thread> ts;
    for (unsigned t = 0; t < T; ++t)
      ts.emplace_back([&, t] {
        for (uint32_t v = bounds[t]; v < bounds[t + 1]; ++v) {
          uint32_t* b = tmp.data() + start[v];
          uint32_t* e = tmp.data() + start[v + 1];
          std::sort(b, e);
          cnt[v] = static_cast<uint32_t>(std::unique(b, e) - b);
        }
      });
    for (auto& t : ts) t.join();
    ts.clear();
    ph("sort");
    // 4. compact into the reference Csr
    auto* g = new Csr();
    g->num_vertices = nv;
    g->row_offsets.assign(static_cast<size_t>(nv) + 1, 0);
    for (uint32_t v = 0; v < nv; ++v) g->row_offsets[v + 1] = g->row_offsets[v] + cnt[v];
    g->col_indices.resize(g->row_offsets[nv]);
    for (unsigned t = 0; t < T; ++t)
      ts.emplace_back([&, t] {
        for (uint32_t v = bounds[t]; v < bounds[t + 1]; ++v)
          std::memcpy(g->col_indices.data() + g->row_offsets[v], tmp.data() + start[v],
                      sizeof(uint32_t) * cnt[v]);
      });
    for (auto& t : ts) t.join();
    ph("compact");
    *out = g;
    return MG_OK;
  } catch (const std::invalid_argument& e) {
    g_gen_err = std::string("ref_graph_rmat_hashed: ") + e.what();
    return MG_EINVAL;
  } catch (const std::exception& e) {
    g_gen_err = std::string("ref_graph_rmat_hashed: ") + e.what();
    return MG_EWORKER;
  }
}

}  // extern "C"
