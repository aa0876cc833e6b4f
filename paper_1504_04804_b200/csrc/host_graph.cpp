// host_graph.cpp — host graph preparation + partitioners + plan builder.
// See host_graph.hpp for the contract; reference lines cited per function.
#include "host_graph.hpp"

#include <immintrin.h>

#include <algorithm>
#include <numeric>
#include <random>
#include <thread>

#include "mgraph_b200.h"
#include "rmat_hash.hpp"

namespace mgb {

namespace {

int pick_threads(int threads) {
  if (threads > 0) return threads;
  unsigned hc = std::thread::hardware_concurrency();
  return hc ? static_cast<int>(std::min(hc, 64u)) : 4;
}

template <class F>
void parallel_for(uint64_t n, int threads, F&& f) {
  threads = pick_threads(threads);
  if (n < 4096 || threads <= 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> ts;
  uint64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    uint64_t lo = t * chunk, hi = std::min<uint64_t>(n, lo + chunk);
    if (lo >= hi) break;
    ts.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& t : ts) t.join();
}

// sort every row by (dst, weight); weights travel with their arc
void sort_rows(HostCsr& g, int threads) {
  const bool weighted = g.weighted();
  parallel_for(g.nv, threads, [&](uint64_t lo, uint64_t hi) {
    std::vector<std::pair<uint32_t, uint32_t>> tmp;
    for (uint64_t v = lo; v < hi; ++v) {
      uint32_t b = g.off[v], e = g.off[v + 1];
      if (e - b <= 1) continue;
      if (!weighted) {
        std::sort(g.col.begin() + b, g.col.begin() + e);
        continue;
      }
      tmp.clear();
      for (uint32_t i = b; i < e; ++i) tmp.emplace_back(g.col[i], g.w[i]);
      std::sort(tmp.begin(), tmp.end());
      for (uint32_t i = b; i < e; ++i) {
        g.col[i] = tmp[i - b].first;
        g.w[i] = tmp[i - b].second;
      }
    }
  });
}

}  // namespace

// build_csr (csr.cpp:27-69): counting placement by source, rows sorted by
// neighbour (then weight), duplicates kept
HostCsr csr_from_arcs(const std::vector<Arc>& arcs, uint32_t nv, bool weighted) {
  for (const Arc& a : arcs) {
    if (a.src >= nv || a.dst >= nv)
      throw Error(MG_EINVAL, "build_csr: edge endpoint " + std::to_string(a.src) + "->" +
                                 std::to_string(a.dst) + " out of range [0," +
                                 std::to_string(nv) + ")");
  }
  if (arcs.size() > 0xFFFFFFFFull) throw Error(MG_EINVAL, "build_csr: more than 2^32-1 arcs");
  HostCsr g;
  g.nv = nv;
  g.off.assign(static_cast<size_t>(nv) + 1, 0);
  for (const Arc& a : arcs) g.off[a.src + 1]++;
  std::partial_sum(g.off.begin(), g.off.end(), g.off.begin());
  g.col.resize(arcs.size());
  if (weighted) g.w.resize(arcs.size());
  std::vector<uint32_t> cur(g.off.begin(), g.off.end() - 1);
  for (const Arc& a : arcs) {
    uint32_t pos = cur[a.src]++;
    g.col[pos] = a.dst;
    if (weighted) g.w[pos] = a.w;
  }
  sort_rows(g, 0);
  return g;
}

// symmetrize_dedup (csr.cpp:82-108): drop self-loops, mirror, keep one arc
// per (src,dst) with the minimum weight.  Same result as the reference's
// global sort, computed row-parallel: bucket mirrored arcs by source, then
// sort+unique each row.
HostCsr symmetrize_dedup(const HostCsr& g, int threads) {
  const bool weighted = g.weighted();
  const uint32_t nv = g.nv;
  std::vector<uint64_t> cnt(static_cast<size_t>(nv) + 1, 0);
  for (uint32_t u = 0; u < nv; ++u) {
    for (uint32_t e = g.off[u]; e < g.off[u + 1]; ++e) {
      uint32_t v = g.col[e];
      if (u == v) continue;
      cnt[u + 1]++;
      cnt[v + 1]++;
    }
  }
  std::partial_sum(cnt.begin(), cnt.end(), cnt.begin());
  std::vector<uint64_t> cur(cnt.begin(), cnt.end() - 1);
  std::vector<uint32_t> dst(cnt.back());
  std::vector<uint32_t> wt(weighted ? cnt.back() : 0);
  for (uint32_t u = 0; u < nv; ++u) {
    for (uint32_t e = g.off[u]; e < g.off[u + 1]; ++e) {
      uint32_t v = g.col[e];
      if (u == v) continue;
      uint64_t a = cur[u]++, b = cur[v]++;
      dst[a] = v;
      dst[b] = u;
      if (weighted) wt[a] = wt[b] = g.w[e];
    }
  }
  // per-row sort + unique (min weight first), then compact
  std::vector<uint32_t> keep(nv, 0);
  parallel_for(nv, threads, [&](uint64_t lo, uint64_t hi) {
    std::vector<std::pair<uint32_t, uint32_t>> tmp;
    for (uint64_t u = lo; u < hi; ++u) {
      uint64_t b = cnt[u], e = cnt[u + 1];
      if (e == b) continue;
      if (!weighted) {
        std::sort(dst.begin() + b, dst.begin() + e);
        uint64_t k = b;
        for (uint64_t i = b; i < e; ++i)
          if (i == b || dst[i] != dst[i - 1]) dst[k++] = dst[i];
        keep[u] = static_cast<uint32_t>(k - b);
      } else {
        tmp.clear();
        for (uint64_t i = b; i < e; ++i) tmp.emplace_back(dst[i], wt[i]);
        std::sort(tmp.begin(), tmp.end());
        uint64_t k = b;
        for (size_t i = 0; i < tmp.size(); ++i) {
          if (i && tmp[i].first == tmp[i - 1].first) continue;
          dst[k] = tmp[i].first;
          wt[k] = tmp[i].second;
          ++k;
        }
        keep[u] = static_cast<uint32_t>(k - b);
      }
    }
  });
  HostCsr out;
  out.nv = nv;
  out.off.assign(static_cast<size_t>(nv) + 1, 0);
  uint64_t total = 0;
  for (uint32_t u = 0; u < nv; ++u) {
    total += keep[u];
    if (total > 0xFFFFFFFFull) throw Error(MG_EINVAL, "symmetrize: more than 2^32-1 arcs");
    out.off[u + 1] = static_cast<uint32_t>(total);
  }
  out.col.resize(total);
  if (weighted) out.w.resize(total);
  parallel_for(nv, threads, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t u = lo; u < hi; ++u) {
      std::copy(dst.begin() + cnt[u], dst.begin() + cnt[u] + keep[u], out.col.begin() + out.off[u]);
      if (weighted)
        std::copy(wt.begin() + cnt[u], wt.begin() + cnt[u] + keep[u], out.w.begin() + out.off[u]);
    }
  });
  return out;
}

// assign_random_weights (generate.cpp:64-79): hash of the unordered pair
HostCsr assign_weights(const HostCsr& g, uint32_t lo, uint32_t hi, uint64_t seed) {
  if (lo > hi) throw Error(MG_EINVAL, "assign_random_weights: lo > hi");
  HostCsr out = g;
  out.w.assign(out.col.size(), 0);
  const uint64_t span = static_cast<uint64_t>(hi) - lo + 1;
  parallel_for(out.nv, 0, [&](uint64_t b, uint64_t e) {
    for (uint64_t u = b; u < e; ++u) {
      for (uint32_t i = out.off[u]; i < out.off[u + 1]; ++i) {
        uint64_t v = out.col[i];
        uint64_t x = std::min<uint64_t>(u, v), y = std::max<uint64_t>(u, v);
        uint64_t h = mix64(seed ^ mix64(x * 0x100000001b3ULL + y));
        out.w[i] = lo + static_cast<uint32_t>(h % span);
      }
    }
  });
  return out;
}

// validate_csr (csr.cpp:110-125)
void validate(const HostCsr& g) {
  if (g.off.size() != static_cast<size_t>(g.nv) + 1)
    throw Error(MG_EINVAL, "csr: row_offsets length mismatch");
  if (g.off.front() != 0) throw Error(MG_EINVAL, "csr: row_offsets[0] != 0");
  for (size_t v = 0; v < g.nv; ++v)
    if (g.off[v] > g.off[v + 1]) throw Error(MG_EINVAL, "csr: row_offsets not nondecreasing");
  if (g.col.size() != g.off.back()) throw Error(MG_EINVAL, "csr: col_indices length mismatch");
  for (uint32_t v : g.col)
    if (v >= g.nv) throw Error(MG_EINVAL, "csr: neighbor out of range");
  if (!g.w.empty() && g.w.size() != g.col.size())
    throw Error(MG_EINVAL, "csr: edge_values length mismatch");
}

// rmat_generate (generate.cpp:25-62): one mt19937_64 uniform double per bit
// per edge, quadrant by cumulative thresholds a, a+b, a+b+c
std::vector<Arc> rmat_arcs(int scale, int ef, double a, double b, double c, double d,
                           uint64_t seed) {
  if (scale < 1) throw Error(MG_EINVAL, "rmat_generate: scale must be >= 1");
  if (ef < 1) throw Error(MG_EINVAL, "rmat_generate: edge_factor must be >= 1");
  if (std::abs(a + b + c + d - 1.0) > 1e-9)
    throw Error(MG_EINVAL, "rmat_generate: quadrant probabilities must sum to 1");
  const uint64_t m = (1ull << scale) * static_cast<uint64_t>(ef);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  const double t1 = a, t2 = a + b, t3 = a + b + c;
  std::vector<Arc> arcs(m);
  for (uint64_t i = 0; i < m; ++i) {
    uint64_t u = 0, v = 0;
    for (int k = 0; k < scale; ++k) {
      double r = uni(rng);
      uint64_t bu = r >= t2 ? 1 : 0;
      uint64_t bv = (r >= t1 && r < t2) || r >= t3 ? 1 : 0;
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    arcs[i] = {static_cast<uint32_t>(u), static_cast<uint32_t>(v), 0};
  }
  return arcs;
}

std::vector<Arc> grid_arcs(uint32_t rows, uint32_t cols) {  // generate.cpp:81-92
  std::vector<Arc> e;
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t c = 0; c < cols; ++c) {
      uint32_t v = r * cols + c;
      if (c + 1 < cols) e.push_back({v, v + 1, 0});
      if (r + 1 < rows) e.push_back({v, v + cols, 0});
    }
  return e;
}

std::vector<Arc> path_arcs(uint32_t n) {  // generate.cpp:94-97
  std::vector<Arc> e;
  for (uint32_t v = 0; v + 1 < n; ++v) e.push_back({v, v + 1, 0});
  return e;
}

HostCsr rmat_hashed(int scale, int ef, uint64_t seed, int threads) {
  if (scale < 1 || scale > 31) throw Error(MG_EINVAL, "rmat_hashed: scale must be in [1,31]");
  if (ef < 1) throw Error(MG_EINVAL, "rmat_hashed: edge_factor must be >= 1");
  const uint64_t m = (1ull << scale) * static_cast<uint64_t>(ef);
  const uint32_t nv = 1u << scale;
  const uint64_t sm = mix64_hd(seed);
  std::vector<uint32_t> eu(m), ev(m);
  parallel_for(m, threads, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) rmat_hashed_edge(sm, i, scale, &eu[i], &ev[i]);
  });
  // directed CSR of the raw draws, then the reference's symmetrize_dedup
  HostCsr raw;
  raw.nv = nv;
  raw.off.assign(static_cast<size_t>(nv) + 1, 0);
  for (uint64_t i = 0; i < m; ++i) raw.off[eu[i] + 1]++;
  std::partial_sum(raw.off.begin(), raw.off.end(), raw.off.begin());
  raw.col.resize(m);
  std::vector<uint32_t> cur(raw.off.begin(), raw.off.end() - 1);
  for (uint64_t i = 0; i < m; ++i) raw.col[cur[eu[i]]++] = ev[i];
  std::vector<uint32_t>().swap(eu);
  std::vector<uint32_t>().swap(ev);
  return symmetrize_dedup(raw, threads);
}

// partition_random (partition.cpp:31-40)
std::vector<uint32_t> partition_random(uint32_t nv, uint32_t n, uint64_t seed) {
  if (n == 0) throw Error(MG_EINVAL, "partition_random: n == 0");
  std::vector<uint32_t> owner(nv);
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<uint32_t> pick(0, n - 1);
  for (auto& o : owner) o = pick(rng);
  return owner;
}

// partition_biased_random (partition.cpp:42-85): shuffled single pass; each
// vertex samples p with weight (1-bias)/n + bias * (share of its already
// assigned neighbours on p)
std::vector<uint32_t> partition_biased(const HostCsr& g, uint32_t n, uint64_t seed, double bias) {
  if (n == 0) throw Error(MG_EINVAL, "partition_biased_random: n == 0");
  if (bias < 0.0 || bias > 1.0)
    throw Error(MG_EINVAL, "partition_biased_random: bias outside [0,1]");
  std::vector<uint32_t> owner(g.nv, n);
  std::mt19937_64 rng(seed);
  std::vector<uint32_t> order(g.nv);
  std::iota(order.begin(), order.end(), 0u);
  std::shuffle(order.begin(), order.end(), rng);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  std::vector<double> wgt(n);
  std::vector<uint32_t> seen(n);
  for (uint32_t v : order) {
    std::fill(seen.begin(), seen.end(), 0u);
    uint64_t assigned = 0;
    for (uint32_t e = g.off[v]; e < g.off[v + 1]; ++e) {
      uint32_t o = owner[g.col[e]];
      if (o < n) {
        seen[o]++;
        assigned++;
      }
    }
    double total = 0.0;
    for (uint32_t p = 0; p < n; ++p) {
      double share = assigned ? static_cast<double>(seen[p]) / assigned : 1.0 / n;
      wgt[p] = (1.0 - bias) / n + bias * share;
      total += wgt[p];
    }
    double r = uni(rng) * total;
    uint32_t pick = n - 1;
    for (uint32_t p = 0; p < n; ++p) {
      if (r < wgt[p]) {
        pick = p;
        break;
      }
      r -= wgt[p];
    }
    owner[v] = pick;
  }
  return owner;
}

// build_partition_plan (partition.cpp:121-209)
HostPlan build_plan(const HostCsr& g, const std::vector<uint32_t>& owner, uint32_t n, int dup) {
  if (owner.size() != g.nv)
    throw Error(MG_EINVAL, "build_partition_plan: assignment length != |V|");
  if (n == 0) throw Error(MG_EINVAL, "build_partition_plan: n == 0");
  for (uint32_t o : owner)
    if (o >= n) throw Error(MG_EINVAL, "build_partition_plan: owner out of range");
  HostPlan P;
  P.n = n;
  P.dup = dup;
  P.nv = g.nv;
  P.ne = g.ne();
  P.owner = owner;
  P.locals.assign(n, {});
  for (uint32_t v = 0; v < g.nv; ++v) P.locals[owner[v]].push_back(v);

  // borders[i][j]: distinct out-neighbours of i's vertices hosted on j != i
  P.borders.assign(n, std::vector<std::vector<uint32_t>>(n));
  {
    std::vector<uint32_t> mark(g.nv, kInvalid);  // last partition that recorded v
    for (uint32_t p = 0; p < n; ++p) {
      for (uint32_t u : P.locals[p]) {
        for (uint32_t e = g.off[u]; e < g.off[u + 1]; ++e) {
          uint32_t v = g.col[e];
          uint32_t q = owner[v];
          if (q == p || mark[v] == p) continue;
          mark[v] = p;
          P.borders[p][q].push_back(v);
        }
      }
    }
    for (auto& row : P.borders)
      for (auto& b : row) std::sort(b.begin(), b.end());
  }

  const bool weighted = g.weighted();
  P.sub.resize(n);
  if (dup == MG_DUP_ALL) {
    for (uint32_t p = 0; p < n; ++p) {
      HostCsr& s = P.sub[p];
      s.nv = g.nv;
      s.off.assign(static_cast<size_t>(g.nv) + 1, 0);
      for (uint32_t u : P.locals[p]) s.off[u + 1] = g.deg(u);
      std::partial_sum(s.off.begin(), s.off.end(), s.off.begin());
      s.col.resize(s.off.back());
      if (weighted) s.w.resize(s.off.back());
      for (uint32_t u : P.locals[p]) {
        std::copy(g.col.begin() + g.off[u], g.col.begin() + g.off[u + 1], s.col.begin() + s.off[u]);
        if (weighted)
          std::copy(g.w.begin() + g.off[u], g.w.begin() + g.off[u + 1], s.w.begin() + s.off[u]);
      }
    }
  } else {
    P.l2g.resize(n);
    P.g2l.assign(n, std::vector<uint32_t>(g.nv, kInvalid));
    for (uint32_t p = 0; p < n; ++p) {
      std::vector<uint32_t>& l2g = P.l2g[p];
      std::vector<uint32_t>& g2l = P.g2l[p];
      l2g = P.locals[p];  // hosted first, IDs [0, |L_p|)
      std::vector<uint32_t> proxies;
      for (uint32_t q = 0; q < n; ++q)
        proxies.insert(proxies.end(), P.borders[p][q].begin(), P.borders[p][q].end());
      std::sort(proxies.begin(), proxies.end());
      proxies.erase(std::unique(proxies.begin(), proxies.end()), proxies.end());
      l2g.insert(l2g.end(), proxies.begin(), proxies.end());
      for (uint32_t l = 0; l < l2g.size(); ++l) g2l[l2g[l]] = l;
      HostCsr& s = P.sub[p];
      const uint32_t nl = static_cast<uint32_t>(P.locals[p].size());
      s.nv = static_cast<uint32_t>(l2g.size());
      s.off.assign(static_cast<size_t>(s.nv) + 1, 0);
      for (uint32_t l = 0; l < nl; ++l) s.off[l + 1] = g.deg(l2g[l]);
      std::partial_sum(s.off.begin(), s.off.end(), s.off.begin());
      s.col.resize(s.off.back());
      if (weighted) s.w.resize(s.off.back());
      for (uint32_t l = 0; l < nl; ++l) {
        uint32_t u = l2g[l], d = s.off[l];
        for (uint32_t e = g.off[u]; e < g.off[u + 1]; ++e, ++d) {
          s.col[d] = g2l[g.col[e]];
          if (weighted) s.w[d] = g.w[e];
        }
      }
    }
  }
  return P;
}

// Locality order for gather-heavy kernels (PageRank pull): the discovery order
// of a FIFO breadth-first search (Cuthill-McKee without the degree sort),
// started at the lowest-ID unvisited vertex of every component.  Neighbours
// end up within one BFS level band of each other, so a pull over rows in this
// order gathers from a narrow window instead of the whole vertex array.
// Returns perm[old] = new.
std::vector<uint32_t> bfs_locality_order(const uint32_t* off, const uint32_t* col, uint32_t nv) {
  std::vector<uint32_t> perm(nv, kInvalid), queue(nv);
  uint32_t next = 0;
  for (uint32_t s = 0; s < nv; ++s) {
    if (perm[s] != kInvalid) continue;
    uint32_t head = next, tail = next;
    perm[s] = next++;
    queue[tail++] = s;
    while (head < tail) {
      const uint32_t u = queue[head++];
      for (uint32_t e = off[u]; e < off[u + 1]; ++e) {
        const uint32_t v = col[e];
        if (perm[v] == kInvalid) {
          perm[v] = next++;
          queue[tail++] = v;
        }
      }
    }
  }
  return perm;
}

// byte levels -> u32 labels (255 -> kInvalid = the unreached label), the host
// half of the split label download; cloned for AVX2 where the CPU has it
__attribute__((target_clones("avx2", "default"))) void widen_labels_u8(const uint8_t* src,
                                                                         uint32_t* dst,
                                                                         size_t n) {
  for (size_t i = 0; i < n; ++i) {
    const uint32_t v = src[i];
    dst[i] = v == 255u ? kInvalid : v;
  }
}

// 4-bit levels (two per byte, 15 -> kInvalid) -> u32 labels [lo, hi)
static inline uint32_t nib_at(const uint8_t* src, size_t i) {
  const uint32_t v = (src[i >> 1] >> ((i & 1) * 4)) & 15u;
  return v == 15u ? kInvalid : v;
}

__attribute__((target("avx2"))) static void widen_labels_u4_avx2(const uint8_t* src,
                                                                  uint32_t* dst, size_t lo,
                                                                  size_t hi) {
  size_t i = lo;
  for (; i < hi && (i & 31); ++i) dst[i] = nib_at(src, i);
  const __m128i m4 = _mm_set1_epi8(0x0F);
  const __m256i f = _mm256_set1_epi32(15);
  for (; i + 32 <= hi; i += 32) {  // 16 bytes -> 32 labels
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + (i >> 1)));
    const __m128i l = _mm_and_si128(b, m4), h = _mm_and_si128(_mm_srli_epi16(b, 4), m4);
    const __m128i p0 = _mm_unpacklo_epi8(l, h), p1 = _mm_unpackhi_epi8(l, h);
    __m256i w[4] = {_mm256_cvtepu8_epi32(p0), _mm256_cvtepu8_epi32(_mm_srli_si128(p0, 8)),
                    _mm256_cvtepu8_epi32(p1), _mm256_cvtepu8_epi32(_mm_srli_si128(p1, 8))};
    for (int k = 0; k < 4; ++k) {
      w[k] = _mm256_or_si256(w[k], _mm256_cmpeq_epi32(w[k], f));  // 15 -> 0xFFFFFFFF
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i + 8 * k), w[k]);
    }
  }
  for (; i < hi; ++i) dst[i] = nib_at(src, i);
}

void widen_labels_u4(const uint8_t* src, uint32_t* dst, size_t lo, size_t hi) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) return widen_labels_u4_avx2(src, dst, lo, hi);
  for (size_t i = lo; i < hi; ++i) dst[i] = nib_at(src, i);
}

}  // namespace mgb
