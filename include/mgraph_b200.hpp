// mgraph_b200.hpp — header-only C++ mirror of the reference's public API
// (proj/core/include/mgraph/{csr,partition,engine,primitives}.hpp) over the
// C-ABI in mgraph_b200.h.  Same names, argument meaning and exception types,
// so the reference's callers (tools/mgraph.cpp run_once, the unit tests,
// acceptance.cpp) switch by changing the include and the namespace:
//
//     #include "mgraph_b200.hpp"
//     namespace mg = mgraph_b200;          // was: mgraph
//     mg::Csr g = mg::Csr::rmat(18, 16, 1);
//     auto plan = mg::build_partition_plan(g, mg::partition_random(g.num_vertices(), 4, 7),
//                                          mg::Duplication::All);
//     mg::BfsResult r = mg::bfs(plan, {.source = 0});
//
// Link: -L<repo>/paper_1504_04804_b200 -lmgraph_b200 (libmgraph_b200.so).
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mgraph_b200.h"

namespace mgraph_b200 {

using VertexId = uint32_t;
using EdgeId = uint32_t;
using Weight = uint32_t;
using Label = uint32_t;
using Dist = uint64_t;
using Value = double;

inline constexpr VertexId kInvalidVertex = MG_INVALID_VERTEX;
inline constexpr Label kInfLabel = MG_INF_LABEL;
inline constexpr Dist kInfDist = MG_INF_DIST;

// types.hpp:47-49
struct CapacityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
// status -> the reference's exception classes (SURVEY §8(b) "errors")
inline void check(int rc) {
  if (rc == MG_OK) return;
  std::string msg = mg_last_error();
  if (rc == MG_EINVAL) throw std::invalid_argument(msg);
  if (rc == MG_ECAPACITY) throw CapacityError(msg);
  throw std::runtime_error(msg);
}
template <class T>
T* ptr(std::vector<T>& v) {
  return v.empty() ? nullptr : v.data();
}
}  // namespace detail

// ---------------------------------------------------------------------------
// Csr (csr.hpp:38-52) — owned host CSR

struct WeightedEdge {
  VertexId src = 0, dst = 0;
  Weight weight = 0;
};
using EdgeList = std::vector<WeightedEdge>;

class Csr {
 public:
  Csr() = default;
  explicit Csr(mg_graph* h) : h_(h) {}
  Csr(Csr&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  Csr& operator=(Csr&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  Csr(const Csr&) = delete;
  ~Csr() {
    if (h_) mg_graph_destroy(h_);
  }

  // rmat_generate -> build_csr -> symmetrize_dedup (fixtures.hpp:56-63)
  static Csr rmat(int scale, int edge_factor, uint64_t seed, double a = 0.57, double b = 0.19,
                  double c = 0.19, double d = 0.05, bool symmetrize = true) {
    mg_graph* h = nullptr;
    detail::check(mg_graph_rmat(scale, edge_factor, a, b, c, d, seed, symmetrize ? 1 : 0, &h));
    return Csr(h);
  }
  // build_csr (csr.cpp:27-69)
  static Csr build(const EdgeList& edges, VertexId num_vertices, bool with_weights = false) {
    std::vector<uint32_t> s, t, w;
    for (const auto& e : edges) {
      s.push_back(e.src);
      t.push_back(e.dst);
      w.push_back(e.weight);
    }
    mg_graph* h = nullptr;
    detail::check(mg_graph_from_edges(num_vertices, edges.size(), detail::ptr(s), detail::ptr(t),
                                      with_weights ? detail::ptr(w) : nullptr, &h));
    return Csr(h);
  }
  static Csr path(VertexId n) {
    mg_graph* h = nullptr;
    detail::check(mg_graph_path(n, &h));
    return Csr(h);
  }
  static Csr grid(VertexId rows, VertexId cols) {
    mg_graph* h = nullptr;
    detail::check(mg_graph_grid(rows, cols, &h));
    return Csr(h);
  }
  Csr symmetrize_dedup() const {  // csr.cpp:82-108
    mg_graph* h = nullptr;
    detail::check(mg_graph_symmetrize(h_, &h));
    return Csr(h);
  }
  Csr with_random_weights(Weight lo, Weight hi, uint64_t seed) const {  // generate.cpp:64-79
    mg_graph* h = nullptr;
    detail::check(mg_graph_assign_weights(h_, lo, hi, seed, &h));
    return Csr(h);
  }

  VertexId num_vertices() const { return info().nv; }
  EdgeId num_edges() const { return static_cast<EdgeId>(info().ne); }
  bool has_weights() const { return info().w != 0; }
  const mg_graph* handle() const { return h_; }

 private:
  struct Info {
    uint32_t nv;
    uint64_t ne;
    int w;
  };
  Info info() const {
    Info i{};
    detail::check(mg_graph_info(h_, &i.nv, &i.ne, &i.w));
    return i;
  }
  mg_graph* h_ = nullptr;
};

// ---------------------------------------------------------------------------
// partitioners (partition.hpp) — kept from the reference

struct Assignment {
  std::vector<uint32_t> owner;
  uint32_t num_partitions = 1;
};

inline Assignment partition_random(VertexId num_vertices, uint32_t n, uint64_t seed) {
  Assignment a;
  a.owner.resize(num_vertices);
  a.num_partitions = n;
  detail::check(mg_partition_random(num_vertices, n, seed, detail::ptr(a.owner)));
  return a;
}

inline Assignment partition_biased_random(const Csr& g, uint32_t n, uint64_t seed, double bias) {
  Assignment a;
  a.owner.resize(g.num_vertices());
  a.num_partitions = n;
  detail::check(mg_partition_biased_random(g.handle(), n, seed, bias, detail::ptr(a.owner)));
  return a;
}

enum class Duplication { All, OneHop };

// build_partition_plan (partition.cpp:121-209) + upload to the GPU(s)
class PartitionPlan {
 public:
  PartitionPlan(const Csr& g, const Assignment& a, Duplication dup,
                const std::vector<int>& devices = {}) {
    detail::check(mg_plan_create(g.handle(), a.owner.data(), a.num_partitions,
                                 dup == Duplication::All ? MG_DUP_ALL : MG_DUP_ONEHOP,
                                 devices.empty() ? nullptr : devices.data(), &h_));
  }
  PartitionPlan(PartitionPlan&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  PartitionPlan(const PartitionPlan&) = delete;
  ~PartitionPlan() {
    if (h_) mg_plan_destroy(h_);
  }
  uint32_t num_partitions() const {
    uint32_t nv, n;
    uint64_t ne;
    detail::check(mg_plan_info(h_, &nv, &ne, &n));
    return n;
  }
  VertexId num_global_vertices() const {
    uint32_t nv, n;
    uint64_t ne;
    detail::check(mg_plan_info(h_, &nv, &ne, &n));
    return nv;
  }
  mg_plan* handle() const { return h_; }

 private:
  mg_plan* h_ = nullptr;
};

inline PartitionPlan build_partition_plan(const Csr& g, const Assignment& a, Duplication dup,
                                          const std::vector<int>& devices = {}) {
  return PartitionPlan(g, a, dup, devices);
}

// BorderMetrics (partition.cpp:211-242)
struct BorderMetrics {
  std::vector<std::vector<uint64_t>> pair_border;
  std::vector<uint64_t> partition_border;
  uint64_t total_border = 0;
  uint64_t edge_cut = 0;
};

inline BorderMetrics border_metrics(const PartitionPlan& plan) {
  const uint32_t n = plan.num_partitions();
  std::vector<uint64_t> flat(static_cast<size_t>(n) * n);
  BorderMetrics m;
  detail::check(mg_plan_border_metrics(plan.handle(), flat.data(), &m.edge_cut));
  m.pair_border.assign(n, std::vector<uint64_t>(n));
  m.partition_border.assign(n, 0);
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < n; ++j) {
      m.pair_border[i][j] = flat[i * n + j];
      m.partition_border[i] += flat[i * n + j];
      m.total_border += flat[i * n + j];
    }
  return m;
}

// ---------------------------------------------------------------------------
// engine configuration + statistics (engine.hpp:261-315, frontier.hpp:63-69)

enum class CommMode { Selective, Broadcast };
enum class AllocPolicyKind { JustEnough, FixedPrealloc, Maximum, PreallocFused };
enum class FusedMode { Auto, On, Off };
using SizingFactors = std::map<std::string, double>;

struct AllocationPolicy {
  AllocPolicyKind kind = AllocPolicyKind::JustEnough;
  SizingFactors factors;
  uint64_t hard_cap_bytes = 0;
};

struct DropPackage {
  uint32_t src = 0, dst = 0;
  uint64_t iteration = 0;
};

struct EngineConfig {
  AllocationPolicy policy;
  FusedMode fused = FusedMode::Auto;
  std::optional<CommMode> comm_override;
  uint32_t h_inflation = 1;
  std::optional<DropPackage> drop_package;
  uint64_t max_supersteps = 1000000;
  bool dobfs_exact_cost = false;  // extension: see mg_config

  mg_config to_c() const {
    mg_config c;
    mg_config_default(&c);
    c.policy = static_cast<int>(policy.kind);
    c.hard_cap_bytes = policy.hard_cap_bytes;
    static const char* roles[] = {"advance_output", "filter_output", "input_frontier", "outbox",
                                  "inbox"};
    for (int r = 0; r < MG_NUM_ROLES; ++r) {
      auto it = policy.factors.find(roles[r]);
      c.factors[r] = it == policy.factors.end() ? 0.0 : it->second;
    }
    c.fused = static_cast<int>(fused);
    c.comm_override = comm_override ? static_cast<int>(*comm_override) : MG_COMM_DEFAULT;
    c.h_inflation = h_inflation;
    if (drop_package) {
      c.drop_enabled = 1;
      c.drop_src = drop_package->src;
      c.drop_dst = drop_package->dst;
      c.drop_iteration = drop_package->iteration;
    }
    c.max_supersteps = max_supersteps;
    c.dobfs_exact_cost = dobfs_exact_cost ? 1 : 0;
    return c;
  }
};

struct RunStats {
  uint32_t n = 1;
  std::string communication = "selective", stop_reason;
  uint64_t supersteps = 0, edges_examined = 0, combine_ops = 0, wire_records = 0;
  uint64_t peak_bytes = 0, reallocs = 0;
  double wall_ms = 0, exchange_ms = 0, device_ms = 0;
  std::vector<std::vector<uint64_t>> h_matrix;
  std::vector<std::vector<uint64_t>> h_per_iter_by_src;
  std::vector<uint64_t> out_per_iter, edges_per_iter, combine_per_iter;

  uint64_t h_total() const {
    uint64_t t = 0;
    for (auto& r : h_matrix)
      for (auto v : r) t += v;
    return t;
  }
  uint64_t h_from(uint32_t i) const {
    uint64_t t = 0;
    for (auto v : h_matrix[i]) t += v;
    return t;
  }
};

namespace detail {
inline std::vector<uint64_t> last_array(mg_plan* p, int which) {
  uint64_t len = 0;
  check(mg_plan_last_array(p, which, nullptr, 0, &len));
  std::vector<uint64_t> v(len);
  check(mg_plan_last_array(p, which, v.data(), len, &len));
  return v;
}
inline RunStats stats(mg_plan* p, const mg_stats& s) {
  static const char* stops[] = {"frontiers_empty", "stop_condition", "max_supersteps",
                                "worker_error"};
  RunStats r;
  r.n = s.n;
  r.communication = s.communication == MG_COMM_BROADCAST ? "broadcast" : "selective";
  r.stop_reason = stops[s.stop_reason & 3];
  r.supersteps = s.supersteps;
  r.edges_examined = s.edges_examined;
  r.combine_ops = s.combine_ops;
  r.wire_records = s.wire_records;
  r.peak_bytes = s.peak_bytes;
  r.reallocs = s.reallocs;
  r.wall_ms = s.wall_ms;
  r.exchange_ms = s.exchange_ms;
  r.device_ms = s.device_ms;
  auto flat = last_array(p, MG_ARR_H_MATRIX);
  r.h_matrix.assign(s.n, std::vector<uint64_t>(s.n));
  for (uint32_t i = 0; i < s.n; ++i)
    for (uint32_t j = 0; j < s.n; ++j) r.h_matrix[i][j] = flat[i * s.n + j];
  auto hp = last_array(p, MG_ARR_H_PER_ITER);
  for (size_t k = 0; s.n && k + s.n <= hp.size(); k += s.n)
    r.h_per_iter_by_src.emplace_back(hp.begin() + k, hp.begin() + k + s.n);
  r.out_per_iter = last_array(p, MG_ARR_OUT_PER_ITER);
  r.edges_per_iter = last_array(p, MG_ARR_EDGES_PER_ITER);
  r.combine_per_iter = last_array(p, MG_ARR_COMBINE_PER_ITER);
  return r;
}
}  // namespace detail

// ---------------------------------------------------------------------------
// primitives (primitives.hpp)

struct BfsOptions {
  VertexId source = 0;
  bool mark_preds = false;
};
struct BfsResult {
  std::vector<Label> labels;
  std::vector<VertexId> preds;
  RunStats stats;
};

inline BfsResult bfs(const PartitionPlan& plan, const BfsOptions& opt,
                     const EngineConfig& cfg = {}) {
  BfsResult r;
  const VertexId nv = plan.num_global_vertices();
  r.labels.assign(nv, kInfLabel);
  if (opt.mark_preds) r.preds.assign(nv, kInvalidVertex);
  mg_config c = cfg.to_c();
  mg_stats s;
  detail::check(mg_bfs(plan.handle(), opt.source, opt.mark_preds, &c, r.labels.data(),
                       detail::ptr(r.preds), &s));
  r.stats = detail::stats(plan.handle(), s);
  return r;
}

enum class Direction { Forward, Backward };

struct DobfsOptions {
  VertexId source = 0;
  double do_a = 0.01;
  double do_b = 0.1;
  bool mark_preds = false;
};
struct DobfsResult {
  std::vector<Label> labels;
  std::vector<VertexId> preds;
  std::vector<int> direction_log;
  uint64_t forward_edges = 0, backward_edges = 0;
  RunStats stats;
};

inline DobfsResult dobfs(const PartitionPlan& plan, const DobfsOptions& opt,
                         const EngineConfig& cfg = {}) {
  DobfsResult r;
  const VertexId nv = plan.num_global_vertices();
  r.labels.assign(nv, kInfLabel);
  if (opt.mark_preds) r.preds.assign(nv, kInvalidVertex);
  std::vector<int32_t> dl(4096);
  uint64_t len = 0;
  mg_config c = cfg.to_c();
  mg_stats s;
  detail::check(mg_dobfs(plan.handle(), opt.source, opt.do_a, opt.do_b, opt.mark_preds, &c,
                         r.labels.data(), detail::ptr(r.preds), dl.data(), dl.size(), &len,
                         &r.forward_edges, &r.backward_edges, &s));
  r.direction_log.assign(dl.begin(), dl.begin() + (len < dl.size() ? len : dl.size()));
  r.stats = detail::stats(plan.handle(), s);
  return r;
}

struct SsspResult {
  std::vector<Dist> dists;
  std::vector<VertexId> preds;
  RunStats stats;
};

inline SsspResult sssp(const PartitionPlan& plan, VertexId source, bool mark_preds = false,
                       const EngineConfig& cfg = {}) {
  SsspResult r;
  const VertexId nv = plan.num_global_vertices();
  r.dists.assign(nv, kInfDist);
  if (mark_preds) r.preds.assign(nv, kInvalidVertex);
  mg_config c = cfg.to_c();
  mg_stats s;
  detail::check(mg_sssp(plan.handle(), source, mark_preds, &c, r.dists.data(),
                        detail::ptr(r.preds), &s));
  r.stats = detail::stats(plan.handle(), s);
  return r;
}

struct CcResult {
  std::vector<VertexId> components;
  RunStats stats;
};

inline CcResult cc(const PartitionPlan& plan, const EngineConfig& cfg = {}) {
  CcResult r;
  r.components.assign(plan.num_global_vertices(), 0);
  mg_config c = cfg.to_c();
  mg_stats s;
  detail::check(mg_cc(plan.handle(), &c, r.components.data(), &s));
  r.stats = detail::stats(plan.handle(), s);
  return r;
}

struct BcResult {
  std::vector<double> bc, sigma;
  std::vector<Label> labels;
  RunStats stats;
};

inline BcResult bc(const PartitionPlan& plan, VertexId source, const EngineConfig& cfg = {}) {
  BcResult r;
  const VertexId nv = plan.num_global_vertices();
  r.bc.assign(nv, 0.0);
  r.sigma.assign(nv, 0.0);
  r.labels.assign(nv, kInfLabel);
  mg_config c = cfg.to_c();
  mg_stats s;
  detail::check(mg_bc(plan.handle(), source, &c, r.bc.data(), r.sigma.data(), r.labels.data(),
                      &s));
  r.stats = detail::stats(plan.handle(), s);
  return r;
}

struct PrOptions {
  double damping = 0.85;
  double epsilon = 0.01;
  uint64_t max_iter = 1000;
};
struct PrResult {
  std::vector<double> ranks;
  uint64_t iterations = 0;
  std::vector<double> rank_sums;
  RunStats stats;
};

inline PrResult pagerank(const PartitionPlan& plan, const PrOptions& opt,
                         const EngineConfig& cfg = {}) {
  PrResult r;
  r.ranks.assign(plan.num_global_vertices(), 0.0);
  std::vector<double> sums(opt.max_iter + 2 < (1u << 20) ? opt.max_iter + 2 : (1u << 20));
  uint64_t len = 0;
  mg_config c = cfg.to_c();
  mg_stats s;
  detail::check(mg_pagerank(plan.handle(), opt.damping, opt.epsilon, opt.max_iter, &c,
                            r.ranks.data(), &r.iterations, sums.data(), sums.size(), &len, &s));
  r.rank_sums.assign(sums.begin(), sums.begin() + (len < sums.size() ? len : sums.size()));
  r.stats = detail::stats(plan.handle(), s);
  return r;
}

}  // namespace mgraph_b200
