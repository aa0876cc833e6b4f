// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// An extern "C" wrapper around the UNMODIFIED reference library compiled from
// /root/reference/proj/core/src/*.cpp (see oracle/Makefile).  It lets the
// parity tests, smoke() and bench.py's cpu_baseline / --impl reference leg call
// the reference's own engine (`run_primitive`, engine.hpp:712) and sequential
// oracles (reference.cpp:26-172) on exactly the inputs the CUDA path sees.
// Signatures mirror include/mgraph_b200.h with a `ref_` prefix; the status /
// stats structs are shared so both sides report the same RunStats fields.

#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "mgraph/csr.hpp"
#include "mgraph/generate.hpp"
#include "mgraph/partition.hpp"
#include "mgraph/primitives.hpp"
#include "mgraph/reference.hpp"
#include "mgraph_b200.h"

using namespace mgraph;

namespace {

thread_local std::string g_err;
thread_local RunStats g_last;

template <class F>
int guard(F&& f) {
  try {
    f();
    return MG_OK;
  } catch (const CapacityError& e) {
    g_err = e.what();
    return MG_ECAPACITY;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return MG_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MG_EWORKER;
  }
}

EngineConfig to_cfg(const mg_config* c) {
  EngineConfig cfg;
  if (!c) return cfg;
  cfg.policy.kind = static_cast<AllocPolicyKind>(c->policy);
  cfg.policy.hard_cap_bytes = c->hard_cap_bytes;
  static const char* roles[] = {"advance_output", "filter_output", "input_frontier", "outbox",
                                "inbox"};
  for (int r = 0; r < MG_NUM_ROLES; ++r)
    if (c->factors[r] != 0.0) cfg.policy.factors[roles[r]] = c->factors[r];
  cfg.fused = static_cast<FusedMode>(c->fused);
  if (c->comm_override >= 0) cfg.comm_override = static_cast<CommMode>(c->comm_override);
  cfg.h_inflation = c->h_inflation;
  if (c->drop_enabled) cfg.drop_package = DropPackage{c->drop_src, c->drop_dst, c->drop_iteration};
  cfg.max_supersteps = c->max_supersteps;
  return cfg;
}

void fill_stats(const RunStats& s, mg_stats* out) {
  g_last = s;
  if (!out) return;
  std::memset(out, 0, sizeof(*out));
  out->n = s.n;
  out->communication = s.communication == "broadcast" ? MG_COMM_BROADCAST : MG_COMM_SELECTIVE;
  out->stop_reason = s.stop_reason == "stop_condition"   ? MG_STOP_CONDITION
                     : s.stop_reason == "max_supersteps" ? MG_STOP_MAX_SUPERSTEPS
                     : s.stop_reason == "worker_error"   ? MG_STOP_WORKER_ERROR
                                                         : MG_STOP_FRONTIERS_EMPTY;
  out->supersteps = s.supersteps;
  out->edges_examined = s.edges_examined;
  out->combine_ops = s.combine_ops;
  out->h_total = s.h_total();
  out->wire_records = s.wire_records;
  out->peak_bytes = s.peak_bytes;
  out->reallocs = s.reallocs;
  out->wall_ms = s.wall_ms;
  out->exchange_ms = s.exchange_ms;
}

template <class T>
void copy_out(const std::vector<T>& v, T* dst) {
  if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(T));
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- graphs
int ref_graph_from_csr(uint32_t nv, uint64_t ne, const uint32_t* off, const uint32_t* col,
                       const uint32_t* w, void** out) {
  return guard([&] {
    auto* g = new Csr();
    g->num_vertices = nv;
    g->row_offsets.assign(off, off + nv + 1);
    g->col_indices.assign(col, col + ne);
    if (w) g->edge_values.assign(w, w + ne);
    validate_csr(*g);
    *out = g;
  });
}

int ref_graph_from_edges(uint32_t nv, uint64_t m, const uint32_t* src, const uint32_t* dst,
                         const uint32_t* w, void** out) {
  return guard([&] {
    EdgeList e(m);
    for (uint64_t i = 0; i < m; ++i) e[i] = {src[i], dst[i], w ? w[i] : 0u};
    *out = new Csr(build_csr(e, nv, w != nullptr));
  });
}

int ref_graph_rmat(int scale, int ef, uint64_t seed, int symmetrize, void** out) {
  return guard([&] {
    RmatParams p;
    p.scale = scale;
    p.edge_factor = ef;
    Csr g = build_csr(rmat_generate(p, seed), VertexId{1} << scale);
    *out = new Csr(symmetrize ? symmetrize_dedup(g) : std::move(g));
  });
}

int ref_graph_symmetrize(const void* g, void** out) {
  return guard([&] { *out = new Csr(symmetrize_dedup(*static_cast<const Csr*>(g))); });
}

int ref_graph_assign_weights(const void* g, uint32_t lo, uint32_t hi, uint64_t seed, void** out) {
  return guard(
      [&] { *out = new Csr(assign_random_weights(*static_cast<const Csr*>(g), lo, hi, seed)); });
}

int ref_graph_grid(uint32_t rows, uint32_t cols, void** out) {
  return guard([&] {
    *out = new Csr(symmetrize_dedup(build_csr(grid_edges(rows, cols), rows * cols)));
  });
}

int ref_graph_path(uint32_t n, void** out) {
  return guard([&] { *out = new Csr(symmetrize_dedup(build_csr(path_edges(n), n))); });
}

void ref_graph_info(const void* gp, uint32_t* nv, uint64_t* ne, int* w) {
  const Csr* g = static_cast<const Csr*>(gp);
  *nv = g->num_vertices;
  *ne = g->num_edges();
  *w = g->has_weights() ? 1 : 0;
}

void ref_graph_copy(const void* gp, uint32_t* off, uint32_t* col, uint32_t* w) {
  const Csr* g = static_cast<const Csr*>(gp);
  copy_out(g->row_offsets, off);
  copy_out(g->col_indices, col);
  copy_out(g->edge_values, w);
}

void ref_graph_destroy(void* g) { delete static_cast<Csr*>(g); }

// ---------------------------------------------------------------- partitioning
int ref_partition_random(uint32_t nv, uint32_t n, uint64_t seed, uint32_t* owner) {
  return guard([&] { copy_out(partition_random(nv, n, seed).owner, owner); });
}

int ref_partition_biased(const void* g, uint32_t n, uint64_t seed, double bias, uint32_t* owner) {
  return guard([&] {
    copy_out(partition_biased_random(*static_cast<const Csr*>(g), n, seed, bias).owner, owner);
  });
}

int ref_plan_create(const void* g, const uint32_t* owner, uint32_t n, int dup, void** out) {
  return guard([&] {
    const Csr* csr = static_cast<const Csr*>(g);
    Assignment a;
    a.num_partitions = n;
    a.owner.assign(owner, owner + csr->num_vertices);
    *out = new PartitionPlan(
        build_partition_plan(*csr, a, dup == MG_DUP_ALL ? Duplication::All : Duplication::OneHop));
  });
}

void ref_plan_destroy(void* p) { delete static_cast<PartitionPlan*>(p); }

// pair_border n*n, edge_cut
void ref_plan_border_metrics(const void* p, uint64_t* pair, uint64_t* cut) {
  BorderMetrics m = border_metrics(*static_cast<const PartitionPlan*>(p));
  uint32_t n = static_cast<uint32_t>(m.pair_border.size());
  if (pair)
    for (uint32_t i = 0; i < n; ++i)
      for (uint32_t j = 0; j < n; ++j) pair[i * n + j] = m.pair_border[i][j];
  if (cut) *cut = m.edge_cut;
}

// sub-graph of partition p: sizes then arrays (for plan-equality tests)
void ref_plan_subgraph_info(const void* pp, uint32_t p, uint32_t* nv, uint64_t* ne,
                            uint32_t* nlocal) {
  const PartitionPlan* plan = static_cast<const PartitionPlan*>(pp);
  *nv = plan->subgraphs[p].num_vertices;
  *ne = plan->subgraphs[p].num_edges();
  *nlocal = plan->local_count(p);
}

void ref_plan_subgraph_copy(const void* pp, uint32_t p, uint32_t* off, uint32_t* col,
                            uint32_t* w, uint32_t* l2g) {
  const PartitionPlan* plan = static_cast<const PartitionPlan*>(pp);
  const Csr& s = plan->subgraphs[p];
  copy_out(s.row_offsets, off);
  copy_out(s.col_indices, col);
  copy_out(s.edge_values, w);
  if (l2g && plan->duplication == Duplication::OneHop) copy_out(plan->local_to_global[p], l2g);
}

// ---------------------------------------------------------------- primitives
int ref_bfs(const void* p, uint32_t src, int preds, const mg_config* c, uint32_t* labels,
            uint32_t* pred_out, mg_stats* st) {
  return guard([&] {
    BfsResult r = bfs(*static_cast<const PartitionPlan*>(p),
                      {.source = src, .mark_preds = preds != 0}, to_cfg(c));
    copy_out(r.labels, labels);
    copy_out(r.preds, pred_out);
    fill_stats(r.stats, st);
  });
}

int ref_dobfs(const void* p, uint32_t src, double do_a, double do_b, int preds,
              const mg_config* c, uint32_t* labels, uint32_t* pred_out, int32_t* dirlog,
              uint64_t cap, uint64_t* len, uint64_t* fwd, uint64_t* bwd, mg_stats* st) {
  return guard([&] {
    DobfsResult r = dobfs(*static_cast<const PartitionPlan*>(p),
                          {.source = src, .do_a = do_a, .do_b = do_b, .mark_preds = preds != 0},
                          to_cfg(c));
    copy_out(r.labels, labels);
    copy_out(r.preds, pred_out);
    if (len) *len = r.direction_log.size();
    for (uint64_t i = 0; dirlog && i < r.direction_log.size() && i < cap; ++i)
      dirlog[i] = r.direction_log[i];
    if (fwd) *fwd = r.forward_edges;
    if (bwd) *bwd = r.backward_edges;
    fill_stats(r.stats, st);
  });
}

int ref_sssp(const void* p, uint32_t src, int preds, const mg_config* c, uint64_t* dists,
             uint32_t* pred_out, mg_stats* st) {
  return guard([&] {
    SsspResult r = sssp(*static_cast<const PartitionPlan*>(p), src, preds != 0, to_cfg(c));
    copy_out(r.dists, reinterpret_cast<Dist*>(dists));
    copy_out(r.preds, pred_out);
    fill_stats(r.stats, st);
  });
}

int ref_cc(const void* p, const mg_config* c, uint32_t* comp, mg_stats* st) {
  return guard([&] {
    CcResult r = cc(*static_cast<const PartitionPlan*>(p), to_cfg(c));
    copy_out(r.components, comp);
    fill_stats(r.stats, st);
  });
}

int ref_bc(const void* p, uint32_t src, const mg_config* c, double* bcv, double* sigma,
           uint32_t* labels, mg_stats* st) {
  return guard([&] {
    BcResult r = bc(*static_cast<const PartitionPlan*>(p), src, to_cfg(c));
    copy_out(r.bc, bcv);
    copy_out(r.sigma, sigma);
    copy_out(r.labels, labels);
    fill_stats(r.stats, st);
  });
}

int ref_pagerank(const void* p, double damping, double eps, uint64_t max_iter, const mg_config* c,
                 double* ranks, uint64_t* iters, double* sums, uint64_t cap, uint64_t* len,
                 mg_stats* st) {
  return guard([&] {
    PrResult r = pagerank(*static_cast<const PartitionPlan*>(p),
                          {.damping = damping, .epsilon = eps, .max_iter = max_iter}, to_cfg(c));
    copy_out(r.ranks, ranks);
    if (iters) *iters = r.iterations;
    if (len) *len = r.rank_sums.size();
    for (uint64_t i = 0; sums && i < r.rank_sums.size() && i < cap; ++i) sums[i] = r.rank_sums[i];
    fill_stats(r.stats, st);
  });
}

// arrays of the last run on this thread (same `which` codes as the product)
uint64_t ref_last_array(int which, uint64_t* buf, uint64_t cap) {
  std::vector<uint64_t> flat;
  const RunStats& s = g_last;
  switch (which) {
    case MG_ARR_H_MATRIX:
      for (const auto& row : s.h_matrix) flat.insert(flat.end(), row.begin(), row.end());
      break;
    case MG_ARR_H_PER_ITER:
      for (const auto& row : s.h_per_iter_by_src) flat.insert(flat.end(), row.begin(), row.end());
      break;
    case MG_ARR_OUT_PER_ITER: flat = s.out_per_iter; break;
    case MG_ARR_EDGES_PER_ITER: flat = s.edges_per_iter; break;
    case MG_ARR_COMBINE_PER_ITER: flat = s.combine_per_iter; break;
    default: break;
  }
  for (uint64_t i = 0; buf && i < flat.size() && i < cap; ++i) buf[i] = flat[i];
  return flat.size();
}

void ref_last_buffer_stats(uint32_t worker, int role, uint64_t* reallocs, uint64_t* peak_items,
                           uint64_t* peak_bytes) {
  *reallocs = *peak_items = *peak_bytes = 0;
  if (worker >= g_last.worker_buffers.size()) return;
  auto it = g_last.worker_buffers[worker].find(static_cast<BufferRole>(role));
  if (it == g_last.worker_buffers[worker].end()) return;
  *reallocs = it->second.realloc_count;
  *peak_items = it->second.peak_items;
  *peak_bytes = it->second.peak_bytes;
}

int ref_direction_decide(int current, double fv, double bv, double do_a, double do_b,
                         int switched) {
  DirectionState s;
  s.current = current ? Direction::Backward : Direction::Forward;
  s.fv = fv;
  s.bv = bv;
  s.do_a = do_a;
  s.do_b = do_b;
  s.switched_to_backward_once = switched != 0;
  return direction_decide(s) == Direction::Backward ? 1 : 0;
}

// ---------------------------------------------------------------- sequential oracles
void ref_seq_bfs(const void* g, uint32_t src, uint32_t* out) {
  copy_out(reference::bfs_levels(*static_cast<const Csr*>(g), src), out);
}
void ref_seq_dijkstra(const void* g, uint32_t src, uint64_t* out) {
  copy_out(reference::dijkstra(*static_cast<const Csr*>(g), src), reinterpret_cast<Dist*>(out));
}
void ref_seq_cc(const void* g, uint32_t* out) {
  copy_out(reference::connected_components(*static_cast<const Csr*>(g)), out);
}
void ref_seq_bc(const void* g, uint32_t src, double* out) {
  copy_out(reference::brandes_bc(*static_cast<const Csr*>(g), src), out);
}
uint64_t ref_seq_pagerank(const void* g, double d, double eps, uint64_t max_iter, double* ranks,
                          double* sums, uint64_t cap) {
  auto r = reference::pagerank_power(*static_cast<const Csr*>(g), d, eps, max_iter);
  copy_out(r.ranks, ranks);
  for (uint64_t i = 0; sums && i < r.rank_sums.size() && i < cap; ++i) sums[i] = r.rank_sums[i];
  return r.iterations;
}

}  // extern "C"
