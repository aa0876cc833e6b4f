// api.cu — C-ABI surface for graphs, partitioners, plans and run statistics
// (include/mgraph_b200.h).  Primitive entry points live in prims.cu.
#include <cstring>
#include <functional>
#include <memory>

#include "engine.cuh"

namespace mgb {
const char* last_error();
int run_guarded(const std::function<void()>& f);
Plan* plan_from_host(const HostPlan& H, const int* devices, std::shared_ptr<HostCsr> g, int only);
}  // namespace mgb

using namespace mgb;


namespace {
int wrap(const std::function<void()>& f) { return run_guarded(f); }

// undirected cut of a device-resident graph (border_metrics, partition.cpp:
// 224-240): arcs (u,v) with different owners, each pair once — from the
// smaller endpoint, or from u when the reverse arc is absent (rows sorted:
// binary search).  One warp per row.
__global__ void edge_cut_kernel(const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                                const uint8_t* __restrict__ owner, uint32_t nv,
                                unsigned long long* out) {
  unsigned long long c = 0;
  const uint32_t warps = gridDim.x * blockDim.x / 32;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) / 32; u < nv; u += warps) {
    const uint8_t ou = owner[u];
    for (uint32_t e = off[u] + lane_id(); e < off[u + 1]; e += 32) {
      const uint32_t v = col[e];
      if (owner[v] == ou) continue;
      if (v > u) {
        ++c;
        continue;
      }
      uint32_t lo = off[v], hi = off[v + 1];
      while (lo < hi) {
        const uint32_t m = (lo + hi) >> 1;
        if (col[m] < u) lo = m + 1;
        else hi = m;
      }
      if (lo == off[v + 1] || col[lo] != u) ++c;
    }
  }
  warp_add_u64(out, c);
}

uint64_t device_edge_cut(Plan& P) {
  if (P.n == 1) return 0;
  const uint32_t me = P.local_workers.front();
  Worker& w = *P.workers[me];
  const bool single = !P.g_off.ptr && P.n == 1;
  if (!P.g_off.ptr && !single) throw Error(MG_EINVAL, "plan holds no global graph");
  const uint32_t* d_off = single ? w.off.ptr : P.g_off.ptr;
  const uint32_t* d_col = single ? w.col.ptr : P.g_col.ptr;
  DeviceGuard dg(w.dev);
  DevArray<unsigned long long> out;
  out.alloc(1);
  MGB_CUDA(cudaMemsetAsync(out.ptr, 0, 8, w.stream));
  MGB_LAUNCH(edge_cut_kernel, grid_for((uint64_t)P.nv * 32, 256, num_sms() * 16), 256, 0, w.stream,
             d_off, d_col, w.owner.ptr, P.nv, out.ptr);
  unsigned long long c = 0;
  MGB_CUDA(cudaMemcpyAsync(&c, out.ptr, 8, cudaMemcpyDeviceToHost, w.stream));
  MGB_CUDA(cudaStreamSynchronize(w.stream));
  return c;
}
mg_graph* box(HostCsr&& g) { return new mg_graph{std::make_shared<HostCsr>(std::move(g))}; }
Plan& plan_of(const mg_plan* p) {
  if (!p) throw Error(MG_EINVAL, "null plan");
  return *reinterpret_cast<Plan*>(const_cast<mg_plan*>(p));
}
}  // namespace

extern "C" {

const char* mg_last_error(void) { return last_error(); }
const char* mg_version(void) { return "mgraph-b200 0.1 (sm_100a)"; }
uint64_t mg_kernel_launch_count(void) { return g_launches.load(); }

int mg_graph_from_csr(uint32_t nv, uint64_t ne, const uint32_t* off, const uint32_t* col,
                      const uint32_t* w, mg_graph** out) {
  return wrap([&] {
    HostCsr g;
    g.nv = nv;
    g.off.assign(off, off + nv + 1);
    g.col.assign(col, col + ne);
    if (w) g.w.assign(w, w + ne);
    validate(g);
    *out = box(std::move(g));
  });
}

int mg_graph_from_edges(uint32_t nv, uint64_t m, const uint32_t* src, const uint32_t* dst,
                        const uint32_t* w, mg_graph** out) {
  return wrap([&] {
    std::vector<Arc> arcs(m);
    for (uint64_t i = 0; i < m; ++i) arcs[i] = {src[i], dst[i], w ? w[i] : 0u};
    *out = box(csr_from_arcs(arcs, nv, w != nullptr));
  });
}

int mg_graph_rmat(int scale, int ef, double a, double b, double c, double d, uint64_t seed,
                  int symmetrize, mg_graph** out) {
  return wrap([&] {
    if (scale < 1 || scale > 31) throw Error(MG_EINVAL, "rmat_generate: scale must be in [1,31]");
    HostCsr g = csr_from_arcs(rmat_arcs(scale, ef, a, b, c, d, seed), 1u << scale, false);
    *out = box(symmetrize ? symmetrize_dedup(g) : std::move(g));
  });
}

int mg_graph_symmetrize(const mg_graph* g, mg_graph** out) {
  return wrap([&] { *out = box(symmetrize_dedup(*g->g)); });
}

int mg_graph_assign_weights(const mg_graph* g, uint32_t lo, uint32_t hi, uint64_t seed,
                            mg_graph** out) {
  return wrap([&] { *out = box(assign_weights(*g->g, lo, hi, seed)); });
}

int mg_graph_grid(uint32_t rows, uint32_t cols, mg_graph** out) {
  return wrap([&] {
    *out = box(symmetrize_dedup(csr_from_arcs(grid_arcs(rows, cols), rows * cols, false)));
  });
}

int mg_graph_path(uint32_t n, mg_graph** out) {
  return wrap([&] { *out = box(symmetrize_dedup(csr_from_arcs(path_arcs(n), n, false))); });
}

int mg_graph_info(const mg_graph* g, uint32_t* nv, uint64_t* ne, int* w) {
  return wrap([&] {
    if (nv) *nv = g->g->nv;
    if (ne) *ne = g->g->ne();
    if (w) *w = g->g->weighted() ? 1 : 0;
  });
}

int mg_graph_arrays(const mg_graph* g, const uint32_t** off, const uint32_t** col,
                    const uint32_t** w) {
  return wrap([&] {
    if (off) *off = g->g->off.data();
    if (col) *col = g->g->col.data();
    if (w) *w = g->g->weighted() ? g->g->w.data() : nullptr;
  });
}

void mg_graph_destroy(mg_graph* g) { delete g; }

int mg_graph_rmat_hashed(int scale, int ef, uint64_t seed, int threads, mg_graph** out) {
  return wrap([&] { *out = box(rmat_hashed(scale, ef, seed, threads)); });
}

int mg_partition_random(uint32_t nv, uint32_t n, uint64_t seed, uint32_t* owner) {
  return wrap([&] {
    auto o = partition_random(nv, n, seed);
    std::memcpy(owner, o.data(), o.size() * 4);
  });
}

int mg_partition_biased_random(const mg_graph* g, uint32_t n, uint64_t seed, double bias,
                               uint32_t* owner) {
  return wrap([&] {
    auto o = partition_biased(*g->g, n, seed, bias);
    std::memcpy(owner, o.data(), o.size() * 4);
  });
}

int mg_plan_create(const mg_graph* g, const uint32_t* owner, uint32_t n, int dup,
                   const int* devices, mg_plan** out) {
  return wrap([&] {
    if (!g) throw Error(MG_EINVAL, "mg_plan_create: null graph");
    if (dup != MG_DUP_ALL && dup != MG_DUP_ONEHOP)
      throw Error(MG_EINVAL, "mg_plan_create: unknown duplication mode");
    std::vector<uint32_t> own(g->g->nv, 0);
    if (owner) own.assign(owner, owner + g->g->nv);
    else if (n != 1) throw Error(MG_EINVAL, "mg_plan_create: owner map required for n > 1");
    HostPlan H = build_plan(*g->g, own, n, dup);
    *out = reinterpret_cast<mg_plan*>(plan_from_host(H, devices, g->g, -1));
  });
}

void mg_plan_destroy(mg_plan* p) { plan_free(reinterpret_cast<Plan*>(p)); }

int mg_plan_info(const mg_plan* p, uint32_t* nv, uint64_t* ne, uint32_t* n) {
  return wrap([&] {
    Plan& P = plan_of(p);
    if (nv) *nv = P.nv;
    if (ne) *ne = P.ne;
    if (n) *n = P.n;
  });
}

// BorderMetrics (partition.cpp:211-242)
int mg_plan_border_metrics(const mg_plan* p, uint64_t* pair, uint64_t* cut) {
  return wrap([&] {
    Plan& P = plan_of(p);
    if (pair)
      for (uint32_t i = 0; i < P.n; ++i)
        for (uint32_t j = 0; j < P.n; ++j) pair[i * P.n + j] = P.pair_border[i][j];
    if (cut && !P.host_graph) {  // device-built plan: count on the GPU
      *cut = device_edge_cut(P);
      return;
    }
    if (cut) {
      const HostCsr& g = *P.host_graph;
      uint64_t c = 0;  // undirected edges {u,v} with different owners, counted once
      for (uint32_t u = 0; u < g.nv; ++u)
        for (uint32_t e = g.off[u]; e < g.off[u + 1]; ++e) {
          uint32_t v = g.col[e];
          if (P.owner_host[u] == P.owner_host[v]) continue;
          // count the pair once: from its smaller endpoint, or from u when the
          // reverse arc is absent (directed input)
          bool rev = false;
          if (v > u) {
            c++;
            continue;
          }
          for (uint32_t f = g.off[v]; f < g.off[v + 1]; ++f)
            if (g.col[f] == u) {
              rev = true;
              break;
            }
          if (!rev) c++;
        }
      *cut = c;
    }
  });
}

int mg_plan_download_graph(const mg_plan* p, mg_graph** out) {
  return wrap([&] {
    Plan& P = plan_of(p);
    if (P.host_graph) {
      *out = new mg_graph{P.host_graph};
      return;
    }
    // n == 1 device plans: worker 0's sub-CSR is the global CSR
    const bool single = !P.g_off.ptr && P.n == 1 && P.workers[0];
    if (!P.g_off.ptr && !single) throw Error(MG_EINVAL, "plan holds no global graph");
    const uint32_t* d_off = single ? P.workers[0]->off.ptr : P.g_off.ptr;
    const uint32_t* d_col = single ? P.workers[0]->col.ptr : P.g_col.ptr;
    const uint32_t* d_w = single ? P.workers[0]->w.ptr : P.g_w.ptr;
    HostCsr g;
    g.nv = P.nv;
    g.off.resize((size_t)P.nv + 1);
    g.col.resize(P.ne);
    DeviceGuard dg(P.devices[0]);
    MGB_CUDA(cudaMemcpy(g.off.data(), d_off, 4ull * (P.nv + 1), cudaMemcpyDeviceToHost));
    MGB_CUDA(cudaMemcpy(g.col.data(), d_col, 4ull * P.ne, cudaMemcpyDeviceToHost));
    if (d_w) {
      g.w.resize(P.ne);
      MGB_CUDA(cudaMemcpy(g.w.data(), d_w, 4ull * P.ne, cudaMemcpyDeviceToHost));
    }
    *out = box(std::move(g));
  });
}

int mg_plan_last_d2h_bytes(const mg_plan* p, uint64_t* bytes) {
  return wrap([&] { *bytes = plan_of(p).last_d2h_bytes; });
}

int mg_plan_set_profiling(mg_plan* p, int enable) {
  return wrap([&] { plan_of(p).profile = enable != 0; });
}

int mg_plan_last_array(const mg_plan* p, int which, uint64_t* buf, uint64_t cap, uint64_t* len) {
  return wrap([&] {
    Plan& P = plan_of(p);
    std::vector<uint64_t> flat;
    switch (which) {
      case MG_ARR_H_MATRIX:
        for (auto& r : P.h_matrix) flat.insert(flat.end(), r.begin(), r.end());
        break;
      case MG_ARR_H_PER_ITER:
        for (auto& r : P.h_per_iter) flat.insert(flat.end(), r.begin(), r.end());
        break;
      case MG_ARR_OUT_PER_ITER: flat = P.out_per_iter; break;
      case MG_ARR_EDGES_PER_ITER: flat = P.edges_per_iter; break;
      case MG_ARR_COMBINE_PER_ITER: flat = P.combine_per_iter; break;
      case MG_ARR_DIRECTION_LOG: flat.assign(P.last_dir_log.begin(), P.last_dir_log.end()); break;
      default: throw Error(MG_EINVAL, "mg_plan_last_array: unknown array");
    }
    if (len) *len = flat.size();
    for (uint64_t i = 0; buf && i < flat.size() && i < cap; ++i) buf[i] = flat[i];
  });
}

int mg_plan_last_buffer_stats(const mg_plan* p, uint32_t worker, int role, uint64_t* reallocs,
                              uint64_t* peak_items, uint64_t* peak_bytes) {
  return wrap([&] {
    Plan& P = plan_of(p);
    if (worker >= P.last_buffers.size() || role < 0 || role >= MG_NUM_ROLES)
      throw Error(MG_EINVAL, "mg_plan_last_buffer_stats: out of range");
    const BufferStats& b = P.last_buffers[worker][role];
    if (reallocs) *reallocs = b.realloc_count;
    if (peak_items) *peak_items = b.peak_items;
    if (peak_bytes) *peak_bytes = b.peak_bytes;
  });
}

}  // extern "C"
