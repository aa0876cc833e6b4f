// Operator-API test: user-defined primitives written against
// include/mgraph_b200_spec.cuh (PrimitiveSpec + run_primitive, the reference's
// engine.hpp:587-626,712) and compiled with nvcc, as a reference user would.
//
//   worker_failure   test_engine.cpp:272-287 — a hook throwing on worker 1
//                    aborts the run with the same exception; the plan stays
//                    usable
//   microbench       cost_model.cpp:76-112 — one self-loop vertex per worker,
//                    pipeline(in, accept-all, 1) until S supersteps: the
//                    per-superstep latency l of the BSP cost model
//   assoc8           a BFS-shaped spec shipping 8 vertex + 8 value associates
//                    per record (engine.hpp:645-646): labels equal the built-in
//                    bfs, every received associate checked on the device, H
//                    equal to the built-in bfs's
//   labelprop        a broadcast-mode spec (min-label propagation with a keep
//                    stamp, combine = min): components equal the built-in cc
// Built and run by tests/test_operator_api.py.
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "mgraph_b200_spec.cuh"

namespace mg = mgraph_b200;
using namespace mg;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                               \
  do {                                                            \
    if (cond) {                                                   \
      ++g_pass;                                                   \
    } else {                                                      \
      ++g_fail;                                                   \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                             \
  } while (0)

static Assignment assign(std::vector<uint32_t> o, uint32_t n) {
  Assignment a;
  a.owner = std::move(o);
  a.num_partitions = n;
  return a;
}

// ---------------------------------------------------------------- worker failure
struct NoDev {
  __device__ bool combine(uint32_t, const uint32_t*, const double*, uint32_t) const {
    return false;
  }
};

static void worker_failure() {
  PartitionPlan plan = build_partition_plan(Csr::path(4), assign({0, 0, 1, 1}, 2),
                                            Duplication::All);
  PrimitiveSpec<int, NoDev> spec;
  spec.name = "boom";
  spec.init = [](int&, WorkerHandle& h) {
    if (h.worker() == 1) throw std::runtime_error("worker 1 failed");
    h.push_initial(0);
  };
  spec.iteration_body = [](int&, WorkerHandle&, const Frontier&, Frontier&) {};
  spec.device = [](int&, WorkerHandle&) { return NoDev{}; };
  bool ok = false;
  try {
    (void)run_primitive(spec, plan, EngineConfig{});
  } catch (const std::runtime_error& e) {
    ok = std::string(e.what()) == "worker 1 failed";
  }
  CHECK(ok);
  // the same plan serves the next call (test_engine.cpp:289-295 trace)
  BfsResult r = bfs(plan, {.source = 0});
  CHECK(r.labels == (std::vector<Label>{0, 1, 2, 3}));
  CHECK(r.stats.supersteps == 4 && r.stats.h_total() == 2);
  // the engine validates the spec like the reference (E:716-730)
  PrimitiveSpec<int, NoDev> bad = spec;
  bad.init = nullptr;
  bad.num_vertex_associates = 9;
  bool inv = false;
  try {
    (void)run_primitive(bad, plan, EngineConfig{});
  } catch (const std::invalid_argument&) {
    inv = true;
  }
  CHECK(inv);
  PrimitiveSpec<int, NoDev> fixed = spec;
  fixed.init = nullptr;
  fixed.communication = CommMode::Broadcast;
  EngineConfig cfg;
  cfg.comm_override = CommMode::Selective;
  inv = false;
  try {
    (void)run_primitive(fixed, plan, cfg);
  } catch (const std::invalid_argument&) {
    inv = true;
  }
  CHECK(inv);
}

// ---------------------------------------------------------------- microbench
struct NopDev {
  __device__ bool visit(uint32_t, uint32_t, uint32_t) const { return true; }
  __device__ bool keep(uint32_t) const { return true; }
  __device__ bool combine(uint32_t, const uint32_t*, const double*, uint32_t) const {
    return false;
  }
};
struct NopState {};

static void microbench(uint32_t n_workers, uint64_t supersteps) {
  EdgeList edges;
  for (VertexId v = 0; v < n_workers; ++v) edges.push_back({v, v, 0});
  std::vector<uint32_t> own(n_workers);
  for (VertexId v = 0; v < n_workers; ++v) own[v] = v;
  PartitionPlan plan = build_partition_plan(Csr::build(edges, n_workers),
                                            assign(own, n_workers), Duplication::All);
  PrimitiveSpec<NopState, NopDev> spec;
  spec.name = "microbench";
  spec.communication = CommMode::Selective;
  spec.init = [](NopState&, WorkerHandle& h) { h.push_initial(h.worker()); };
  spec.iteration_body = [](NopState&, WorkerHandle& h, const Frontier& in, Frontier&) {
    h.pipeline(in, NopDev{}, 1);
  };
  spec.device = [](NopState&, WorkerHandle&) { return NopDev{}; };
  spec.stop_condition = [supersteps](const GlobalView& v) {
    return v.iteration + 1 >= supersteps;
  };
  (void)run_primitive(spec, plan, EngineConfig{});  // warm
  auto rr = run_primitive(spec, plan, EngineConfig{});
  CHECK(rr.stats.supersteps == supersteps);
  CHECK(rr.stats.edges_examined == supersteps * n_workers);  // one self-loop per worker
  CHECK(rr.stats.h_total() == 0);
  std::printf("microbench workers=%u supersteps=%llu per_iter_us=%.2f device_ms=%.3f\n",
              n_workers, (unsigned long long)rr.stats.supersteps,
              rr.stats.wall_ms * 1000.0 / (double)rr.stats.supersteps, rr.stats.device_ms);
}

// ---------------------------------------------------------------- 8 associates
__device__ __forceinline__ uint32_t tag(uint32_t v, int k) { return v * 2654435761u + 97u * k; }

struct Assoc8Dev {
  uint32_t* labels;
  uint32_t* stamp;
  uint32_t* bad;
  OwnerView ow;
  uint32_t iter;
  __device__ bool prefilter(uint32_t v) const { return labels[v] == kInfLabel; }
  __device__ bool visit(uint32_t, uint32_t v, uint32_t) const {
    return atomicCAS(&labels[v], kInfLabel, iter + 1) == kInfLabel;
  }
  __device__ bool keep(uint32_t v) const { return atomicExch(&stamp[v], iter + 1) != iter + 1; }
  __device__ void gather(uint32_t v, uint32_t* va, double* vv) const {
    for (int k = 0; k < 8; ++k) {
      va[k] = tag(v, k);
      vv[k] = (double)labels[v] + 0.25 * k;
    }
  }
  __device__ bool combine(uint32_t v, const uint32_t* va, const double* vv, uint32_t it) const {
    for (int k = 0; k < 8; ++k)
      if (va[k] != tag(v, k) || vv[k] != (double)(it + 1) + 0.25 * k) atomicAdd(bad, 1u);
    uint32_t cand = it + 1;
    return cand < atomicMin(&labels[v], cand) && ow.hosts(v);
  }
};
struct Assoc8State {
  DeviceArray<uint32_t> labels, stamp, bad;
};

static void assoc8(uint32_t n) {
  Csr g = Csr::rmat(12, 16, 1);
  Assignment a = partition_random(g.num_vertices(), n, 7);
  PartitionPlan plan = build_partition_plan(g, a, Duplication::All);
  const VertexId src = 0;
  PrimitiveSpec<Assoc8State, Assoc8Dev> spec;
  spec.name = "bfs8";
  spec.num_vertex_associates = 8;
  spec.num_value_associates = 8;
  spec.init = [&](Assoc8State& s, WorkerHandle& h) {
    const uint32_t nv = h.num_local_vertices();
    s.labels.resize(nv);
    s.stamp.resize(nv);
    s.bad.resize(1);
    cudaMemsetAsync(s.labels.data(), 0xFF, 4ull * nv, h.stream());
    cudaMemsetAsync(s.stamp.data(), 0, 4ull * nv, h.stream());
    cudaMemsetAsync(s.bad.data(), 0, 4, h.stream());
    const uint32_t zero = 0;
    cudaMemcpyAsync(s.labels.data() + src, &zero, 4, cudaMemcpyHostToDevice, h.stream());
    cudaStreamSynchronize(h.stream());
    if (h.hosts_local(src)) h.push_initial(src);
  };
  spec.device = [](Assoc8State& s, WorkerHandle& h) {
    return Assoc8Dev{s.labels.data(), s.stamp.data(), s.bad.data(), h.owner_view(),
                     (uint32_t)h.iteration()};
  };
  spec.iteration_body = [&](Assoc8State& s, WorkerHandle& h, const Frontier& in, Frontier&) {
    h.pipeline(in, spec.device(s, h), h.num_local_vertices());
  };
  auto rr = run_primitive(spec, plan, EngineConfig{});
  BfsResult want = bfs(plan, {.source = src});
  std::vector<Label> got(g.num_vertices(), kInfLabel);
  uint32_t bad = 0;
  for (uint32_t p = 0; p < n; ++p) {
    auto lab = rr.states[p].labels.to_host();
    for (VertexId v = 0; v < g.num_vertices(); ++v)
      if (a.owner[v] == p) got[v] = lab[v];
    bad += rr.states[p].bad.to_host()[0];
  }
  CHECK(got == want.labels);
  CHECK(bad == 0);
  CHECK(rr.stats.supersteps == want.stats.supersteps);
  CHECK(rr.stats.h_matrix == want.stats.h_matrix);
  CHECK(rr.stats.edges_examined == want.stats.edges_examined);
}

// ---------------------------------------------------------------- label propagation
struct LpDev {
  uint32_t* comp;
  uint32_t* stamp;
  uint32_t iter;
  __device__ bool visit(uint32_t u, uint32_t v, uint32_t) const {
    const uint32_t c = comp[u];
    return c < atomicMin(&comp[v], c);
  }
  __device__ bool keep(uint32_t v) const { return atomicExch(&stamp[v], iter + 1) != iter + 1; }
  __device__ void gather(uint32_t v, uint32_t* va, double*) const { va[0] = comp[v]; }
  __device__ bool combine(uint32_t v, const uint32_t* va, const double*, uint32_t) const {
    return va[0] < atomicMin(&comp[v], va[0]);
  }
};
struct LpState {
  DeviceArray<uint32_t> comp, stamp;
};
__global__ void iota_k(uint32_t* a, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[i] = i;
}

static void labelprop(uint32_t n) {
  Csr g = Csr::rmat(11, 4, 3);  // several components
  Assignment a = partition_random(g.num_vertices(), n, 5);
  PartitionPlan plan = build_partition_plan(g, a, Duplication::All);
  PrimitiveSpec<LpState, LpDev> spec;
  spec.name = "labelprop";
  spec.num_vertex_associates = 1;
  spec.communication = CommMode::Broadcast;
  spec.init = [](LpState& s, WorkerHandle& h) {
    const uint32_t nv = h.num_local_vertices();
    s.comp.resize(nv);
    s.stamp.resize(nv);
    iota_k<<<64, 256, 0, h.stream()>>>(s.comp.data(), nv);
    cudaMemsetAsync(s.stamp.data(), 0, 4ull * nv, h.stream());
    for (VertexId v : h.hosted_local()) h.push_initial(v);
  };
  spec.device = [](LpState& s, WorkerHandle& h) {
    return LpDev{s.comp.data(), s.stamp.data(), (uint32_t)h.iteration()};
  };
  spec.iteration_body = [&](LpState& s, WorkerHandle& h, const Frontier& in, Frontier&) {
    h.pipeline(in, spec.device(s, h), h.num_local_vertices());
  };
  auto rr = run_primitive(spec, plan, EngineConfig{});
  CcResult want = cc(plan);
  std::vector<VertexId> got(g.num_vertices());
  for (uint32_t p = 0; p < n; ++p) {
    auto c = rr.states[p].comp.to_host();
    for (VertexId v = 0; v < g.num_vertices(); ++v)
      if (a.owner[v] == p) got[v] = c[v];
  }
  CHECK(got == want.components);
  CHECK(rr.stats.communication == "broadcast");
}

int main(int argc, char** argv) {
  const bool bench_only = argc > 1 && std::strcmp(argv[1], "--microbench") == 0;
  if (!bench_only) {
    worker_failure();
    for (uint32_t n : {1u, 2u, 4u}) assoc8(n);
    for (uint32_t n : {1u, 3u}) labelprop(n);
  }
  for (uint32_t n : {1u, 2u, 4u}) microbench(n, 200);
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
