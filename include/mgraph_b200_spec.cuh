// mgraph_b200_spec.cuh — the reference's operator API for user-defined
// primitives: PrimitiveSpec<State> + run_primitive (engine.hpp:587-626, :712),
// WorkerHandle services (engine.hpp:478-582), GlobalView / WorkerReport
// (engine.hpp:216-253), compiled with nvcc against the engine templates.
//
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
//        -I<repo>/include -I<repo>/paper_1504_04804_b200/csrc my_primitive.cu \
//        -L<repo>/paper_1504_04804_b200 -lmgraph_b200 -Xlinker -rpath=<repo>/paper_1504_04804_b200
//
// The contract is the reference's, split along the host/device line:
//
//   host hooks — std::function members, as in the reference, run by the host
//   thread that drives the worker and launching device work through the
//   WorkerHandle:   init, iteration_body, comm_selector, stop_condition,
//                   finalize, plus `device` (below);
//   device hooks — members of a functor set `Dev` that the spec's `device`
//   hook returns for every superstep; it is copied by value into the sm_100a
//   kernels (advance / filter / split+pack / merge):
//       __device__ bool combine(VertexId v, const VertexId* va, const Value* vv,
//                               uint32_t iteration) const;            required
//       __device__ void gather(VertexId v, VertexId* va, Value* vv) const;   opt.
//       __device__ bool send_filter(uint32_t peer, VertexId v) const;       opt.
//       __device__ bool visit(VertexId u, VertexId v, EdgeId e) const;      opt.
//       __device__ bool keep(VertexId v) const;                             opt.
//       __device__ bool prefilter(VertexId v) const;  (cheap read-only pre-test
//                                                       of visit; opt.)
//   Missing optional hooks take the reference's defaults (no associates, send
//   everything, accept every arc / vertex).  combine must be commutative and
//   associative over receipt order (records of one superstep merge in
//   parallel); its return value decides enqueueing, deduplicated per superstep
//   by the engine's merge stamp (engine.hpp:823-852).
//
// State is a host-side struct per worker (device arrays it allocates in init
// are its own; DeviceArray<T> below frees them with the state).  Up to 8
// vertex and 8 value associates per record (engine.hpp:645-646).  An exception
// thrown by any host hook on any worker stops the run and propagates unchanged
// (E:773-782); engine errors map to std::invalid_argument / CapacityError /
// std::runtime_error as in the reference.
//
// B200 notes: user primitives run on Duplicate-All plans (local ID = global
// ID); a superstep may ship each vertex to a peer at most once (dedup in keep,
// as every reference spec does) — the inbox holds |V_src| records per source.
#pragma once

#include <functional>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "engine.cuh"
#include "mgraph_b200.hpp"

namespace mgraph_b200 {

using mgb::GlobalView;
using mgb::GraphView;
using mgb::OwnerView;
using mgb::WorkerReport;
constexpr int kMaxAssociates = mgb::kMaxAssoc;

// owned device array for primitive state (freed with the State that holds it)
template <class T>
class DeviceArray {
 public:
  DeviceArray() = default;
  explicit DeviceArray(uint64_t n) { resize(n); }
  DeviceArray(DeviceArray&& o) noexcept { *this = std::move(o); }
  DeviceArray& operator=(DeviceArray&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  DeviceArray(const DeviceArray&) = delete;
  ~DeviceArray() {
    if (p_) cudaFree(p_);
  }
  void resize(uint64_t n) {
    if (n == n_) return;
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = n;
    if (n) MGB_CUDA(cudaMalloc(&p_, n * sizeof(T)));
  }
  T* data() const { return p_; }
  uint64_t size() const { return n_; }
  std::vector<T> to_host() const {
    std::vector<T> h(n_);
    if (n_) MGB_CUDA(cudaMemcpy(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost));
    return h;
  }

 private:
  T* p_ = nullptr;
  uint64_t n_ = 0;
};

// a frontier as the body sees it: device IDs + length (input), or the output
// buffer + its device-side length counter
struct Frontier {
  VertexId* data = nullptr;   // device pointer
  uint32_t size = 0;          // input: host-known length
  uint32_t* device_count = nullptr;  // output: appended length lives on the device
};

namespace detail {

template <class D, class = void>
struct has_visit : std::false_type {};
template <class D>
struct has_visit<D, std::void_t<decltype(std::declval<const D&>().visit(0u, 0u, 0u))>>
    : std::true_type {};
template <class D, class = void>
struct has_keep : std::false_type {};
template <class D>
struct has_keep<D, std::void_t<decltype(std::declval<const D&>().keep(0u))>> : std::true_type {};
template <class D, class = void>
struct has_prefilter : std::false_type {};
template <class D>
struct has_prefilter<D, std::void_t<decltype(std::declval<const D&>().prefilter(0u))>>
    : std::true_type {};
template <class D, class = void>
struct has_gather : std::false_type {};
template <class D>
struct has_gather<D, std::void_t<decltype(std::declval<const D&>().gather(
                         0u, (VertexId*)nullptr, (Value*)nullptr))>> : std::true_type {};
template <class D, class = void>
struct has_send_filter : std::false_type {};
template <class D>
struct has_send_filter<D, std::void_t<decltype(std::declval<const D&>().send_filter(0u, 0u))>>
    : std::true_type {};

// the user's functor set in the shape the engine kernels call (operators.cuh,
// engine.cuh), with the reference's defaults for the optional hooks
template <class Dev>
struct DevAdapter {
  static constexpr int kAssocCap = mgb::kMaxAssoc;
  Dev d;
  __device__ __forceinline__ bool visit(uint32_t u, uint32_t v, uint32_t e) const {
    if constexpr (has_visit<Dev>::value) return d.visit(u, v, e);
    else return true;
  }
  __device__ __forceinline__ bool keep(uint32_t v) const {
    if constexpr (has_keep<Dev>::value) return d.keep(v);
    else return true;
  }
  __device__ __forceinline__ bool prefilter(uint32_t v) const {
    if constexpr (has_prefilter<Dev>::value) return d.prefilter(v);
    else return true;
  }
  __device__ __forceinline__ bool combine(uint32_t v, const uint32_t* va, const double* vv,
                                          uint32_t it) const {
    return d.combine(v, va, vv, it);
  }
  __device__ __forceinline__ void gather(uint32_t v, uint32_t* va, double* vv) const {
    if constexpr (has_gather<Dev>::value) d.gather(v, va, vv);
  }
  __device__ __forceinline__ bool send_filter(uint32_t q, uint32_t v) const {
    if constexpr (has_send_filter<Dev>::value) return d.send_filter(q, v);
    else return true;
  }
  __device__ __forceinline__ uint32_t peer_id(uint32_t v, uint32_t, uint32_t) const {
    return v;  // Duplicate-All: local ID = global ID on every worker
  }
};

static __global__ void spec_add_u64_kernel(unsigned long long* dst, unsigned long long v) {
  *dst += v;
}

}  // namespace detail

// WorkerHandle (engine.hpp:478-582): one worker's view inside the hooks
class WorkerHandle {
 public:
  explicit WorkerHandle(mgb::Ctx& c) : c_(c) {}

  uint32_t worker() const { return c_.w->p; }
  uint32_t num_workers() const { return c_.P->n; }
  uint64_t iteration() const { return c_.iter; }
  bool fused_traversal() const { return c_.fused; }
  VertexId num_local_vertices() const { return c_.w->nv; }
  VertexId local_count() const { return static_cast<VertexId>(c_.w->hosted_host.size()); }
  // hosted vertices as local IDs: host copy, and the device array
  const std::vector<VertexId>& hosted_local() const { return c_.w->hosted_host; }
  const VertexId* hosted_local_device() const { return c_.w->hosted.ptr; }
  VertexId to_global(VertexId local) const { return local; }
  VertexId to_local(VertexId global) const { return global; }
  uint32_t owner_of_global(VertexId global) const { return c_.P->owner_host[global]; }
  bool hosts_local(VertexId local) const { return c_.P->owner_host[local] == c_.w->p; }

  // device-side views for the user's kernels / functors
  cudaStream_t stream() const { return c_.w->stream; }
  GraphView subgraph() const { return c_.graph(); }
  OwnerView owner_view() const { return c_.owner_view(); }

  // seed the initial frontier (valid inside init only)
  void push_initial(VertexId local) { c_.push_initial({local}); }

  // operators over the superstep's input frontier (E:516-541); the results
  // land in the worker's advance / output buffers like the reference's
  // advance_out / output frontiers.  `in` must be the body's input frontier.
  template <class Dev>
  void run_advance(const Frontier& in, const Dev& d) {
    check_input(in);
    mgb::Worker& w = *c_.w;
    w.advance_out.ensure(c_.degsum(), w.stream);
    c_.run_advance(detail::DevAdapter<Dev>{d}, w.advance_out.ptr, &c_.ctr()->adv_cnt);
  }
  // filter the advance output into the output frontier (order-free compaction)
  template <class Dev>
  void run_filter(const Dev& d) {
    mgb::Worker& w = *c_.w;
    uint32_t adv = 0;
    MGB_CUDA(cudaMemcpyAsync(&adv, &c_.ctr()->adv_cnt, 4, cudaMemcpyDeviceToHost, w.stream));
    MGB_CUDA(cudaStreamSynchronize(w.stream));
    c_.ensure_output(adv < w.nv ? adv : w.nv);
    if (adv == 0) return;
    MGB_LAUNCH(mgb::filter_kernel<detail::DevAdapter<Dev>>, mgb::grid_for(adv, 256), 256, 0,
               w.stream, detail::DevAdapter<Dev>{d}, w.advance_out.ptr, &c_.ctr()->adv_cnt,
               w.output.ptr, &c_.ctr()->out_cnt);
  }
  // fused or two-stage traversal per the active policy (E:528-541);
  // dedup_bound caps the output when keep() deduplicates
  template <class Dev>
  void pipeline(const Frontier& in, const Dev& d, uint64_t dedup_bound) {
    check_input(in);
    c_.pipeline(detail::DevAdapter<Dev>{d}, dedup_bound);
  }
  // a body with its own kernels: room for `capacity` output vertices; append
  // through out.device_count (atomicAdd) — the engine reads the length there
  Frontier reserve_output(uint64_t capacity) {
    c_.ensure_output(capacity);
    return {c_.w->output.ptr, 0, &c_.ctr()->out_cnt};
  }

  const GlobalView* previous_view() const { return c_.prev; }
  WorkerReport& report() { return c_.report; }
  void count_edges(uint64_t k) {
    if (k) MGB_LAUNCH(detail::spec_add_u64_kernel, 1, 1, 0, c_.w->stream, &c_.ctr()->edges, k);
  }

 private:
  void check_input(const Frontier& in) const {
    if (in.data != c_.w->input.ptr || in.size != c_.in_count)
      throw std::invalid_argument("operators run on the superstep's input frontier");
  }
  mgb::Ctx& c_;
};

// PrimitiveSpec (engine.hpp:587-626); Dev = the device functor set
template <class State, class Dev>
struct PrimitiveSpec {
  std::string name;
  int num_vertex_associates = 0;  // per-vertex IDs shipped (predecessors etc.), <= 8
  int num_value_associates = 0;   // per-vertex scalars shipped, <= 8
  CommMode communication = CommMode::Selective;
  bool allow_comm_override = false;
  std::optional<Duplication> duplication_required = Duplication::All;

  // seed state and the initial frontier
  std::function<void(State&, WorkerHandle&)> init;
  // one superstep of local computation: consume `in`, emit into the output
  // (through h.pipeline / h.run_advance + h.run_filter / h.reserve_output)
  std::function<void(State&, WorkerHandle&, const Frontier& in, Frontier& out)> iteration_body;
  // the device hooks for this superstep (combine, gather, send_filter, ...)
  std::function<Dev(State&, WorkerHandle&)> device;
  // per-superstep routing override, evaluated after the body
  std::function<CommMode(const State&, const WorkerHandle&)> comm_selector;
  // custom stop rule at the barrier; default: every frontier empty
  std::function<bool(const GlobalView&)> stop_condition;
  // after the loop, with the final view
  std::function<void(State&, WorkerHandle&, const GlobalView&)> finalize;
};

template <class State>
struct RunResult {
  std::vector<State> states;  // per worker (local workers only in multi-process plans)
  RunStats stats;
};

namespace detail {

// the spec in the shape of the engine's primitive hooks (engine.cuh)
template <class State, class Dev>
struct SpecPrim {
  const PrimitiveSpec<State, Dev>& spec;
  std::vector<State>& states;
  const char* name;
  int nva, nvv, communication;
  bool allow_comm_override;
  int dup_required;
  bool has_stop_condition;
  bool reports_deg = false;

  SpecPrim(const PrimitiveSpec<State, Dev>& s, std::vector<State>& st)
      : spec(s), states(st), name(s.name.c_str()), nva(s.num_vertex_associates),
        nvv(s.num_value_associates),
        communication(s.communication == CommMode::Broadcast ? MG_COMM_BROADCAST
                                                             : MG_COMM_SELECTIVE),
        allow_comm_override(s.allow_comm_override),
        dup_required(!s.duplication_required ? -1
                     : *s.duplication_required == Duplication::All ? MG_DUP_ALL
                                                                   : MG_DUP_ONEHOP),
        has_stop_condition(static_cast<bool>(s.stop_condition)) {}

  uint64_t inbox_bound(mgb::Plan& P, uint32_t src, uint32_t, int) const {
    return P.workers[src] ? P.workers[src]->nv : P.nv;
  }
  void init(mgb::Ctx& c) {
    WorkerHandle h(c);
    if (spec.init) spec.init(states[c.w->p], h);
  }
  void body(mgb::Ctx& c) {
    WorkerHandle h(c);
    Frontier in{c.w->input.ptr, c.in_count, nullptr};
    Frontier out = h.reserve_output(0);
    spec.iteration_body(states[c.w->p], h, in, out);
  }
  int comm_selector(mgb::Ctx& c, int comm) {
    if (!spec.comm_selector) return comm;
    WorkerHandle h(c);
    return spec.comm_selector(states[c.w->p], h) == CommMode::Broadcast ? MG_COMM_BROADCAST
                                                                       : MG_COMM_SELECTIVE;
  }
  void after_merge(mgb::Ctx&) {}
  mgb::DenseView dense_view(mgb::Ctx&) const { return {}; }  // records only
  bool stop_condition(const GlobalView& v) { return spec.stop_condition(v); }
  void finalize(mgb::Ctx& c, const GlobalView& v) {
    if (!spec.finalize) return;
    WorkerHandle h(c);
    spec.finalize(states[c.w->p], h, v);
  }
  DevAdapter<Dev> dev(mgb::Ctx& c) {
    WorkerHandle h(c);
    return {spec.device(states[c.w->p], h)};
  }
};

}  // namespace detail

// run_primitive (engine.hpp:712-981) for a user spec on an uploaded plan
template <class State, class Dev>
RunResult<State> run_primitive(const PrimitiveSpec<State, Dev>& spec, const PartitionPlan& plan,
                               const EngineConfig& cfg = EngineConfig{}) {
  if (!spec.iteration_body || !spec.device || !plan.handle())
    throw std::invalid_argument(spec.name + ": iteration_body and device hooks are required");
  mgb::Plan& P = *reinterpret_cast<mgb::Plan*>(plan.handle());
  if (P.dup != MG_DUP_ALL)
    throw std::invalid_argument(spec.name + ": user primitives need a Duplicate-All plan");
  RunResult<State> rr;
  rr.states.resize(P.n);
  detail::SpecPrim<State, Dev> prim(spec, rr.states);
  const mg_config c = cfg.to_c();
  P.last = mg_stats{};
  try {
    mgb::run_primitive(P, prim, c);
  } catch (const mgb::Error& e) {  // engine errors -> the reference's exception types
    if (e.code == MG_EINVAL) throw std::invalid_argument(e.what());
    if (e.code == MG_ECAPACITY) throw CapacityError(e.what());
    throw std::runtime_error(e.what());
  }
  rr.stats = detail::stats(plan.handle(), P.last);
  return rr;
}

}  // namespace mgraph_b200
