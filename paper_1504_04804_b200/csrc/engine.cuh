// engine.cuh — the BSP superstep engine on B200 (reference run_primitive,
// engine.hpp:712-981) as a host C++ enactor driving sm_100a kernels.
//
// Per superstep, for every worker (partition) p:
//   body        primitive kernels (advance/filter/compute) -> output        (E:874-875)
//   split+pack  one kernel: owner(v)==p -> next_input, else the record (id +
//               gathered associates) is stored straight into the destination
//               worker's inbox slot [parity][p] — a peer-HBM store over NVLink
//               when the destination is another GPU                        (E:877-915)
//   publish     per-destination record counts written into the peer's slot
//               counters; an event orders them before the peer's merge      (E:361-391)
//   merge       combine() every received record, enqueue once via the merge
//               stamp                                                        (E:823-852)
//   report      one D2H of the worker counters; the host reduces the
//               WorkerReports into a GlobalView and applies the stop rule   (E:784-820)
// Only the final report needs a host round trip: pack->merge ordering across
// workers uses CUDA events (cudaStreamWaitEvent), not a host barrier.
#pragma once

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <optional>
#include <type_traits>

#include "operators.cuh"

namespace mgb {

struct WorkerReport {  // engine.hpp:216-223
  uint64_t out_frontier = 0, next_frontier = 0, edges_delta = 0, combine_delta = 0;
  double f[4] = {0, 0, 0, 0};
  uint64_t u[4] = {0, 0, 0, 0};
};

struct GlobalView {  // engine.hpp:225-253
  uint32_t iteration = 0, num_workers = 1;
  std::vector<WorkerReport> reports;
  uint64_t total_out = 0, total_next = 0, inflight_records = 0;
  double sum_f(int k) const {
    double s = 0;
    for (auto& r : reports) s += r.f[k];
    return s;
  }
  double max_f(int k) const {
    double s = 0;
    for (auto& r : reports) s = s > r.f[k] ? s : r.f[k];
    return s;
  }
  uint64_t max_u(int k) const {
    uint64_t s = 0;
    for (auto& r : reports) s = s > r.u[k] ? s : r.u[k];
    return s;
  }
  bool all_u_equal(int k, uint64_t v) const {
    for (auto& r : reports)
      if (r.u[k] != v) return false;
    return true;
  }
};

// multi-process report all-gather (fabric.cu)
void fabric_exchange_reports(Plan& P, const WorkerReport& r, const Counters& c,
                             std::vector<WorkerReport>& reports,
                             std::vector<std::vector<uint32_t>>& sends, bool& overflow);

// Associates a functor set may ship per record: the slot tables hold
// kMaxAssoc (8, as the reference's fixed arrays, engine.hpp:645-646); the
// per-thread staging in split/merge is sized by the functor's kAssocCap
// (default 2, what the built-in primitives need) so their registers do not pay
// for the general case.
template <class F, class = void>
struct AssocCap {
  static constexpr int value = 2;
};
template <class F>
struct AssocCap<F, std::void_t<decltype(F::kAssocCap)>> {
  static constexpr int value = F::kAssocCap;
};

// ---------------------------------------------------------------------------
// Dense exchange (broadcast primitives).  A broadcast superstep ships every
// output vertex to every peer (E:880-890).  When a worker's output is large,
// the same information is smaller as a dense array over its local ID space:
//   kind 1  DOBFS: the discovery bitmap vis & ~vis_prev (|V|/8 bytes instead of
//           4 bytes per record once the output holds >= |V|/32 vertices);
//   kind 2  CC: the whole comp[] array (4 B/vertex instead of 8 B/record once
//           more than half the vertices changed) — with min-combine this is an
//           all-gather + local MIN reduction, and vertices outside the sender's
//           delta are no-ops at the receiver (their value was broadcast before).
// The sender decides on the device from its output length; the slot count
// carries kDenseFlag, so each receiver merges each source in the format it was
// sent.  H, C and wire records are counted in records, as the reference does.
constexpr uint32_t kDenseFlag = 0x80000000u;

struct DenseView {
  int kind = 0;                      // 0: records only, 1: bitmap, 2: u32 values
  const uint32_t* cur = nullptr;     // 1: visited bitmap now; 2: the value array
  const uint32_t* prev = nullptr;    // 1: visited bitmap before this superstep's body
  uint32_t* vis = nullptr;           // 1: the receiver's visited bitmap (merge pre-test)
  uint32_t words = 0;                // bitmap words / values
  uint32_t threshold = 0xFFFFFFFFu;  // dense once the output holds >= threshold vertices
};

// ---------------------------------------------------------------------------
// split + pack: route every output vertex (engine.hpp:880-909) and store the
// remote records directly into the destination inbox slot.  Slot positions are
// reserved once per warp and destination (broadcast: one ballot; selective:
// lanes grouped by destination with match.any), not once per record: a single
// per-destination counter hit by every record serialises at its L2 slice.

template <class F>
__global__ void __launch_bounds__(256)
    split_pack_kernel(F f, OwnerView ow, GraphView g, const uint32_t* __restrict__ out,
                      Counters* ctr, uint32_t* __restrict__ next, const SlotView* __restrict__ table,
                      uint32_t n, int broadcast, unsigned long long drop_mask, int nva, int nvv,
                      int want_deg, DenseView dv) {
  constexpr int A = AssocCap<F>::value;
  const uint32_t cnt = ctr->out_cnt;
  const bool dense = broadcast && dv.kind != 0 && cnt >= dv.threshold;
  const unsigned lane = lane_id(), lt = (1u << lane) - 1u;
  unsigned long long my_deg = 0;
  for (uint32_t base = blockIdx.x * blockDim.x; base < cnt; base += gridDim.x * blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const bool valid = i < cnt;
    uint32_t v = 0, q = ow.p;
    if (valid) {
      v = out[i];
      q = broadcast ? ow.p : ow.owner_of_local(v);
    }
    const bool local = valid && q == ow.p;
    const uint32_t slot = warp_append(&ctr->next_cnt, local);
    if (local) {
      next[slot] = v;
      if (want_deg) my_deg += g.off[v + 1] - g.off[v];
    }
    uint32_t va[A];
    double vv[A];
    if (broadcast) {
      if (dense) continue;
      if (valid) f.gather(v, va, vv);
      const unsigned m = __ballot_sync(0xffffffffu, valid);
      if (!m) continue;
      const unsigned leader = __ffs(m) - 1;
      for (uint32_t d = 0; d < n; ++d) {
        if (d == ow.p || ((drop_mask >> d) & 1ull)) continue;
        uint32_t b = 0;
        if (lane == leader) b = atomicAdd(&ctr->send_cnt[d], (uint32_t)__popc(m));
        b = __shfl_sync(0xffffffffu, b, leader);
        if (!valid) continue;
        const uint32_t pos = b + __popc(m & lt);
        const SlotView& s = table[d];
        if (pos >= s.cap) {
          atomicExch(&ctr->overflow, 1u);
          continue;
        }
        s.ids[pos] = v;
#pragma unroll
        for (int a = 0; a < A; ++a)
          if (a < nva) s.va[a][pos] = va[a];
#pragma unroll
        for (int a = 0; a < A; ++a)
          if (a < nvv) s.vv[a][pos] = vv[a];
      }
    } else {
      // send_filter before the drop test: its side effects (SSSP last_sent)
      // happen for a dropped package too, as in the reference (E:424-432)
      bool send = valid && !local && f.send_filter(q, v);
      if (send && ((drop_mask >> q) & 1ull)) send = false;
      if (send) f.gather(v, va, vv);
      const unsigned m = __ballot_sync(0xffffffffu, send);
      if (!send) continue;
      const unsigned grp = __match_any_sync(m, q);
      const unsigned leader = __ffs(grp) - 1;
      uint32_t b = 0;
      if (lane == leader) b = atomicAdd(&ctr->send_cnt[q], (uint32_t)__popc(grp));
      b = __shfl_sync(grp, b, leader);
      const uint32_t pos = b + __popc(grp & lt);
      const SlotView& s = table[q];
      if (pos >= s.cap) {
        atomicExch(&ctr->overflow, 1u);
        continue;
      }
      s.ids[pos] = f.peer_id(v, q, i);
#pragma unroll
      for (int a = 0; a < A; ++a)
        if (a < nva) s.va[a][pos] = va[a];
#pragma unroll
      for (int a = 0; a < A; ++a)
        if (a < nvv) s.vv[a][pos] = vv[a];
    }
  }
  if (dense) {
    // the whole array, 16 bytes per store, into every peer's slot
    if (blockIdx.x == 0 && threadIdx.x == 0)
      for (uint32_t d = 0; d < n; ++d)
        if (d != ow.p && !((drop_mask >> d) & 1ull)) ctr->send_cnt[d] = cnt | kDenseFlag;
    const uint32_t n4 = dv.words / 4;
    const uint32_t items = n4 + (dv.words - 4 * n4);  // uint4 stores, then the tail words
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < items; k += stride) {
      const bool vec = k < n4;
      uint4 w4 = make_uint4(0u, 0u, 0u, 0u);
      uint32_t w1 = 0;
      if (vec) {
        w4 = reinterpret_cast<const uint4*>(dv.cur)[k];
        if (dv.kind == 1) {
          const uint4 p4 = reinterpret_cast<const uint4*>(dv.prev)[k];
          w4 = make_uint4(w4.x & ~p4.x, w4.y & ~p4.y, w4.z & ~p4.z, w4.w & ~p4.w);
        }
      } else {
        const uint32_t j = n4 * 4 + (k - n4);
        w1 = dv.kind == 1 ? (dv.cur[j] & ~dv.prev[j]) : dv.cur[j];
      }
      for (uint32_t d = 0; d < n; ++d) {
        if (d == ow.p || ((drop_mask >> d) & 1ull)) continue;
        uint32_t* dst = table[d].ids;
        if (vec) reinterpret_cast<uint4*>(dst)[k] = w4;
        else dst[n4 * 4 + (k - n4)] = w1;
      }
    }
  }
  if (want_deg) warp_add_u64(&ctr->next_deg, my_deg);
}

// publish per-destination counts into the peers' slot counters; the system
// fence makes the record stores visible before the count (P2P over NVLink)
// (multi-process, device protocol: then raise this superstep's publish flag
// in every peer's mailbox once all counts are out)
// (epoch_dev: the device-driven loop keeps the epoch in device memory)
static __global__ void publish_kernel(const Counters* ctr, uint32_t* const* cnt_ptr, uint32_t n,
                                      uint32_t p, Mailbox* const* mbox, uint32_t parity,
                                      uint32_t epoch, const uint32_t* epoch_dev = nullptr) {
  if (epoch_dev) epoch = *epoch_dev;
  uint32_t d = threadIdx.x;
  __threadfence_system();
  if (d < n && d != p) *cnt_ptr[d] = ctr->send_cnt[d] < 0xFFFFFFFFu ? ctr->send_cnt[d] : 0u;
  if (!mbox) return;
  __threadfence_system();
  __syncthreads();
  if (d < n && d != p) *reinterpret_cast<volatile uint32_t*>(&mbox[d]->pub[parity][p]) = epoch;
}

// ~60 s at ~2 GHz: a peer that never arrives turns into an error, not a hang
constexpr long long kSpinCycles = 120000000000ll;

// multi-process, device protocol: the merge may start once every peer raised
// its publish flag for this superstep (replaces the host barrier, E:922)
static __global__ void mp_wait_pub_kernel(Mailbox* mine, uint32_t parity, uint32_t epoch,
                                          uint32_t n, uint32_t me, uint32_t* err,
                                          const uint32_t* epoch_dev = nullptr) {
  if (epoch_dev) epoch = *epoch_dev;
  const uint32_t q = threadIdx.x;
  if (q < n && q != me) {
    const volatile uint32_t* f = &mine->pub[parity][q];
    const long long t0 = clock64();
    while (*f != epoch) {
      __nanosleep(200);
      if (clock64() - t0 > kSpinCycles) {
        atomicExch(err, 1u);
        break;
      }
    }
  }
  __threadfence();
}

// host-known part of a WorkerReport (set by the primitive's host hooks)
struct HostReportPart {
  double f[4];
  unsigned long long u[4];
  int next_is_out;
};

// multi-process, device protocol: build this rank's WorkerReport, store it
// into every rank's mailbox (arrival flag last), hand the own counters to the
// host and clear them, wait for all ranks' reports and copy the n reports to
// the mapped host page — the WorkerReport all-gather of the completion step
// (E:784-820) without a host barrier
static __global__ void mp_report_kernel(Counters* ctr, Counters* host_ctr, HostReportPart hp,
                                        Mailbox* const* mbox, uint32_t n, uint32_t me,
                                        uint32_t epoch, DevReport* host_out, uint32_t* err,
                                        const uint32_t* epoch_dev = nullptr) {
  if (epoch_dev) epoch = *epoch_dev;
  const uint32_t slot = epoch & 1u;
  if (threadIdx.x == 0) {
    DevReport r;
    r.out_frontier = ctr->out_cnt;
    r.next_frontier = hp.next_is_out ? ctr->out_cnt : ctr->next_cnt;
    r.edges_delta = ctr->edges;
    r.combine_delta = ctr->combine;
    for (int k = 0; k < 4; ++k) {
      r.f[k] = hp.f[k] != 0.0 ? hp.f[k] : ctr->f[k];
      r.u[k] = hp.u[k] != 0ull ? hp.u[k] : ctr->u[k];
    }
    for (uint32_t q = 0; q < kMaxMpRanks; ++q) r.send_cnt[q] = q < n ? ctr->send_cnt[q] : 0u;
    r.overflow = ctr->overflow;
    r.epoch = 0;
    for (uint32_t d = 0; d < n; ++d) {
      DevReport* dst = &mbox[d]->rep[slot][me];
      const uint32_t* src = reinterpret_cast<const uint32_t*>(&r);
      uint32_t* o = reinterpret_cast<uint32_t*>(dst);
      for (uint32_t i = 0; i + 1 < sizeof(DevReport) / 4; ++i) o[i] = src[i];
    }
    __threadfence_system();
    for (uint32_t d = 0; d < n; ++d)
      *reinterpret_cast<volatile uint32_t*>(&mbox[d]->rep[slot][me].epoch) = epoch;
  }
  __syncthreads();
  {  // own counters to the host (unless null), cleared for the next superstep
    uint32_t* src = reinterpret_cast<uint32_t*>(ctr);
    volatile uint32_t* dst = reinterpret_cast<volatile uint32_t*>(host_ctr);
    for (uint32_t i = threadIdx.x; i < sizeof(Counters) / 4; i += blockDim.x) {
      if (dst) dst[i] = src[i];
      src[i] = 0u;
    }
  }
  const uint32_t q = threadIdx.x;
  if (q < n) {
    const volatile uint32_t* f = &mbox[me]->rep[slot][q].epoch;
    const long long t0 = clock64();
    while (*f != epoch) {
      __nanosleep(200);
      if (clock64() - t0 > kSpinCycles) {
        atomicExch(err, 1u);
        break;
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (!host_out) return;
  const uint32_t words = n * (uint32_t)(sizeof(DevReport) / 4);
  const volatile uint32_t* src = reinterpret_cast<const volatile uint32_t*>(mbox[me]->rep[slot]);
  volatile uint32_t* dst = reinterpret_cast<volatile uint32_t*>(host_out);
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
}

// merge (engine.hpp:823-852): combine every received record; an accepted
// vertex is enqueued once per superstep through the merge stamp
template <class F>
__global__ void __launch_bounds__(256)
    merge_kernel(F f, const SlotView* __restrict__ slots, const uint32_t* __restrict__ inbox_cnt,
                 uint32_t p, uint32_t stamp, uint32_t iteration, uint32_t* merge_stamp,
                 uint32_t* __restrict__ next, Counters* ctr, GraphView g, int nva, int nvv,
                 int enqueue, int want_deg, const uint32_t* iter_dev = nullptr) {
  if (iter_dev) {  // device-driven loop: the superstep index lives in device memory
    iteration = *iter_dev;
    stamp = iteration + 1;
  }
  const uint32_t src = blockIdx.y;
  if (src == p) return;
  const uint32_t cnt = inbox_cnt[src];
  if (cnt & kDenseFlag) return;  // merge_dense_kernel
  const SlotView s = slots[src];
  if (threadIdx.x == 0 && blockIdx.x == 0) ctr->recv_cnt[src] = cnt;
  unsigned long long my_deg = 0, my_comb = 0;
  for (uint32_t base = blockIdx.x * blockDim.x; base < cnt; base += gridDim.x * blockDim.x) {
    uint32_t i = base + threadIdx.x;
    bool push = false;
    uint32_t v = 0;
    if (i < cnt) {
      v = s.ids[i];
      constexpr int A = AssocCap<F>::value;
      uint32_t va[A];
      double vv[A];
#pragma unroll
      for (int a = 0; a < A; ++a) va[a] = a < nva ? s.va[a][i] : 0u;
#pragma unroll
      for (int a = 0; a < A; ++a) vv[a] = a < nvv ? s.vv[a][i] : 0.0;
      ++my_comb;
      bool accepted = f.combine(v, va, vv, iteration);
      if (accepted && enqueue) push = atomicExch(&merge_stamp[v], stamp) != stamp;
    }
    uint32_t slot = warp_append(&ctr->next_cnt, push);
    if (push) {
      next[slot] = v;
      if (want_deg) my_deg += g.off[v + 1] - g.off[v];
    }
  }
  if (want_deg) warp_add_u64(&ctr->next_deg, my_deg);
  warp_add_u64(&ctr->combine, my_comb);
}

// merge of a dense slot (see DenseView): kind 1 combines every bit the
// receiver has not visited yet (a visited vertex cannot take an equal-or-later
// label, so combine() on it would be a no-op); kind 2 combines every value
// (no-ops outside the sender's delta).  C counts the sender's records.
template <class F>
__global__ void __launch_bounds__(256)
    merge_dense_kernel(F f, DenseView dv, const SlotView* __restrict__ slots,
                       const uint32_t* __restrict__ inbox_cnt, uint32_t p, uint32_t stamp,
                       uint32_t iteration, uint32_t* merge_stamp, uint32_t* __restrict__ next,
                       Counters* ctr, GraphView g, int want_deg,
                       const uint32_t* iter_dev = nullptr) {
  if (iter_dev) {
    iteration = *iter_dev;
    stamp = iteration + 1;
  }
  constexpr int A = AssocCap<F>::value;
  const uint32_t src = blockIdx.y;
  if (src == p) return;
  const uint32_t c = inbox_cnt[src];
  if (!(c & kDenseFlag)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctr->recv_cnt[src] = c & ~kDenseFlag;
    atomicAdd(&ctr->combine, (unsigned long long)(c & ~kDenseFlag));
  }
  const uint32_t* __restrict__ words = slots[src].ids;
  uint32_t va[A];
  double vv[A];
#pragma unroll
  for (int a = 0; a < A; ++a) {
    va[a] = 0u;
    vv[a] = 0.0;
  }
  unsigned long long my_deg = 0;
  for (uint32_t base = blockIdx.x * blockDim.x; base < dv.words; base += gridDim.x * blockDim.x) {
    const uint32_t k = base + threadIdx.x;
    if (dv.kind == 1) {
      uint32_t cand = 0;
      if (k < dv.words) {
        cand = words[k];
        if (cand) cand &= ~__ldcg(&dv.vis[k]);
      }
      while (__any_sync(0xffffffffu, cand != 0)) {
        bool push = false;
        uint32_t v = 0;
        if (cand) {
          v = k * 32 + (__ffs(cand) - 1);
          cand &= cand - 1;
          if (f.combine(v, va, vv, iteration)) push = atomicExch(&merge_stamp[v], stamp) != stamp;
        }
        const uint32_t slot = warp_append(&ctr->next_cnt, push);
        if (push) {
          next[slot] = v;
          if (want_deg) my_deg += g.off[v + 1] - g.off[v];
        }
      }
    } else {
      bool push = false;
      if (k < dv.words) {
        va[0] = words[k];
        if (f.combine(k, va, vv, iteration)) push = atomicExch(&merge_stamp[k], stamp) != stamp;
      }
      const uint32_t slot = warp_append(&ctr->next_cnt, push);
      if (push) {
        next[slot] = k;
        if (want_deg) my_deg += g.off[k + 1] - g.off[k];
      }
    }
  }
  if (want_deg) warp_add_u64(&ctr->next_deg, my_deg);
}

// degree sum of a frontier (init: the advance bound of superstep 0)
static __global__ void degsum_kernel(GraphView g, const uint32_t* __restrict__ in, uint32_t n,
                              unsigned long long* out) {
  unsigned long long d = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t v = in[i];
    d += g.off[v + 1] - g.off[v];
  }
  warp_add_u64(out, d);
}

// same, with the length read on the device (n == 1 path: output becomes input)
static __global__ void degsum_dev_kernel(GraphView g, const uint32_t* __restrict__ in,
                                         const uint32_t* n_ptr, unsigned long long* out) {
  const uint32_t n = *n_ptr;
  unsigned long long d = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t v = in[i];
    d += g.off[v + 1] - g.off[v];
  }
  warp_add_u64(out, d);
}

constexpr uint64_t kUnknownDeg = ~0ull;

// end of superstep: the counters go to the worker's mapped pinned page (one
// small kernel instead of a D2H copy) and are cleared for the next superstep
// (instead of a memset at its start)
static __global__ void report_kernel(Counters* ctr, Counters* host) {
  uint32_t* src = reinterpret_cast<uint32_t*>(ctr);
  volatile uint32_t* dst = reinterpret_cast<volatile uint32_t*>(host);
  for (uint32_t i = threadIdx.x; i < sizeof(Counters) / 4; i += blockDim.x) {
    dst[i] = src[i];
    src[i] = 0u;
  }
}

// ---------------------------------------------------------------------------
// per-(run, worker) context: the WorkerHandle of the reference (engine.hpp:478-582)

struct RunState;

struct Ctx {
  Plan* P = nullptr;
  Worker* w = nullptr;
  RunState* run = nullptr;
  uint64_t iter = 0;
  const GlobalView* prev = nullptr;
  bool fused = false;
  bool want_deg = true;     // exact advance bounds tracked (policy != max)
  uint32_t in_count = 0;    // input frontier length (host-known)
  uint64_t in_degsum = 0;   // sum of its out-degrees (host-known)
  WorkerReport report;      // host-side f/u fields set by hooks

  uint32_t worker() const { return w->p; }
  uint32_t num_workers() const { return P->n; }
  cudaStream_t stream() const { return w->stream; }
  OwnerView owner_view() const {
    return {w->owner.ptr, w->l2g.ptr, w->p, w->nlocal, P->dup};
  }
  GraphView graph() const { return w->graph(); }
  Counters* ctr() const { return w->ctr.ptr; }

  // seed the initial frontier (valid inside init only), E:511-514
  void push_initial(const std::vector<uint32_t>& vs);

  void ensure_output(uint64_t items) { w->output.ensure(items, w->stream); }

  // advance over the input frontier (E:516-520): edge-balanced expansion
  template <class F, bool kFused>
  void lb_advance(const F& f, uint32_t* dst, uint32_t* dst_cnt) {
    if (in_count == 0) return;
    const uint32_t nb = (in_count + kLbBlock - 1) / kLbBlock;
    if (w->lb_row.n < in_count) w->lb_row.alloc(in_count);
    if (w->lb_pref.n < in_count) w->lb_pref.alloc(in_count);
    if (w->lb_bsum.n < nb + 1ull) w->lb_bsum.alloc(nb + 1ull);
    MGB_LAUNCH(lb_degree_kernel, nb, kLbBlock, 0, w->stream, w->off.ptr, w->input.ptr, in_count,
               w->lb_row.ptr, w->lb_pref.ptr, w->lb_bsum.ptr);
    MGB_LAUNCH(lb_scan_kernel, 1, 1024, 0, w->stream, w->lb_bsum.ptr, nb, w->lb_bsum.ptr + nb,
               &ctr()->edges);
    // tile table: exact when the degree sum is known, else bounded by 2|E_i|
    // (an input frontier may hold a vertex twice, e.g. SSSP, E:901-904 + E:845)
    const uint64_t max_deg = in_degsum == kUnknownDeg ? 2 * w->ne + 1 : in_degsum;
    const uint64_t max_tiles = max_deg / kTile + 2 + kMinTiles;
    if (w->lb_tile.n < max_tiles + 1) w->lb_tile.alloc(max_tiles + 1);
    MGB_LAUNCH(lb_tiles_kernel, grid_for(max_tiles + 1, 256, num_sms() * 8), 256, 0, w->stream,
               w->lb_pref.ptr, w->lb_bsum.ptr, in_count, w->lb_bsum.ptr + nb, w->lb_tile.ptr,
               (uint32_t)max_tiles);
    const unsigned resident = expand_resident<F, kFused>();
    unsigned grid = in_degsum == kUnknownDeg ? resident
                                             : grid_for(in_degsum, lb_tile_size(in_degsum), resident);
    MGB_LAUNCH((lb_expand_kernel<F, kFused>), grid, kExpBlock, 0, w->stream, f, graph(),
               w->input.ptr, in_count, w->lb_row.ptr, w->lb_pref.ptr, w->lb_bsum.ptr,
               w->lb_bsum.ptr + nb, w->lb_tile.ptr, dst, dst_cnt);
  }

  template <class F>
  void run_advance(const F& f, uint32_t* dst, uint32_t* dst_cnt) {
    lb_advance<F, false>(f, dst, dst_cnt);
  }

  // exact degree sum of the input when the producer did not provide it
  uint64_t degsum() {
    if (in_degsum != kUnknownDeg) return in_degsum;
    unsigned long long* tmp = &ctr()->next_deg;  // free until split/merge of this superstep
    MGB_CUDA(cudaMemsetAsync(tmp, 0, 8, w->stream));
    if (in_count)
      MGB_LAUNCH(degsum_kernel, grid_for(in_count, 256, num_sms() * 8), 256, 0, w->stream, graph(),
                 w->input.ptr, in_count, tmp);
    unsigned long long h = 0;
    MGB_CUDA(cudaMemcpyAsync(&h, tmp, 8, cudaMemcpyDeviceToHost, w->stream));
    MGB_CUDA(cudaMemsetAsync(tmp, 0, 8, w->stream));
    MGB_CUDA(cudaStreamSynchronize(w->stream));
    in_degsum = h;
    return h;
  }

  // fused or two-stage traversal per the active policy (E:528-541); the
  // result lands in w->output with its length in ctr()->out_cnt
  template <class F>
  void pipeline(const F& f, uint64_t dedup_bound) {
    if (fused) {
      uint64_t b = in_degsum < dedup_bound ? in_degsum : dedup_bound;  // unknown -> bound
      ensure_output(b);
      lb_advance<F, true>(f, w->output.ptr, &ctr()->out_cnt);
    } else {
      w->advance_out.ensure(degsum(), w->stream);
      run_advance(f, w->advance_out.ptr, &ctr()->adv_cnt);
      // filter_output_bound(advance_out.size(), |V_i|) (frontier.hpp:204-208): the
      // unfused path reads the advance length back to size the filter exactly
      uint32_t adv = 0;
      MGB_CUDA(cudaMemcpyAsync(&adv, &ctr()->adv_cnt, 4, cudaMemcpyDeviceToHost, w->stream));
      MGB_CUDA(cudaStreamSynchronize(w->stream));
      ensure_output(adv < dedup_bound ? adv : dedup_bound);
      if (adv == 0) return;
      MGB_LAUNCH(filter_kernel<F>, grid_for(adv, 256, num_sms() * 8), 256, 0, w->stream, f,
                 w->advance_out.ptr, &ctr()->adv_cnt, w->output.ptr, &ctr()->out_cnt);
    }
  }
};

struct RunState {
  int comm = MG_COMM_SELECTIVE;
  std::vector<GlobalView> views;
  std::vector<uint32_t> in_count, next_count;
  std::vector<uint64_t> in_deg, next_deg;
  std::vector<cudaEvent_t> packed;  // per worker, recorded after publish
  std::vector<uint32_t> dense_words;  // per worker: words of its dense view this superstep
};

struct SmallList {
  uint32_t n, v[8];
};
static __global__ void put_small_kernel(uint32_t* dst, SmallList l) {
  if (threadIdx.x < l.n) dst[threadIdx.x] = l.v[threadIdx.x];
}

inline void Ctx::push_initial(const std::vector<uint32_t>& vs) {
  uint32_t& nc = run->next_count[w->p];
  w->next_input.ensure(nc + vs.size(), w->stream, nc);
  if (vs.size() <= 8) {  // sources: by kernel argument, no host round trip
    SmallList l{static_cast<uint32_t>(vs.size()), {}};
    for (size_t i = 0; i < vs.size(); ++i) l.v[i] = vs[i];
    if (!vs.empty()) MGB_LAUNCH(put_small_kernel, 1, 32, 0, w->stream, w->next_input.ptr + nc, l);
  } else {
    MGB_CUDA(cudaMemcpyAsync(w->next_input.ptr + nc, vs.data(), vs.size() * 4,
                             cudaMemcpyHostToDevice, w->stream));
    MGB_CUDA(cudaStreamSynchronize(w->stream));  // vs is a host temporary
  }
  nc += static_cast<uint32_t>(vs.size());
}

// allocate / grow the receiver inbox arena of worker w for slot capacities caps[src]
void ensure_inboxes(Plan& P, Worker& w, int nva, int nvv, const std::vector<uint64_t>& caps);
// refresh every local worker's send tables (after any arena changed)
void build_send_tables(Plan& P);
void prepare_worker(Plan& P, Worker& w, const mg_config& cfg);
void collect_buffer_stats(Plan& P);

// the primitive's device functor set: one type (dev()), or a choice of two
// made per run (SSSP's u32 / u64 distances: dev32() / dev64())
template <class Prim, class Fn>
auto with_dev(Prim& prim, Ctx& c, Fn&& fn) -> decltype(prim.dev(c), void()) {
  fn(prim.dev(c));
}
template <class Prim, class Fn>
auto with_dev(Prim& prim, Ctx& c, Fn&& fn) -> decltype(prim.dev32(c), void()) {
  if (prim.narrow) fn(prim.dev32(c));
  else fn(prim.dev64(c));
}

// ---------------------------------------------------------------------------
// device-driven superstep loop (a primitive may run the whole loop as one
// CUDA graph; the enactor then rebuilds its statistics from the history)
struct DeviceLoopOut {
  uint32_t supersteps = 0;
  int stop_reason = MG_STOP_FRONTIERS_EMPTY;
  std::vector<uint64_t> out, next, edges, combine;
  std::vector<std::vector<uint64_t>> h_src;     // per superstep: records sent by each worker
  std::vector<std::vector<uint64_t>> h_matrix;  // [src][dst] totals
  uint64_t wire = 0, xbytes = 0;
};

template <class Prim>
auto try_device_loop(Prim& prim, Plan& P, std::vector<Ctx>& ctx, RunState& rs,
                     const mg_config& cfg, DeviceLoopOut& o, int)
    -> decltype(prim.device_loop(P, ctx, rs, cfg, o)) {
  return prim.device_loop(P, ctx, rs, cfg, o);
}
template <class Prim>
bool try_device_loop(Prim&, Plan&, std::vector<Ctx>&, RunState&, const mg_config&,
                     DeviceLoopOut&, long) {
  return false;
}

// ---------------------------------------------------------------------------
// the enactor

// MG_TRACE_HOST=1: host timestamps of the enactor's phases on stderr
struct HostTrace {
  bool on = getenv("MG_TRACE_HOST") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void operator()(const char* what, uint64_t i = 0) const {
    if (!on) return;
    double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0)
                    .count();
    fprintf(stderr, "[trace] %9.1f us  %s %llu\n", us, what, (unsigned long long)i);
  }
};

// does the primitive leave a DOBFS label array behind (DobfsPrim)?  Every
// other run invalidates the incremental label reset (Worker::dobfs_labels_ok)
template <class Prim>
auto keeps_dobfs_labels(const Prim& p, int) -> decltype(bool(p.keeps_dobfs_labels)) {
  return p.keeps_dobfs_labels;
}
template <class Prim>
bool keeps_dobfs_labels(const Prim&, long) {
  return false;
}

template <class Prim>
void run_primitive(Plan& P, Prim& prim, const mg_config& cfg) {
  HostTrace trace;
  trace("enter");
  const uint32_t n = P.n;
  if (!keeps_dobfs_labels(prim, 0))
    for (uint32_t p : P.local_workers) P.workers[p]->dobfs_labels_ok = false;
  if (prim.nva < 0 || prim.nva > kMaxAssoc || prim.nvv < 0 || prim.nvv > kMaxAssoc)
    throw Error(MG_EINVAL, std::string(prim.name) + ": at most " + std::to_string(kMaxAssoc) +
                               " vertex and value associates per record");
  if (prim.dup_required >= 0 && P.dup != prim.dup_required)
    throw Error(MG_EINVAL, std::string(prim.name) + ": requires --dup " +
                               (prim.dup_required == MG_DUP_ALL ? "all" : "onehop"));
  for (int r = 0; r < MG_NUM_ROLES; ++r)
    if (cfg.factors[r] < 0.0)
      throw Error(MG_EINVAL, std::string("sizing factor for ") +
                                 (r == 0 ? "advance_output" : r == 1 ? "filter_output" :
                                  r == 2 ? "input_frontier" : r == 3 ? "outbox" : "inbox") +
                                 " must not be negative");
  int comm = prim.communication;
  if (cfg.comm_override >= 0 && cfg.comm_override != prim.communication) {
    if (!prim.allow_comm_override)
      throw Error(MG_EINVAL, std::string(prim.name) + ": communication mode is fixed to " +
                                 (prim.communication == MG_COMM_SELECTIVE ? "selective"
                                                                          : "broadcast"));
    comm = cfg.comm_override;
  }
  // exact advance bounds are tracked unless the policy preallocated the maximum
  const bool want_deg = cfg.policy != MG_POLICY_MAX;
  const bool fused = cfg.fused == MG_FUSED_ON || (cfg.fused == MG_FUSED_AUTO &&
                                                  cfg.policy == MG_POLICY_FUSED);
  RunState rs;
  rs.comm = comm;
  rs.in_count.assign(n, 0);
  rs.next_count.assign(n, 0);
  rs.in_deg.assign(n, 0);
  rs.next_deg.assign(n, 0);
  rs.packed.assign(n, nullptr);
  rs.dense_words.assign(n, 0);
  // a hook or kernel that throws mid-run (a worker failure, E:773-782) must not
  // leak the per-run events: the plan stays usable for the next call
  struct EventGuard {
    std::vector<cudaEvent_t>& ev;
    ~EventGuard() {
      for (auto& e : ev)
        if (e) cudaEventDestroy(e), e = nullptr;
    }
  } event_guard{rs.packed};

  std::vector<Ctx> ctx(n);
  for (uint32_t p : P.local_workers) {
    Worker& w = *P.workers[p];
    DeviceGuard dg(w.dev);
    prepare_worker(P, w, cfg);
    std::vector<uint64_t> caps(n, 0);
    for (uint32_t s = 0; s < n; ++s)
      if (s != p) caps[s] = prim.inbox_bound(P, s, p, comm);
    ensure_inboxes(P, w, prim.nva, prim.nvv, caps);
    MGB_CUDA(cudaEventCreateWithFlags(&rs.packed[p], cudaEventDisableTiming));
    ctx[p].P = &P;
    ctx[p].w = &w;
    ctx[p].run = &rs;
    ctx[p].fused = fused;
    ctx[p].want_deg = want_deg;
  }
  trace("workers prepared");
  if (P.shm) fabric_sync(P);  // collective: map peers' (possibly regrown) arenas
  const bool dev_fabric = P.shm && P.device_fabric;
  uint32_t* mp_err = dev_fabric ? reinterpret_cast<uint32_t*>(P.host_reports_dev + kMaxMpRanks)
                                : nullptr;
  uint32_t* mp_err_host = dev_fabric ? reinterpret_cast<uint32_t*>(P.host_reports + kMaxMpRanks)
                                     : nullptr;
  if (dev_fabric) *reinterpret_cast<volatile uint32_t*>(mp_err_host) = 0;
  build_send_tables(P);
  trace("send tables");
  P.h_matrix.assign(n, std::vector<uint64_t>(n, 0));
  P.prof_ms = 0;
  P.prof_bytes = 0;
  P.prof_launches = 0;
  P.prof2_ms = 0;
  P.prof2_bytes = 0;
  P.prof2_launches = 0;
  P.h_per_iter.clear();
  P.out_per_iter.clear();
  P.edges_per_iter.clear();
  P.combine_per_iter.clear();
  uint64_t launches0 = g_launches.load();
  uint64_t total_edges = 0, total_combine = 0, wire = 0, xbytes = 0;
  const uint32_t inflation = cfg.h_inflation ? cfg.h_inflation : 1;
  int stop_reason = MG_STOP_FRONTIERS_EMPTY;

  auto t0 = std::chrono::steady_clock::now();
  for (uint32_t p : P.local_workers) {
    Worker& w = *P.workers[p];
    DeviceGuard dg(w.dev);
    MGB_CUDA(cudaEventRecord(w.ev_start, w.stream));
    MGB_CUDA(cudaMemsetAsync(w.ctr.ptr, 0, sizeof(Counters), w.stream));
    // the merge stamp is only read by the merge kernel (n > 1)
    if (n > 1)
      MGB_CUDA(cudaMemsetAsync(w.merge_stamp.ptr, 0, sizeof(uint32_t) * w.nv, w.stream));
    trace("ctr cleared");
    prim.init(ctx[p]);
    trace("prim init");
    // advance bound of superstep 0 (only tracked when the policy sizes buffers
    // exactly; the max policy needs no host round trip before superstep 0)
    if (want_deg) {
      if (rs.next_count[p])
        MGB_LAUNCH(degsum_kernel, grid_for(rs.next_count[p], 256, 1024), 256, 0, w.stream,
                   w.graph(), w.next_input.ptr, rs.next_count[p], &w.ctr.ptr->next_deg);
      MGB_LAUNCH(report_kernel, 1, 128, 0, w.stream, w.ctr.ptr, w.host_ctr_dev);
    }
  }
  for (uint32_t p : P.local_workers) {
    if (want_deg) {
      MGB_CUDA(cudaStreamSynchronize(P.workers[p]->stream));
      rs.next_deg[p] = P.workers[p]->host_ctr->next_deg;
    } else {
      rs.next_deg[p] = kUnknownDeg;
    }
  }

  DeviceLoopOut dlo;
  const bool on_device = try_device_loop(prim, P, ctx, rs, cfg, dlo, 0);
  if (on_device) {
    for (uint32_t t = 0; t < dlo.supersteps; ++t) {
      GlobalView v;
      v.iteration = t;
      v.num_workers = n;
      v.reports.resize(n);
      v.total_out = dlo.out[t];
      v.total_next = dlo.next[t];
      rs.views.push_back(std::move(v));
      P.out_per_iter.push_back(dlo.out[t]);
      P.h_per_iter.push_back(dlo.h_src[t]);
      P.edges_per_iter.push_back(dlo.edges[t]);
      P.combine_per_iter.push_back(dlo.combine[t]);
      total_edges += dlo.edges[t];
      total_combine += dlo.combine[t];
    }
    P.h_matrix = dlo.h_matrix;
    wire = dlo.wire * inflation;
    xbytes = dlo.xbytes;
    stop_reason = dlo.stop_reason;
  }
  for (uint64_t iter = 0; !on_device; ++iter) {
    const GlobalView* prev = rs.views.empty() ? nullptr : &rs.views.back();
    const uint32_t parity = iter & 1u;
    if (dev_fabric) ++P.mp_epoch;  // same sequence on every rank (same decisions)
    std::vector<int> step_comm(n, comm);
    // body + split/pack + publish
    for (uint32_t p : P.local_workers) {
      Worker& w = *P.workers[p];
      Ctx& c = ctx[p];
      DeviceGuard dg(w.dev);
      std::swap(w.input, w.next_input);
      c.in_count = rs.in_count[p] = rs.next_count[p];
      c.in_degsum = rs.in_deg[p] = rs.next_deg[p];
      rs.next_count[p] = 0;
      c.iter = iter;
      c.prev = prev;
      c.report = WorkerReport{};
      // the counters were cleared by the previous report_kernel (or at run start)
      trace("superstep", iter);
      prim.body(c);
      trace("body issued", iter);
      step_comm[p] = prim.comm_selector(c, comm);
      if (n == 1) {
        // single partition: every output vertex is local (E:901-904), so the
        // output buffer simply becomes the next input — no split kernel
        std::swap(w.output.ptr, w.next_input.ptr);
        std::swap(w.output.phys, w.next_input.phys);
        uint64_t oc = w.output.cap;
        w.output.cap = w.next_input.cap;
        w.next_input.cap = oc;
        if (want_deg)
          MGB_LAUNCH(degsum_dev_kernel, num_sms() * 4, 256, 0, w.stream, w.graph(),
                     w.next_input.ptr, &w.ctr.ptr->out_cnt, &w.ctr.ptr->next_deg);
        MGB_CUDA(cudaEventRecord(rs.packed[p], w.stream));
        continue;
      }
      // next_input holds the local part plus everything merged this superstep
      // (a dense slot can merge any vertex; merged vertices are unique)
      const DenseView dv = step_comm[p] == MG_COMM_BROADCAST ? prim.dense_view(c) : DenseView{};
      rs.dense_words[p] = dv.kind ? dv.words : 0;
      uint64_t incoming = 0;
      for (uint32_t s = 0; s < n; ++s) incoming += (s == p) ? 0 : w.slot_cap[s];
      if (prim.dense_view(c).kind && incoming < w.nv) incoming = w.nv;
      w.next_input.ensure(w.output.cap + incoming, w.stream);
      unsigned long long drop = 0;
      if (cfg.drop_enabled && cfg.drop_src == p && cfg.drop_iteration == iter &&
          cfg.drop_dst < 64)
        drop = 1ull << cfg.drop_dst;
      if (n > 1) MGB_CUDA(cudaEventRecord(w.ev_x0, w.stream));
      with_dev(prim, c, [&](auto dev) {
        const uint64_t items = w.output.cap > dv.words ? w.output.cap : dv.words;
        MGB_LAUNCH(split_pack_kernel<decltype(dev)>, grid_for(items, 256, num_sms() * 8), 256, 0,
                   w.stream, dev, c.owner_view(), w.graph(), w.output.ptr, w.ctr.ptr,
                   w.next_input.ptr, w.send_table.ptr + parity * n, n,
                   step_comm[p] == MG_COMM_BROADCAST ? 1 : 0, drop, prim.nva, prim.nvv,
                   (want_deg || prim.reports_deg) ? 1 : 0, dv);
      });
      if (n > 1) {
        MGB_LAUNCH(publish_kernel, 1, 64, 0, w.stream, w.ctr.ptr, w.send_cnt_ptr.ptr + parity * n,
                   n, p, dev_fabric ? P.mbox_ptrs.ptr : nullptr, parity, P.mp_epoch);
        MGB_CUDA(cudaEventRecord(w.ev_x1, w.stream));
      }
      MGB_CUDA(cudaEventRecord(rs.packed[p], w.stream));
    }
    if (dev_fabric) {
      // peers in other processes: wait on the device for their publish flags
      Worker& w = *P.workers[P.rank];
      DeviceGuard dg(w.dev);
      MGB_LAUNCH(mp_wait_pub_kernel, 1, 32, 0, w.stream,
                 reinterpret_cast<Mailbox*>(P.mbox.ptr), parity, P.mp_epoch, n, P.rank, mp_err);
    } else if (P.shm) {
      // peers in other processes: their pack + publish kernels must have
      // completed (system-scope fenced) before this rank merges (E:922)
      for (uint32_t p : P.local_workers) MGB_CUDA(cudaStreamSynchronize(P.workers[p]->stream));
      P.shm->barrier();
    }
    // merge (after every peer's pack: event dependencies, no host barrier)
    for (uint32_t p : P.local_workers) {
      Worker& w = *P.workers[p];
      Ctx& c = ctx[p];
      DeviceGuard dg(w.dev);
      if (n > 1) {
        for (uint32_t s : P.local_workers)
          if (s != p) MGB_CUDA(cudaStreamWaitEvent(w.stream, rs.packed[s], 0));
        uint64_t maxcap = 0;
        for (uint32_t s = 0; s < n; ++s)
          if (s != p && w.slot_cap[s] > maxcap) maxcap = w.slot_cap[s];
        dim3 grid(grid_for(maxcap, 256, num_sms() * 2), n);
        const DenseView dv = prim.dense_view(c);
        with_dev(prim, c, [&](auto dev) {
          MGB_LAUNCH(merge_kernel<decltype(dev)>, grid, 256, 0, w.stream, dev,
                     w.recv_table.ptr + parity * n, w.inbox_cnt.ptr + parity * kMaxWorkers, p,
                     (uint32_t)(iter + 1), (uint32_t)iter, w.merge_stamp.ptr, w.next_input.ptr,
                     w.ctr.ptr, w.graph(), prim.nva, prim.nvv, 1,
                     (want_deg || prim.reports_deg) ? 1 : 0);
          if (dv.kind)
            MGB_LAUNCH(merge_dense_kernel<decltype(dev)>,
                       dim3(grid_for(dv.words, 256, num_sms() * 2), n), 256, 0, w.stream, dev, dv,
                       w.recv_table.ptr + parity * n, w.inbox_cnt.ptr + parity * kMaxWorkers, p,
                       (uint32_t)(iter + 1), (uint32_t)iter, w.merge_stamp.ptr,
                       w.next_input.ptr, w.ctr.ptr, w.graph(),
                       (want_deg || prim.reports_deg) ? 1 : 0);
        });
      }
      prim.after_merge(c);
      if (dev_fabric) {
        HostReportPart hp{};
        for (int k = 0; k < 4; ++k) {
          hp.f[k] = c.report.f[k];
          hp.u[k] = c.report.u[k];
        }
        hp.next_is_out = 0;
        MGB_LAUNCH(mp_report_kernel, 1, 128, 0, w.stream, w.ctr.ptr, w.host_ctr_dev, hp,
                   P.mbox_ptrs.ptr, n, P.rank, P.mp_epoch, P.host_reports_dev, mp_err);
      } else {
        MGB_LAUNCH(report_kernel, 1, 128, 0, w.stream, w.ctr.ptr, w.host_ctr_dev);
      }
    }
    // barrier + completion (E:940, E:784-820)
    GlobalView view;
    view.iteration = static_cast<uint32_t>(iter);
    view.num_workers = n;
    view.reports.resize(n);
    std::vector<uint64_t> h_src(n, 0);
    uint64_t it_edges = 0, it_comb = 0;
    for (uint32_t p : P.local_workers) {
      Worker& w = *P.workers[p];
      trace("sync", iter);
      MGB_CUDA(cudaStreamSynchronize(w.stream));
      trace("synced", iter);
      const Counters& hc = *w.host_ctr;
      if (hc.overflow) throw Error(MG_EWORKER, "inbox overflow on worker " + std::to_string(p));
      WorkerReport r = ctx[p].report;
      r.out_frontier = hc.out_cnt;
      r.next_frontier = n == 1 ? hc.out_cnt : hc.next_cnt;
      r.edges_delta = hc.edges;
      r.combine_delta = hc.combine;
      for (int k = 0; k < 4; ++k) {
        if (r.f[k] == 0.0) r.f[k] = hc.f[k];
        if (r.u[k] == 0) r.u[k] = hc.u[k];
      }
      view.reports[p] = r;
      rs.next_count[p] = (uint32_t)r.next_frontier;
      rs.next_deg[p] = (want_deg || prim.reports_deg) ? hc.next_deg : kUnknownDeg;
      if (n > 1) {
        for (uint32_t q = 0; q < n; ++q) {
          if (q == p) continue;
          const uint64_t len = hc.send_cnt[q] & ~kDenseFlag;  // records (E:391-393)
          P.h_matrix[p][q] += len;
          h_src[p] += len;
          wire += len * inflation;
          xbytes += (hc.send_cnt[q] & kDenseFlag) ? 4ull * rs.dense_words[p]
                                                  : len * (4ull + 4ull * prim.nva + 8ull * prim.nvv);
        }
        float xms = 0;
        cudaEventElapsedTime(&xms, w.ev_x0, w.ev_x1);
        P.last.exchange_ms += xms;
      }
      it_edges += hc.edges;
      it_comb += hc.combine;
    }
    if (P.shm) {
      // multi-process: every rank contributes its report; all ranks then hold
      // the same GlobalView and reach the same stop decision (E:784-820)
      const uint32_t me = P.rank;
      std::vector<WorkerReport> reports;
      std::vector<std::vector<uint32_t>> sends;
      bool overflow = false;
      if (dev_fabric) {  // gathered on the devices by mp_report_kernel
        if (*reinterpret_cast<volatile uint32_t*>(mp_err_host))
          throw Error(MG_EWORKER, "fabric: a peer rank did not arrive within the timeout");
        reports.assign(n, WorkerReport{});
        sends.assign(n, std::vector<uint32_t>(n, 0));
        for (uint32_t q = 0; q < n; ++q) {
          const DevReport& d = P.host_reports[q];
          if (d.epoch != P.mp_epoch) throw Error(MG_EWORKER, "fabric: stale report");
          WorkerReport& x = reports[q];
          x.out_frontier = d.out_frontier;
          x.next_frontier = d.next_frontier;
          x.edges_delta = d.edges_delta;
          x.combine_delta = d.combine_delta;
          for (int k = 0; k < 4; ++k) {
            x.f[k] = d.f[k];
            x.u[k] = d.u[k];
          }
          for (uint32_t e = 0; e < n; ++e) sends[q][e] = d.send_cnt[e] & ~kDenseFlag;
          overflow |= d.overflow != 0;
        }
      } else {
        fabric_exchange_reports(P, view.reports[me], *P.workers[me]->host_ctr, reports, sends,
                                overflow);
      }
      if (overflow) throw Error(MG_EWORKER, "inbox overflow on a peer worker");
      view.reports = reports;
      it_edges = it_comb = 0;
      for (uint32_t q = 0; q < n; ++q) {
        it_edges += reports[q].edges_delta;
        it_comb += reports[q].combine_delta;
        if (q == me) continue;
        h_src[q] = 0;
        for (uint32_t d = 0; d < n; ++d) {
          if (d == q) continue;
          P.h_matrix[q][d] += sends[q][d];
          h_src[q] += sends[q][d];
        }
      }
    }
    for (auto& r : view.reports) {
      view.total_out += r.out_frontier;
      view.total_next += r.next_frontier;
    }
    view.inflight_records = 0;  // every delivered slot was merged this superstep
    P.out_per_iter.push_back(view.total_out);
    P.h_per_iter.push_back(h_src);
    P.edges_per_iter.push_back(it_edges);
    P.combine_per_iter.push_back(it_comb);
    total_edges += it_edges;
    total_combine += it_comb;
    bool stop = false;
    if (iter + 1 >= cfg.max_supersteps) {
      stop = true;
      stop_reason = MG_STOP_MAX_SUPERSTEPS;
    } else {
      bool conv = prim.has_stop_condition ? prim.stop_condition(view)
                                          : (view.total_next == 0 && view.inflight_records == 0);
      if (conv) {
        stop = true;
        stop_reason = prim.has_stop_condition ? MG_STOP_CONDITION : MG_STOP_FRONTIERS_EMPTY;
      }
    }
    rs.views.push_back(std::move(view));
    trace("report done", iter);
    if (stop) break;
  }
  for (uint32_t p : P.local_workers) {
    Worker& w = *P.workers[p];
    DeviceGuard dg(w.dev);
    prim.finalize(ctx[p], rs.views.back());
    MGB_CUDA(cudaEventRecord(w.ev_end, w.stream));
  }
  double dev_ms = 0;
  for (uint32_t p : P.local_workers) {
    Worker& w = *P.workers[p];
    MGB_CUDA(cudaEventSynchronize(w.ev_end));
    float ms = 0;
    cudaEventElapsedTime(&ms, w.ev_start, w.ev_end);
    if (ms > dev_ms) dev_ms = ms;
  }
  auto t1 = std::chrono::steady_clock::now();
  mg_stats& st = P.last;
  st.n = n;
  st.stop_reason = stop_reason;
  st.communication = comm;
  st.policy = cfg.policy;
  st.supersteps = rs.views.size();
  st.edges_examined = total_edges;
  st.combine_ops = total_combine;
  uint64_t h = 0;
  for (auto& row : P.h_matrix)
    for (auto v : row) h += v;
  st.h_total = h;
  st.wire_records = wire;
  st.wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  st.device_ms = dev_ms;
  st.gpu_launches = g_launches.load() - launches0;
  st.exchange_bytes = xbytes;
  st.kernel_ms = P.prof_ms;
  st.kernel_launches = P.prof_launches;
  st.kernel_bytes = P.prof_bytes;
  st.kernel2_ms = P.prof2_ms;
  st.kernel2_launches = P.prof2_launches;
  st.kernel2_bytes = P.prof2_bytes;
  st.device_loop = on_device ? 1 : 0;
  collect_buffer_stats(P);
}

}  // namespace mgb
