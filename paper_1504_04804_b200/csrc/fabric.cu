// fabric.cu — multi-process exchange fabric (one process per GPU, e.g. under
// torchrun).  Each rank owns exactly one worker.  At the start of every run
// the ranks all-gather (through the shared-memory rendezvous, shm_fabric.hpp)
// the CUDA IPC handles of their inbox arenas and slot counters plus the slot
// layout; each rank maps its peers' arenas once per arena generation.  The
// pack kernels then store records straight into the mapped peer HBM over
// NVLink — the reference's ExchangeFabric::deliver (engine.hpp:361-391) —
// and the per-superstep barrier + WorkerReport all-gather reproduce
// Barrier/completion (engine.hpp:449-473, :784-820) across processes.
#include <cstring>
#include <functional>
#include <memory>

#include "engine.cuh"

namespace mgb {
int run_guarded(const std::function<void()>& f);
Plan* plan_from_host(const HostPlan& H, const int* devices, std::shared_ptr<HostCsr> g, int only);
Plan* plan_from_device_csr(uint32_t nv, uint64_t ne, DevArray<uint32_t>& goff,
                           DevArray<uint32_t>& gcol, DevArray<uint32_t>& gw,
                           const std::vector<uint32_t>& owner, uint32_t n, const int* devices,
                           int only);
void device_rmat_csr(int dev, int scale, int ef, uint64_t seed, int with_w, uint32_t lo,
                     uint32_t hi, uint64_t wseed, DevArray<uint32_t>& off, DevArray<uint32_t>& col,
                     DevArray<uint32_t>& w, uint64_t* ne_out);

namespace {


struct SlotOff {
  uint64_t ids, va[kMaxAssoc], vv[kMaxAssoc], cap;
};

struct AttachBlob {
  uint64_t gen;
  uint32_t has_arena, pad;
  cudaIpcMemHandle_t arena;
  cudaIpcMemHandle_t cnt;
  cudaIpcMemHandle_t mbox;
  SlotOff slots[2][kMaxMpRanks];  // [parity][src] in this rank's arena
};
static_assert(sizeof(AttachBlob) <= ShmFabric::kBlobBytes, "attach blob too large");

uint64_t rel(const void* p, const void* base) {
  return p ? static_cast<uint64_t>(static_cast<const uint8_t*>(p) -
                                   static_cast<const uint8_t*>(base))
           : ~0ull;
}

template <class T>
T* at(void* base, uint64_t off) {
  return off == ~0ull ? nullptr : reinterpret_cast<T*>(static_cast<uint8_t*>(base) + off);
}

}  // namespace

// collective: every rank of a multi-process plan calls it at the start of a
// run, after its inbox arena has been sized for the primitive
void fabric_sync(Plan& P) {
  const uint32_t n = P.n, me = P.rank;
  Worker& w = *P.workers[me];
  DeviceGuard dg(w.dev);
  if (!P.mbox.ptr) {  // device-side protocol state, once per plan
    P.mbox.alloc(sizeof(Mailbox));
    MGB_CUDA(cudaMemset(P.mbox.ptr, 0, sizeof(Mailbox)));
    MGB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&P.host_reports),
                           sizeof(DevReport) * (kMaxMpRanks + 1),
                           cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(P.host_reports, 0, sizeof(DevReport) * (kMaxMpRanks + 1));
    MGB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&P.host_reports_dev),
                                      P.host_reports, 0));
    P.device_fabric = getenv("MG_HOST_FABRIC") == nullptr;
  }
  AttachBlob mine;
  std::memset(&mine, 0, sizeof(mine));
  MGB_CUDA(cudaIpcGetMemHandle(&mine.mbox, P.mbox.ptr));
  mine.gen = w.arena_gen;
  mine.has_arena = w.arena.ptr ? 1 : 0;
  if (w.arena.ptr) MGB_CUDA(cudaIpcGetMemHandle(&mine.arena, w.arena.ptr));
  MGB_CUDA(cudaIpcGetMemHandle(&mine.cnt, w.inbox_cnt.ptr));
  for (int par = 0; par < 2; ++par)
    for (uint32_t s = 0; s < n; ++s) {
      const SlotView& v = w.slots[par][s];
      SlotOff& o = mine.slots[par][s];
      o.ids = rel(v.ids, w.arena.ptr);
      for (int a = 0; a < kMaxAssoc; ++a) {
        o.va[a] = rel(v.va[a], w.arena.ptr);
        o.vv[a] = rel(v.vv[a], w.arena.ptr);
      }
      o.cap = v.cap;
    }
  std::vector<AttachBlob> all(n);
  P.shm->allgather(&mine, sizeof(AttachBlob), all.data());
  if (P.peer_arena.empty()) {
    P.peer_arena.assign(n, nullptr);
    P.peer_cnt.assign(n, nullptr);
    P.peer_gen.assign(n, ~0ull);
    P.peer_slots.assign(2 * n, SlotView{});
    P.peer_mbox.assign(n, nullptr);
  }
  for (uint32_t q = 0; q < n; ++q) {
    if (q == me) continue;
    const AttachBlob& b = all[q];
    if (!P.peer_cnt[q])
      MGB_CUDA(cudaIpcOpenMemHandle(&P.peer_cnt[q], b.cnt, cudaIpcMemLazyEnablePeerAccess));
    if (!P.peer_mbox[q])
      MGB_CUDA(cudaIpcOpenMemHandle(&P.peer_mbox[q], b.mbox, cudaIpcMemLazyEnablePeerAccess));
    if (P.peer_gen[q] != b.gen) {
      if (P.peer_arena[q]) MGB_CUDA(cudaIpcCloseMemHandle(P.peer_arena[q]));
      P.peer_arena[q] = nullptr;
      if (b.has_arena)
        MGB_CUDA(cudaIpcOpenMemHandle(&P.peer_arena[q], b.arena, cudaIpcMemLazyEnablePeerAccess));
      P.peer_gen[q] = b.gen;
    }
    for (int par = 0; par < 2; ++par) {
      const SlotOff& o = b.slots[par][me];  // q's slot that receives from me
      SlotView v{};
      v.cap = o.cap;
      if (P.peer_arena[q]) {
        v.ids = at<uint32_t>(P.peer_arena[q], o.ids);
        for (int a = 0; a < kMaxAssoc; ++a) {
          v.va[a] = at<uint32_t>(P.peer_arena[q], o.va[a]);
          v.vv[a] = at<double>(P.peer_arena[q], o.vv[a]);
        }
      } else {
        v.cap = 0;
      }
      P.peer_slots[par * n + q] = v;
    }
  }
  if (!P.mbox_ptrs.ptr) {
    std::vector<Mailbox*> ptrs(n);
    for (uint32_t q = 0; q < n; ++q)
      ptrs[q] = reinterpret_cast<Mailbox*>(q == me ? (void*)P.mbox.ptr : P.peer_mbox[q]);
    P.mbox_ptrs.upload(ptrs.data(), n, w.stream);
    MGB_CUDA(cudaStreamSynchronize(w.stream));
  }
}

// per-superstep report exchange: this rank's WorkerReport + send counts
struct ReportBlob {
  uint64_t out_frontier, next_frontier, edges_delta, combine_delta;
  double f[4];
  uint64_t u[4];
  uint32_t send_cnt[kMaxMpRanks];
  uint32_t overflow, pad;
};

void fabric_exchange_reports(Plan& P, const WorkerReport& r, const Counters& c,
                             std::vector<WorkerReport>& reports,
                             std::vector<std::vector<uint32_t>>& sends, bool& overflow) {
  const uint32_t n = P.n;
  ReportBlob mine;
  std::memset(&mine, 0, sizeof(mine));
  mine.out_frontier = r.out_frontier;
  mine.next_frontier = r.next_frontier;
  mine.edges_delta = r.edges_delta;
  mine.combine_delta = r.combine_delta;
  for (int k = 0; k < 4; ++k) {
    mine.f[k] = r.f[k];
    mine.u[k] = r.u[k];
  }
  for (uint32_t q = 0; q < n && q < kMaxMpRanks; ++q) mine.send_cnt[q] = c.send_cnt[q];
  mine.overflow = c.overflow;
  std::vector<ReportBlob> all(n);
  P.shm->allgather(&mine, sizeof(ReportBlob), all.data());
  reports.assign(n, WorkerReport{});
  sends.assign(n, std::vector<uint32_t>(n, 0));
  overflow = false;
  for (uint32_t q = 0; q < n; ++q) {
    WorkerReport& x = reports[q];
    x.out_frontier = all[q].out_frontier;
    x.next_frontier = all[q].next_frontier;
    x.edges_delta = all[q].edges_delta;
    x.combine_delta = all[q].combine_delta;
    for (int k = 0; k < 4; ++k) {
      x.f[k] = all[q].f[k];
      x.u[k] = all[q].u[k];
    }
    for (uint32_t d = 0; d < n; ++d) sends[q][d] = all[q].send_cnt[d] & ~kDenseFlag;
    overflow |= all[q].overflow != 0;
  }
}

}  // namespace mgb

using namespace mgb;

extern "C" {

int mg_plan_create_mp(const mg_graph* g, const uint32_t* owner, uint32_t n, int dup,
                      uint32_t rank, int device, const char* key, mg_plan** out) {
  return run_guarded([&] {
    if (!key || !*key) throw Error(MG_EINVAL, "mg_plan_create_mp: empty fabric key");
    if (n < 2 || n > kMaxMpRanks || rank >= n)
      throw Error(MG_EINVAL, "mg_plan_create_mp: need 2 <= n <= 32 and rank < n");
    if (!g) throw Error(MG_EINVAL, "mg_plan_create_mp: null graph");
    const std::shared_ptr<HostCsr>& gp = g->g;
    std::vector<uint32_t> own(owner, owner + gp->nv);
    HostPlan H = build_plan(*gp, own, n, dup);
    std::vector<int> devs(n, device);
    Plan* P = plan_from_host(H, devs.data(), gp, (int)rank);
    try {
      P->shm = std::make_unique<ShmFabric>(key, rank, n);
    } catch (...) {
      plan_free(P);
      throw;
    }
    *out = reinterpret_cast<mg_plan*>(P);
  });
}

int mg_plan_create_rmat_device_mp(int scale, int ef, uint64_t seed, int with_w, uint32_t lo,
                                  uint32_t hi, uint64_t wseed, const uint32_t* owner, uint32_t n,
                                  uint32_t rank, int device, const char* key, mg_plan** out) {
  return run_guarded([&] {
    if (!key || !*key) throw Error(MG_EINVAL, "mg_plan_create_rmat_device_mp: empty key");
    if (n < 2 || n > kMaxMpRanks || rank >= n || !owner)
      throw Error(MG_EINVAL, "mg_plan_create_rmat_device_mp: need owner, 2 <= n <= 32");
    const uint32_t nv = 1u << scale;
    std::vector<uint32_t> own(owner, owner + nv);
    for (uint32_t o : own)
      if (o >= n) throw Error(MG_EINVAL, "build_partition_plan: owner out of range");
    DevArray<uint32_t> off, col, w;
    uint64_t ne = 0;
    device_rmat_csr(device, scale, ef, seed, with_w, lo, hi, wseed, off, col, w, &ne);
    std::vector<int> devs(n, device);
    Plan* P = plan_from_device_csr(nv, ne, off, col, w, own, n, devs.data(), (int)rank);
    try {
      P->shm = std::make_unique<ShmFabric>(key, rank, n);
    } catch (...) {
      plan_free(P);
      throw;
    }
    *out = reinterpret_cast<mg_plan*>(P);
  });
}

int mg_fabric_selftest(const char* key, uint32_t rank, uint32_t world, uint32_t rounds) {
  return run_guarded([&] {
    ShmFabric f(key, rank, world, 60.0);
    std::vector<uint64_t> got(world);
    for (uint32_t r = 0; r < rounds; ++r) {
      uint64_t mine = (uint64_t)r * 1000003ull + rank;
      f.allgather(&mine, sizeof(mine), got.data());
      for (uint32_t q = 0; q < world; ++q)
        if (got[q] != (uint64_t)r * 1000003ull + q)
          throw Error(MG_EWORKER, "fabric selftest: wrong value from rank " + std::to_string(q));
      f.barrier();
    }
  });
}

}  // extern "C"
