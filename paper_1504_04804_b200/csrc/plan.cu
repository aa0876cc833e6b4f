// plan.cu — device plan construction (upload of build_partition_plan's
// sub-graphs), inbox arenas, per-run worker preparation and result gathering.
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "engine.cuh"

namespace mgb {

__global__ void max_u32_kernel(const uint32_t* __restrict__ a, uint64_t n, uint32_t* out) {
  uint32_t m = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    m = a[i] > m ? a[i] : m;
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

uint32_t device_max_u32(const uint32_t* a, uint64_t n) {
  DevArray<uint32_t> o;
  o.alloc(1);
  MGB_CUDA(cudaMemset(o.ptr, 0, 4));
  if (n) MGB_LAUNCH(max_u32_kernel, num_sms() * 8, 256, 0, 0, a, n, o.ptr);
  uint32_t h = 0;
  MGB_CUDA(cudaMemcpy(&h, o.ptr, 4, cudaMemcpyDeviceToHost));
  return h;
}

std::atomic<uint64_t> g_launches{0};

Worker& worker(Plan& P, uint32_t p) { return *P.workers[p]; }

static void free_worker(Worker& w) {
  DeviceGuard dg(w.dev);
  cudaDeviceSynchronize();
  w.off.free_(); w.col.free_(); w.w.free_(); w.hosted.free_(); w.owner.free_(); w.l2g.free_();
  w.border.free_(); w.border_dst.free_();
  w.input.release(); w.next_input.release(); w.advance_out.release(); w.output.release();
  w.merge_stamp.free_(); w.lb_row.free_(); w.lb_pref.free_(); w.lb_bsum.free_(); w.lb_tile.free_(); w.arena.free_();
  w.inbox_cnt.free_(); w.send_table.free_(); w.send_cnt_ptr.free_(); w.recv_table.free_(); w.ctr.free_();
  for (auto& a : w.su32) a.free_();
  for (auto& a : w.sf64) a.free_();
  for (auto& a : w.su64) a.free_();
  for (auto& a : w.aux) a.free_();
  w.nonisolated.free_();
  w.pull_rec.free_();
  w.pull_ext.free_();
  for (auto& a : w.ul_buf) a.free_();
  for (int i = 0; i < 2; ++i)
    if (w.loop_exec[i]) cudaGraphExecDestroy(w.loop_exec[i]);
  if (w.mp_exec) cudaGraphExecDestroy(w.mp_exec);
  w.mp_state.free_(); w.mp_hist.free_();
  w.dobfs_lastvis.free_();
  if (w.loop_host) cudaFreeHost(w.loop_host);
  if (w.loop_hist_host) cudaFreeHost(w.loop_hist_host);
  w.loop_state.free_(); w.loop_hist.free_(); w.loop_front[0].free_(); w.loop_front[1].free_();
  w.loop_lb_row.free_(); w.loop_tiles.free_(); w.loop_lb_pref.free_(); w.loop_lb_bsum.free_();
  w.loop_total.free_();
  w.toff.free_(); w.tcol.free_(); w.tlong.free_();
  w.pr_perm.free_(); w.pr_pdeg.free_(); w.pr_iperm.free_();
  w.bc_acc.free_();
  if (w.host_ctr) cudaFreeHost(w.host_ctr);
  if (w.stream) cudaStreamDestroy(w.stream);
  for (cudaEvent_t e : {w.ev_start, w.ev_end, w.ev_x0, w.ev_x1, w.ev_k0, w.ev_k1})
    if (e) cudaEventDestroy(e);
}

void plan_free(Plan* P) {
  if (!P) return;
  if (P->shm) {
    // peers may still be writing into this rank's inboxes: free only after
    // every rank stopped using the fabric
    try {
      for (uint32_t p : P->local_workers) cudaStreamSynchronize(P->workers[p]->stream);
      P->shm->barrier();
    } catch (...) {
    }
  }
  for (auto& w : P->workers)
    if (w) free_worker(*w);
  for (size_t i = 0; i < P->peer_arena.size(); ++i)
    if (P->peer_arena[i]) cudaIpcCloseMemHandle(P->peer_arena[i]);
  for (size_t i = 0; i < P->peer_cnt.size(); ++i)
    if (P->peer_cnt[i]) cudaIpcCloseMemHandle(P->peer_cnt[i]);
  for (size_t i = 0; i < P->peer_mbox.size(); ++i)
    if (P->peer_mbox[i]) cudaIpcCloseMemHandle(P->peer_mbox[i]);
  P->mbox.free_();
  P->mbox_ptrs.free_();
  if (P->host_reports) cudaFreeHost(P->host_reports);
  P->g_off.free_(); P->g_col.free_(); P->g_w.free_();
  if (P->label_stage) cudaFreeHost(P->label_stage);
  P->label_dev.free_();
  P->pool.reset();
  delete P;
}

void init_worker_runtime(Worker& w) {
  DeviceGuard dg(w.dev);
  MGB_CUDA(cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking));
  MGB_CUDA(cudaEventCreate(&w.ev_start));
  MGB_CUDA(cudaEventCreate(&w.ev_end));
  MGB_CUDA(cudaEventCreate(&w.ev_x0));
  MGB_CUDA(cudaEventCreate(&w.ev_x1));
  MGB_CUDA(cudaEventCreate(&w.ev_k0));
  MGB_CUDA(cudaEventCreate(&w.ev_k1));
  w.ctr.alloc(1);
  MGB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&w.host_ctr), sizeof(Counters),
                         cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(w.host_ctr, 0, sizeof(Counters));
  MGB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&w.host_ctr_dev), w.host_ctr, 0));
  w.inbox_cnt.alloc(2 * kMaxWorkers);
  MGB_CUDA(cudaMemset(w.inbox_cnt.ptr, 0, sizeof(uint32_t) * 2 * kMaxWorkers));
  w.merge_stamp.alloc(w.nv ? w.nv : 1);
}

// Upload one partition of a host plan (partition.cpp:157-207 layout)
static void upload_worker(Plan& P, const HostPlan& H, uint32_t p) {
  auto wp = std::make_unique<Worker>();
  Worker& w = *wp;
  w.p = p;
  w.dev = P.devices[p];
  DeviceGuard dg(w.dev);
  const HostCsr& s = H.sub[p];
  w.nv = s.nv;
  w.ne = s.ne();
  w.nlocal = static_cast<uint32_t>(H.locals[p].size());
  init_worker_runtime(w);
  w.off.upload(s.off.data(), s.off.size(), w.stream);
  w.col.upload(s.col.data(), s.col.size(), w.stream);
  if (s.weighted()) w.w.upload(s.w.data(), s.w.size(), w.stream);
  std::vector<uint8_t> own8(H.owner.begin(), H.owner.end());
  w.owner.upload(own8.data(), own8.size(), w.stream);
  if (H.dup == MG_DUP_ALL) {
    w.hosted_host = H.locals[p];
  } else {
    w.hosted_host.resize(w.nlocal);
    std::iota(w.hosted_host.begin(), w.hosted_host.end(), 0u);
    w.l2g.upload(H.l2g[p].data(), H.l2g[p].size(), w.stream);
  }
  w.hosted.upload(w.hosted_host.data(), w.hosted_host.size(), w.stream);
  // static border sub-frontier (PR, primitives.cpp:735-744): local IDs on p,
  // grouped by peer, plus each entry's ID in the destination's local space
  std::vector<uint32_t> border, dst;
  w.border_len.assign(P.n, 0);
  w.border_off.assign(P.n, 0);
  for (uint32_t q = 0; q < P.n; ++q) {
    w.border_off[q] = border.size();
    if (q == p) continue;
    for (uint32_t g : H.borders[p][q]) {
      border.push_back(H.dup == MG_DUP_ALL ? g : H.g2l[p][g]);
      dst.push_back(H.dup == MG_DUP_ALL ? g : H.g2l[q][g]);
    }
    w.border_len[q] = H.borders[p][q].size();
  }
  w.border.upload(border.data(), border.size(), w.stream);
  w.border_dst.upload(dst.data(), dst.size(), w.stream);
  MGB_CUDA(cudaStreamSynchronize(w.stream));
  P.workers[p] = std::move(wp);
}

// only >= 0: multi-process mode, upload partition `only` to devices[only]
Plan* plan_from_host(const HostPlan& H, const int* devices, std::shared_ptr<HostCsr> g,
                     int only) {
  if (H.n > 255 || H.n > kMaxWorkers)
    throw Error(MG_EINVAL, "mg_plan_create: at most 64 partitions are supported");
  int ndev = 0;
  MGB_CUDA(cudaGetDeviceCount(&ndev));
  auto P = new Plan();
  try {
    P->n = H.n;
    P->dup = H.dup;
    P->nv = H.nv;
    P->ne = H.ne;
    P->weighted = g ? g->weighted() : false;
    if (P->weighted)
      for (uint32_t x : g->w) P->max_weight = x > P->max_weight ? x : P->max_weight;
    P->owner_host = H.owner;
    P->host_graph = g;
    P->devices.resize(H.n);
    for (uint32_t p = 0; p < H.n; ++p) {
      P->devices[p] = devices ? devices[p] : 0;
      if ((only < 0 || (int)p == only) && (P->devices[p] < 0 || P->devices[p] >= ndev))
        throw Error(MG_EINVAL, "mg_plan_create: device ordinal out of range");
    }
    if (only >= 0) {
      P->multiprocess = true;
      P->rank = (uint32_t)only;
      P->world = H.n;
    }
    P->workers.resize(H.n);
    P->pair_border.assign(H.n, std::vector<uint64_t>(H.n, 0));
    P->nlocal.assign(H.n, 0);
    for (uint32_t i = 0; i < H.n; ++i) {
      P->nlocal[i] = H.locals[i].size();
      for (uint32_t j = 0; j < H.n; ++j) P->pair_border[i][j] = H.borders[i][j].size();
    }
    // enable peer access between distinct devices used by this plan
    for (uint32_t a = 0; a < H.n && only < 0; ++a)
      for (uint32_t b = 0; b < H.n; ++b) {
        int da = P->devices[a], db = P->devices[b];
        if (da == db) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, da, db);
        if (can) {
          DeviceGuard dg(da);
          cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            throw Error(MG_ECUDA, "cudaDeviceEnablePeerAccess failed");
          cudaGetLastError();
        }
      }
    for (uint32_t p = 0; p < H.n; ++p) {
      if (only >= 0 && (int)p != only) continue;
      upload_worker(*P, H, p);
      P->local_workers.push_back(p);
    }
  } catch (...) {
    plan_free(P);
    throw;
  }
  return P;
}

// ---------------------------------------------------------------------------
// inbox arenas

void ensure_inboxes(Plan& P, Worker& w, int nva, int nvv, const std::vector<uint64_t>& caps) {
  bool fits = nva <= w.nva && nvv <= w.nvv && w.slot_cap.size() == caps.size();
  if (fits)
    for (size_t s = 0; s < caps.size(); ++s)
      if (caps[s] > w.slot_cap[s]) fits = false;
  if (fits) return;
  DeviceGuard dg(w.dev);
  MGB_CUDA(cudaStreamSynchronize(w.stream));
  int ka = nva > w.nva ? nva : w.nva, kv = nvv > w.nvv ? nvv : w.nvv;
  std::vector<uint64_t> newcap(caps.size());
  for (size_t s = 0; s < caps.size(); ++s) {
    uint64_t have = s < w.slot_cap.size() ? w.slot_cap[s] : 0;
    newcap[s] = caps[s] > have ? caps[s] : have;
  }
  uint64_t tot = 0;
  for (uint64_t c : newcap) tot += c;
  if (tot == 0) {  // single worker: no peers, no inbox memory
    std::memset(w.slots, 0, sizeof(w.slots));
    w.slot_cap = newcap;
    w.nva = ka;
    w.nvv = kv;
    return;
  }
  uint64_t per_rec = 4 + 4ull * ka + 8ull * kv;
  uint64_t bytes = 0;
  for (int par = 0; par < 2; ++par)
    for (size_t s = 0; s < caps.size(); ++s) bytes += ((newcap[s] * per_rec + 255) / 256) * 256 + 256 * (1 + ka + kv);
  // inbox memory is charged to the receiving worker's budget (engine.hpp:340-344)
  w.budget.charge(bytes, w.arena.n);
  w.arena.alloc(bytes ? bytes : 256);
  ++w.arena_gen;
  uint8_t* base = w.arena.ptr;
  auto carve = [&](uint64_t b) {
    uint8_t* r = base;
    base += ((b + 255) / 256) * 256;
    return r;
  };
  std::memset(w.slots, 0, sizeof(w.slots));
  for (int par = 0; par < 2; ++par)
    for (size_t s = 0; s < caps.size(); ++s) {
      SlotView& v = w.slots[par][s];
      v.cap = newcap[s];
      v.ids = reinterpret_cast<uint32_t*>(carve(newcap[s] * 4));
      for (int a = 0; a < ka; ++a) v.va[a] = reinterpret_cast<uint32_t*>(carve(newcap[s] * 4));
      for (int a = 0; a < kv; ++a) v.vv[a] = reinterpret_cast<double*>(carve(newcap[s] * 8));
    }
  w.slot_cap = newcap;
  w.nva = ka;
  w.nvv = kv;
  w.stats[MG_ROLE_INBOX].peak_bytes =
      w.stats[MG_ROLE_INBOX].peak_bytes > bytes ? w.stats[MG_ROLE_INBOX].peak_bytes : bytes;
}

void build_send_tables(Plan& P) {
  const uint32_t n = P.n;
  for (uint32_t p : P.local_workers) {
    Worker& w = *P.workers[p];
    DeviceGuard dg(w.dev);
    std::vector<SlotView> table(2 * n);
    std::vector<uint32_t*> cnt(2 * n, nullptr);
    for (int par = 0; par < 2; ++par)
      for (uint32_t q = 0; q < n; ++q) {
        if (q == p) continue;
        if (P.shm) {  // peer in another process: IPC mappings (fabric.cu)
          table[par * n + q] = P.peer_slots[par * n + q];
          cnt[par * n + q] =
              static_cast<uint32_t*>(P.peer_cnt[q]) + par * kMaxWorkers + p;
          continue;
        }
        Worker& d = *P.workers[q];
        table[par * n + q] = d.slots[par][p];
        cnt[par * n + q] = d.inbox_cnt.ptr + par * kMaxWorkers + p;
      }
    std::vector<SlotView> recv(2 * n);
    for (int par = 0; par < 2; ++par)
      for (uint32_t s = 0; s < n; ++s) recv[par * n + s] = w.slots[par][s];
    // the tables change only when an arena is (re)mapped: skip the three
    // synchronous uploads when the device copies are already current
    std::vector<uint8_t> sig(sizeof(SlotView) * 4 * n + sizeof(uint32_t*) * 2 * n);
    std::memcpy(sig.data(), table.data(), sizeof(SlotView) * 2 * n);
    std::memcpy(sig.data() + sizeof(SlotView) * 2 * n, recv.data(), sizeof(SlotView) * 2 * n);
    std::memcpy(sig.data() + sizeof(SlotView) * 4 * n, cnt.data(), sizeof(uint32_t*) * 2 * n);
    if (sig == w.table_sig && w.send_table.ptr) continue;
    if (!w.send_table.ptr || w.send_table.n != 2 * n) w.send_table.alloc(2 * n);
    if (!w.send_cnt_ptr.ptr || w.send_cnt_ptr.n != 2 * n) w.send_cnt_ptr.alloc(2 * n);
    MGB_CUDA(cudaMemcpy(w.send_table.ptr, table.data(), sizeof(SlotView) * 2 * n,
                        cudaMemcpyHostToDevice));
    MGB_CUDA(cudaMemcpy(w.send_cnt_ptr.ptr, cnt.data(), sizeof(uint32_t*) * 2 * n,
                        cudaMemcpyHostToDevice));
    if (!w.recv_table.ptr || w.recv_table.n != 2 * n) w.recv_table.alloc(2 * n);
    MGB_CUDA(cudaMemcpy(w.recv_table.ptr, recv.data(), sizeof(SlotView) * 2 * n,
                        cudaMemcpyHostToDevice));
    w.table_sig = std::move(sig);
  }
}

// AllocationPolicy preallocation (engine.hpp:666-700) + per-run reset
void prepare_worker(Plan& P, Worker& w, const mg_config& cfg) {
  DeviceGuard dg(w.dev);
  for (auto& s : w.stats) s = BufferStats{};
  w.budget.hard_cap = cfg.hard_cap_bytes;
  w.budget.peak = w.budget.allocated;
  w.input.attach(&w.stats[MG_ROLE_INPUT_FRONTIER], &w.budget);
  w.next_input.attach(&w.stats[MG_ROLE_INPUT_FRONTIER], &w.budget);
  w.advance_out.attach(&w.stats[MG_ROLE_ADVANCE_OUTPUT], &w.budget);
  w.output.attach(&w.stats[MG_ROLE_FILTER_OUTPUT], &w.budget);
  // every run starts from empty frontier buffers so the policy's growth
  // behaviour (and its realloc counts) is observable per run
  w.input.reset(); w.next_input.reset(); w.advance_out.reset(); w.output.reset();
  w.budget.allocated = w.arena.n;
  w.budget.peak = w.budget.allocated;
  if (cfg.hard_cap_bytes && w.budget.allocated > cfg.hard_cap_bytes)
    w.budget.charge(0, 0);  // throws CapacityError
  const uint64_t E = w.ne, V = w.nv;
  auto items = [](double f, uint64_t unit) {
    return static_cast<uint64_t>(f * static_cast<double>(unit) + 0.9999);
  };
  switch (cfg.policy) {
    case MG_POLICY_MAX: {
      w.advance_out.prealloc(E, w.stream);
      w.output.prealloc(V, w.stream);
      w.input.prealloc(V, w.stream);
      w.next_input.prealloc(V, w.stream);
      // the advance's load-balancing scratch at its bound too, so no run of a
      // max-policy plan allocates inside its superstep loop
      const uint64_t nb = (V + kLbBlock - 1) / kLbBlock;
      const uint64_t tiles = (2 * E + 1) / kTile + 2 + kMinTiles + 1;
      if (w.lb_row.n < V) w.lb_row.alloc(V ? V : 1);
      if (w.lb_pref.n < V) w.lb_pref.alloc(V ? V : 1);
      if (w.lb_bsum.n < nb + 1) w.lb_bsum.alloc(nb + 1);
      if (w.lb_tile.n < tiles) w.lb_tile.alloc(tiles);
      break;
    }
    case MG_POLICY_FIXED:
    case MG_POLICY_FUSED:
      w.advance_out.prealloc(items(cfg.factors[MG_ROLE_ADVANCE_OUTPUT], E), w.stream);
      w.output.prealloc(items(cfg.factors[MG_ROLE_FILTER_OUTPUT], V), w.stream);
      w.input.prealloc(items(cfg.factors[MG_ROLE_INPUT_FRONTIER], V), w.stream);
      w.next_input.prealloc(items(cfg.factors[MG_ROLE_INPUT_FRONTIER], V), w.stream);
      break;
    default:
      break;
  }
}

void collect_buffer_stats(Plan& P) {
  P.last_buffers.assign(P.n, std::vector<BufferStats>(MG_NUM_ROLES));
  uint64_t peak = 0, reallocs = 0;
  for (uint32_t p : P.local_workers) {
    Worker& w = *P.workers[p];
    for (int r = 0; r < MG_NUM_ROLES; ++r) {
      P.last_buffers[p][r] = w.stats[r];
      reallocs += w.stats[r].realloc_count;
    }
    peak += w.budget.peak;
  }
  P.last.peak_bytes = peak;
  P.last.reallocs = reallocs;
}

// ---------------------------------------------------------------------------
// results: gather each worker's hosted values into global-ID host arrays
// (gather_hosted, primitives.cpp:33-41)

template <class T>
__global__ void compact_hosted_kernel(const T* __restrict__ src, const uint32_t* __restrict__ hosted,
                                      uint32_t n, T* __restrict__ dst) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = src[hosted[i]];
}

template <class T>
void gather_result_t(Plan& P, const std::vector<const T*>& per_worker, T* host_out) {
  if (!host_out) return;
  for (uint32_t p : P.local_workers) {
    Worker& w = *P.workers[p];
    DeviceGuard dg(w.dev);
    const T* src = per_worker[p];
    if (P.n == 1 && P.dup == MG_DUP_ALL) {
      P.last_d2h_bytes += sizeof(T) * (uint64_t)w.nv;
      MGB_CUDA(cudaMemcpyAsync(host_out, src, sizeof(T) * w.nv, cudaMemcpyDeviceToHost, w.stream));
      MGB_CUDA(cudaStreamSynchronize(w.stream));
      continue;
    }
    uint32_t nh = static_cast<uint32_t>(w.hosted_host.size());
    if (nh == 0) continue;
    T* tmp = nullptr;
    MGB_CUDA(cudaMallocAsync(&tmp, sizeof(T) * nh, w.stream));
    MGB_LAUNCH(compact_hosted_kernel<T>, grid_for(nh, 256, 4096), 256, 0, w.stream, src,
               w.hosted.ptr, nh, tmp);
    std::vector<T> h(nh);
    P.last_d2h_bytes += sizeof(T) * (uint64_t)nh;
    MGB_CUDA(cudaMemcpyAsync(h.data(), tmp, sizeof(T) * nh, cudaMemcpyDeviceToHost, w.stream));
    MGB_CUDA(cudaFreeAsync(tmp, w.stream));
    MGB_CUDA(cudaStreamSynchronize(w.stream));
    const uint32_t* l2g = nullptr;
    std::vector<uint32_t> glob;
    if (P.dup == MG_DUP_ONEHOP) {
      // hosted local l -> global: locals sorted, stored as owner scan
      glob.reserve(nh);
      for (uint32_t g = 0; g < P.nv; ++g)
        if (P.owner_host[g] == p) glob.push_back(g);
      l2g = glob.data();
    }
    for (uint32_t i = 0; i < nh; ++i) {
      uint32_t gid = l2g ? l2g[i] : w.hosted_host[i];
      host_out[gid] = h[i];
    }
  }
}

void gather_u32(Plan& P, const std::vector<const uint32_t*>& pw, uint32_t* out) {
  gather_result_t(P, pw, out);
}

// ---------------------------------------------------------------------------
// Level-array download (BFS/DOBFS labels, single partition): PCIe, not the
// GPU, bounds the result copy (268 MB at RMAT-26: ~4.7 ms vs ~1.3 ms of
// traversal).  Labels below 255 fit a byte, so the tail of the array crosses
// PCIe as bytes and the host widens it with a thread pool while the head
// still streams in as u32: the two halves finish together (~2.9 ms).

__global__ void narrow_labels_kernel(const uint32_t* __restrict__ lab, uint32_t n, uint8_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t l = lab[i];
    out[i] = l == kInfLabel ? (uint8_t)255 : (uint8_t)l;
  }
}

// two levels per byte (15 = unreached) when every level is below 15
__global__ void narrow_labels_nib_kernel(const uint32_t* __restrict__ lab, uint32_t n,
                                         uint8_t* out) {
  const uint32_t np = (n + 1) / 2;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
    const uint32_t a = lab[2 * i], b = 2 * i + 1 < n ? lab[2 * i + 1] : kInfLabel;
    out[i] = (uint8_t)((a == kInfLabel ? 15u : a) | ((b == kInfLabel ? 15u : b) << 4));
  }
}

HostPool::HostPool(unsigned n) : n_(n ? n : 1) {
  for (unsigned t = 0; t < n_; ++t)
    threads_.emplace_back([this, t] {
      uint64_t seen = 0;
      for (;;) {
        std::function<void(unsigned, unsigned)> job;
        {
          std::unique_lock<std::mutex> lk(m_);
          cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
          if (stop_) return;
          seen = gen_;
          job = job_;
        }
        job(t, n_);
        {
          std::lock_guard<std::mutex> lk(m_);
          if (--pending_ == 0) done_.notify_all();
        }
      }
    });
}

HostPool::~HostPool() {
  {
    std::lock_guard<std::mutex> lk(m_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : threads_) t.join();
}

void HostPool::run(const std::function<void(unsigned, unsigned)>& f) {
  std::unique_lock<std::mutex> lk(m_);
  job_ = f;
  pending_ = n_;
  ++gen_;
  cv_.notify_all();
  done_.wait(lk, [&] { return pending_ == 0; });
}

void gather_labels_u32(Plan& P, const std::vector<const uint32_t*>& pw, uint32_t* out,
                       uint64_t max_label) {
  if (!out) return;
  const char* env = getenv("MG_D2H_SPLIT");
  const double head = env ? atof(env) : 0.5;  // fraction copied as u32
  if (!(P.n == 1 && P.dup == MG_DUP_ALL) || max_label >= 255 || head >= 1.0) {
    gather_result_t(P, pw, out);
    return;
  }
  Worker& w = *P.workers[P.local_workers.front()];
  DeviceGuard dg(w.dev);
  const uint32_t nv = w.nv;
  const uint32_t m = (uint32_t)(head > 0 ? head * nv : 0);  // [0,m) u32, [m,nv) bytes
  const uint32_t nb = nv - m;
  if (nb < (1u << 20)) {  // small arrays: one plain copy
    gather_result_t(P, pw, out);
    return;
  }
  if (P.label_stage_n < nb) {
    if (P.label_stage) cudaFreeHost(P.label_stage);
    P.label_stage = nullptr;
    MGB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&P.label_stage), nb));
    P.label_stage_n = nb;
    P.label_dev.alloc(nb);
  }
  if (!P.pool) P.pool = std::make_unique<HostPool>(std::thread::hardware_concurrency() > 16
                                                       ? 16
                                                       : std::thread::hardware_concurrency());
  const uint32_t* src = pw[w.p];
  const char* ne = getenv("MG_D2H_NIBBLE");
  const bool nib = max_label < 15 && !(ne && ne[0] == '0');  // 4-bit levels: half the bytes
  const uint32_t nbytes = nib ? (nb + 1) / 2 : nb;
  if (nib)
    MGB_LAUNCH(narrow_labels_nib_kernel, grid_for(nbytes, 256, num_sms() * 8), 256, 0, w.stream,
               src + m, nb, P.label_dev.ptr);
  else
    MGB_LAUNCH(narrow_labels_kernel, grid_for(nb, 256, num_sms() * 8), 256, 0, w.stream, src + m,
               nb, P.label_dev.ptr);
  P.last_d2h_bytes += nbytes + 4ull * m;  // what actually crosses PCIe
  MGB_CUDA(cudaMemcpyAsync(P.label_stage, P.label_dev.ptr, nbytes, cudaMemcpyDeviceToHost,
                           w.stream));
  MGB_CUDA(cudaEventRecord(w.ev_k0, w.stream));
  if (m) MGB_CUDA(cudaMemcpyAsync(out, src, 4ull * m, cudaMemcpyDeviceToHost, w.stream));
  MGB_CUDA(cudaEventSynchronize(w.ev_k0));  // bytes landed: widen while the head streams in
  const uint8_t* stage = P.label_stage;
  uint32_t* dst = out + m;
  P.pool->run([&](unsigned t, unsigned T) {
    const uint64_t lo = (uint64_t)nb * t / T, hi = (uint64_t)nb * (t + 1) / T;
    if (nib)
      widen_labels_u4(stage, dst, lo, hi);
    else
      widen_labels_u8(stage + lo, dst + lo, hi - lo);
  });
  MGB_CUDA(cudaStreamSynchronize(w.stream));
}
void gather_u64(Plan& P, const std::vector<const unsigned long long*>& pw, uint64_t* out) {
  gather_result_t(P, pw, reinterpret_cast<unsigned long long*>(out));
}
void gather_f64(Plan& P, const std::vector<const double*>& pw, double* out) {
  gather_result_t(P, pw, out);
}

}  // namespace mgb
