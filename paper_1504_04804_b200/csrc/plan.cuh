// plan.cuh — the device-resident partition plan and per-worker runtime state.
//
// One Worker per partition (reference WorkerHandle, engine.hpp:478-582), each
// bound to a CUDA device.  Under Duplicate-All (partition.cpp:157-173) every
// worker holds a |V|-row sub-CSR in which only its hosted rows are non-empty,
// so local ID == global ID and ownership is a u8 lookup.  Inboxes (the
// reference ExchangeFabric slots, engine.hpp:320-445) live in the RECEIVING
// worker's HBM; senders' pack kernels store records into them directly — over
// NVLink when the workers sit on different GPUs.
#pragma once

#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"
#include "shm_fabric.hpp"

namespace mgb {

// POD view of one partition's sub-CSR handed to kernels
struct GraphView {
  uint32_t nv;
  uint64_t ne;
  const uint32_t* __restrict__ off;
  const uint32_t* __restrict__ col;
  const uint32_t* __restrict__ w;  // nullptr if unweighted
};

// ownership view: hosts(v) / owner(v) / to_global(v) for the local ID space
struct OwnerView {
  const uint8_t* __restrict__ owner;  // Duplicate-All: owner[global]
  const uint32_t* __restrict__ l2g;   // OneHop: local -> global (nullptr under All)
  uint32_t p;
  uint32_t nlocal;  // OneHop: hosted vertices are local IDs [0, nlocal)
  int dup;
  __device__ __forceinline__ bool hosts(uint32_t v) const {
    return dup == MG_DUP_ALL ? owner[v] == p : v < nlocal;
  }
  __device__ __forceinline__ uint32_t to_global(uint32_t v) const {
    return dup == MG_DUP_ALL ? v : l2g[v];
  }
  __device__ __forceinline__ uint32_t owner_of_local(uint32_t v) const {
    return owner[to_global(v)];
  }
};

// One inbox slot (dst, src, parity): SoA record arrays in the receiver's HBM
struct SlotView {
  uint32_t* ids;
  uint32_t* va[kMaxAssoc];
  double* vv[kMaxAssoc];
  uint64_t cap;
};

// per-worker device counters, copied to pinned host memory once per superstep
struct Counters {
  uint32_t out_cnt;       // body output length (reference WorkerReport.out_frontier)
  uint32_t next_cnt;      // next-input length after split + merge
  uint32_t adv_cnt;       // unfused advance output length
  uint32_t big_cnt;       // advance: vertices deferred to the big-vertex pass
  uint32_t overflow;      // an inbox / buffer bound was violated
  uint32_t misc;
  unsigned long long edges;      // W delta (edges examined)
  unsigned long long combine;    // C delta
  unsigned long long next_deg;   // sum of out-degrees of next_input (advance bound)
  double f[4];                   // primitive-defined scalars (WorkerReport.f)
  unsigned long long u[4];       // primitive-defined scalars (WorkerReport.u)
  uint32_t send_cnt[kMaxWorkers];  // records packed for each destination
  uint32_t recv_cnt[kMaxWorkers];  // records received from each source (merge)
};

// ---------------------------------------------------------------------------
// device-side superstep protocol of multi-process plans (one rank per GPU):
// every rank owns a Mailbox in its HBM, mapped by its peers over CUDA IPC.
// Peers store their publish flags and their superstep reports into it, so the
// "records delivered" barrier and the WorkerReport all-gather + convergence
// test (engine.hpp:449-473, :784-820) run on the devices; the host only
// synchronises its own stream once per superstep.
constexpr uint32_t kMaxMpRanks = 32;

struct DevReport {  // WorkerReport + per-destination send counts, one rank, one superstep
  unsigned long long out_frontier, next_frontier, edges_delta, combine_delta;
  double f[4];
  unsigned long long u[4];
  uint32_t send_cnt[kMaxMpRanks];
  uint32_t overflow;
  uint32_t epoch;  // written last (volatile store): the report's arrival flag
};

struct Mailbox {
  uint32_t pub[2][kMaxMpRanks];   // [parity][src]: epoch whose records src delivered
  DevReport rep[2][kMaxMpRanks];  // [epoch parity][src]
};

struct Worker {
  uint32_t p = 0;
  int dev = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_x0 = nullptr, ev_x1 = nullptr;
  cudaEvent_t ev_k0 = nullptr, ev_k1 = nullptr;  // dominant-kernel timing (profiling)

  // sub-graph
  uint32_t nv = 0;
  uint64_t ne = 0;
  uint32_t nlocal = 0;
  DevArray<uint32_t> off, col, w;
  DevArray<uint32_t> hosted;  // hosted local IDs (reference hosted_local(), engine.hpp:756-763)
  DevArray<uint8_t> owner;    // global owner map (u8; n <= 255)
  DevArray<uint32_t> l2g;     // OneHop only
  DevArray<uint32_t> border;  // static remote sub-frontier (PR): local IDs, grouped by peer
  std::vector<uint64_t> border_len;  // per peer
  std::vector<uint64_t> border_off;  // per peer start in `border`

  // policy-managed frontier buffers (roles of frontier.hpp:33-35)
  MemoryBudget budget;
  BufferStats stats[MG_NUM_ROLES];
  DevBuf<uint32_t> input, next_input, advance_out, output;
  DevArray<uint32_t> merge_stamp;
  DevArray<uint32_t> lb_row;    // advance scratch: row start per frontier entry
  DevArray<unsigned long long> lb_pref, lb_bsum;  // CTA-local degree prefix, CTA offsets
  DevArray<uint32_t> lb_tile;   // first frontier entry of every expansion tile

  // inbox arena (receiver side): [parity][src] slots + counts
  int nva = 0, nvv = 0;
  std::vector<uint64_t> slot_cap;  // per src
  DevArray<uint8_t> arena;
  uint64_t arena_gen = 0;          // bumped whenever the arena is reallocated
  SlotView slots[2][kMaxWorkers];
  DevArray<uint32_t> inbox_cnt;    // [2][kMaxWorkers], written by senders
  // sender side: where this worker's records for each peer go, per parity
  DevArray<SlotView> send_table;   // [2][n]
  DevArray<uint32_t*> send_cnt_ptr;  // [2][n] -> &inbox_cnt[parity][p] at peer
  DevArray<SlotView> recv_table;     // [2][n] device copy of `slots` (merge kernel)
  std::vector<uint8_t> table_sig;    // host image of the three tables last uploaded

  // primitive state arrays (|V_i| entries each), reused across runs; results
  // of the last run stay here until the next run (mg_plan_fetch)
  DevArray<uint32_t> su32[4];
  DevArray<double> sf64[4];
  DevArray<unsigned long long> su64[3];
  DevArray<uint32_t> aux[6];          // primitive-private scratch (bitmaps, queues)
  DevArray<uint32_t> nonisolated;     // hosted vertices with out-degree > 0 (ascending)
  DevArray<uint4> pull_rec;           // DOBFS pull records {v, deg, arc0, arc1} per nonisolated
  DevArray<uint4> pull_ext;           // their 32-byte extensions: arcs 2..9 (stage 1b)
  DevArray<uint32_t> ul_buf[3];       // DOBFS unvisited lists (ping-pong) + long-row queue
  // device-driven DOBFS (graph mode): loop state, history, fixed frontier and
  // advance scratch, the instantiated graphs (by mark_preds)
  DevArray<uint8_t> loop_state, loop_hist;
  void* loop_host = nullptr;       // pinned copy of the loop state
  void* loop_hist_host = nullptr;  // pinned per-superstep history
  DevArray<uint32_t> loop_front[2], loop_lb_row, loop_tiles;
  DevArray<unsigned long long> loop_lb_pref, loop_lb_bsum, loop_total;
  cudaGraphExec_t loop_exec[2] = {nullptr, nullptr};  // by mark_preds
  uint32_t loop_n_pull[2] = {0, 0}, loop_n_push[2] = {0, 0};
  std::vector<const void*> loop_ptrs[2];  // device pointers each graph captured
  // device-driven DOBFS across processes (one partition per rank): loop state,
  // history and the instantiated graph
  DevArray<uint8_t> mp_state, mp_hist;
  cudaGraphExec_t mp_exec = nullptr;
  uint32_t mp_n_pull = 0, mp_n_push = 0, mp_n_fixed = 0;  // kernels per branch / superstep
  std::vector<const void*> mp_ptrs;
  // transpose of the sub-graph (in-arcs from hosted vertices), rows sorted by
  // source; built once per plan for the pull-form PageRank accumulation
  DevArray<uint32_t> toff, tcol, tlong;
  uint32_t n_tlong = 0;
  bool transpose_ready = false;
  bool pr_reordered = false;          // single partition: PR arrays in locality order
  DevArray<uint32_t> pr_perm, pr_pdeg;  // vertex -> ordered position; out-degree by position
  DevArray<uint32_t> pr_iperm;          // ordered position -> vertex
  int cc_symmetric = -1;                // ordered transpose symmetric? (-1: not checked)
  DevArray<double> bc_acc;              // BC: huge-row partial sums
  uint32_t n_nonisolated = 0;
  bool nonisolated_ready = false;
  // DOBFS labels: when the label array holds a completed DOBFS run's result,
  // the next run skips the |V|-entry fill and only resets the vertices the
  // previous run reached and this one does not (dobfs_lastvis = the previous
  // run's visited bitmap).  Any other primitive clears the flag.
  DevArray<uint32_t> dobfs_lastvis;
  bool dobfs_labels_ok = false;
  std::vector<uint32_t> hosted_host;  // hosted local IDs (host copy)
  DevArray<uint32_t> border_dst;      // PR: destination-local ID of every border entry

  // counters
  DevArray<Counters> ctr;
  Counters* host_ctr = nullptr;      // pinned, mapped
  Counters* host_ctr_dev = nullptr;  // its device-side address (report_kernel writes it)

  GraphView graph() const { return {nv, ne, off.ptr, col.ptr, w.ptr}; }
};

// persistent host worker threads (result widening); run() blocks until every
// thread has run f(thread, threads)
class HostPool {
 public:
  explicit HostPool(unsigned n);
  ~HostPool();
  void run(const std::function<void(unsigned, unsigned)>& f);

 private:
  unsigned n_;
  std::vector<std::thread> threads_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  std::function<void(unsigned, unsigned)> job_;
  uint64_t gen_ = 0;
  unsigned pending_ = 0;
  bool stop_ = false;
};

struct Plan {
  uint32_t n = 1;
  int dup = 0;
  uint32_t nv = 0;
  uint64_t ne = 0;
  bool weighted = false;
  uint32_t max_weight = 0;  // largest edge weight (SSSP picks its distance width from it)
  std::vector<int> devices;
  std::vector<std::unique_ptr<Worker>> workers;  // only local workers are populated
  std::vector<uint32_t> local_workers;           // partition ids driven by this process
  std::vector<std::vector<uint64_t>> pair_border;  // |B_{i,j}|
  std::vector<uint64_t> nlocal;                    // |L_i|
  uint64_t edge_cut = 0;
  std::vector<uint32_t> owner_host;  // global owner map (host copy)
  bool multiprocess = false;
  uint32_t rank = 0, world = 1;
  // host copy of the global CSR (kept when built from a host graph)
  std::shared_ptr<HostCsr> host_graph;
  // device copy of the global CSR (device-built plans) on workers[0]'s device
  DevArray<uint32_t> g_off, g_col, g_w;

  // last run
  mg_stats last{};
  std::vector<std::vector<uint64_t>> h_matrix;
  std::vector<std::vector<uint64_t>> h_per_iter;
  std::vector<uint64_t> out_per_iter, edges_per_iter, combine_per_iter;
  std::vector<std::vector<BufferStats>> last_buffers;  // [worker][role]
  // device-resident results of the last run (global ID space, on workers[0].dev)
  int last_result_kind = -1;
  // bytes the last primitive call moved host<->device for its arguments /
  // results (reset at the start of every call; the e2e bench line reports them)
  uint64_t last_h2d_bytes = 0, last_d2h_bytes = 0;
  std::vector<int> last_dir_log;  // DOBFS direction per superstep of the last run

  // live timing of the primitive's dominant kernel (bench roofline)
  bool profile = false;
  double prof_ms = 0, prof_bytes = 0;
  uint64_t prof_launches = 0;
  double prof2_ms = 0, prof2_bytes = 0;
  uint64_t prof2_launches = 0;

  // multi-process fabric (one worker per process): shared-memory rendezvous +
  // CUDA IPC mappings of the peers' inbox arenas and slot counters
  std::unique_ptr<ShmFabric> shm;
  std::vector<void*> peer_arena;     // mapped inbox arenas of peers (by rank)
  std::vector<void*> peer_cnt;       // mapped inbox counters of peers
  std::vector<uint64_t> peer_gen;    // arena generation each mapping belongs to
  std::vector<SlotView> peer_slots;  // [2][n]: peer q's slot for records from this rank
  // device-side protocol (default for multi-process plans; MG_HOST_FABRIC=1
  // selects the shared-memory barrier + all-gather instead)
  bool device_fabric = true;
  DevArray<uint8_t> mbox;              // this rank's Mailbox
  std::vector<void*> peer_mbox;        // mapped peer mailboxes
  DevArray<Mailbox*> mbox_ptrs;        // [n]: every rank's Mailbox (own included)
  DevReport* host_reports = nullptr;   // mapped pinned: [kMaxMpRanks] + error word
  DevReport* host_reports_dev = nullptr;
  uint32_t mp_epoch = 0;               // superstep counter, identical on every rank
  // split label download (gather_labels_u32)
  uint8_t* label_stage = nullptr;      // pinned byte staging
  uint64_t label_stage_n = 0;
  DevArray<uint8_t> label_dev;
  std::unique_ptr<HostPool> pool;
};

struct WorkerReport;
// multi-process fabric (fabric.cu)
void fabric_sync(Plan& P);

Worker& worker(Plan& P, uint32_t p);
uint32_t device_max_u32(const uint32_t* a, uint64_t n);
void init_worker_runtime(Worker& w);
void plan_free(Plan* P);

}  // namespace mgb

// the C-ABI's opaque host graph (include/mgraph_b200.h)
struct mg_graph {
  std::shared_ptr<mgb::HostCsr> g;
};
