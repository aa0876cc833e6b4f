/*
 * mgraph_b200.h — C-ABI of the B200-native multi-GPU graph hot path.
 *
 * This is the drop-in boundary for the reference's (mgraph) hot path: the
 * superstep engine `run_primitive` (proj/core/include/mgraph/engine.hpp:712)
 * and the six primitive entry points declared in
 * proj/core/include/mgraph/primitives.hpp:40,85,97,108,120,138.  The
 * reference's host-side graph preparation (csr.cpp, generate.cpp) and its
 * partitioner (partition.cpp) are kept: they are re-stated here on the host
 * in C++ and produce bit-identical CSRs / owner maps for the same seeds.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch / STL types cross the ABI;
 *   - every entry point returns an mg_status; on failure mg_last_error()
 *     returns a thread-local message (the reference's exception what());
 *   - result buffers are caller-allocated, length |V|, in GLOBAL vertex IDs
 *     (reference primitives.cpp:33-41 gather_hosted), sentinels preserved:
 *     MG_INF_LABEL / MG_INF_DIST / MG_INVALID_VERTEX (types.hpp:43-45);
 *   - passing NULL for a result buffer keeps the result device-resident
 *     (fetch it later with mg_plan_fetch_*), which is how the bench times
 *     the device-only "value" leg.
 */
#ifndef MGRAPH_B200_H
#define MGRAPH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --------------------------------------------------------------------------
 * status codes <-> reference exception classes (SURVEY §8(b) "errors") */
typedef enum mg_status {
  MG_OK = 0,
  MG_EINVAL = 1,     /* std::invalid_argument (primitives.cpp:27-30, engine.hpp:716-730) */
  MG_ECAPACITY = 2,  /* mgraph::CapacityError (frontier.hpp:98-102)                      */
  MG_EPLAN = 3,      /* std::runtime_error: missing proxy (engine.hpp:189-192,641-644)    */
  MG_ECUDA = 4,      /* CUDA runtime failure on a worker device                           */
  MG_EWORKER = 5,    /* any other worker failure (engine.hpp:773-782, rethrown at :962)   */
  MG_ERANGE = 6      /* std::runtime_error from I/O-like misuse (wrong lengths)           */
} mg_status;

#define MG_INF_LABEL 0xFFFFFFFFu
#define MG_INVALID_VERTEX 0xFFFFFFFFu
#define MG_INF_DIST 0xFFFFFFFFFFFFFFFFull

const char* mg_last_error(void);
const char* mg_version(void);

/* --------------------------------------------------------------------------
 * host graph (reference Csr, csr.hpp:38-52): u32 row offsets / u32 columns /
 * optional u32 weights.  Owned by the library; arrays are borrowed views. */
typedef struct mg_graph mg_graph;

/* copy a CSR in (validate_csr semantics, csr.cpp:110-125) */
int mg_graph_from_csr(uint32_t num_vertices, uint64_t num_edges, const uint32_t* row_offsets,
                      const uint32_t* col_indices, const uint32_t* edge_values /* nullable */,
                      mg_graph** out);
/* build_csr (csr.cpp:27-69): rows sorted by neighbour, duplicates kept */
int mg_graph_from_edges(uint32_t num_vertices, uint64_t num_edges, const uint32_t* src,
                        const uint32_t* dst, const uint32_t* weight /* nullable */,
                        mg_graph** out);
/* rmat_generate (generate.cpp:25-62) -> build_csr -> optionally symmetrize_dedup */
int mg_graph_rmat(int scale, int edge_factor, double a, double b, double c, double d,
                  uint64_t seed, int symmetrize, mg_graph** out);
/* symmetrize_dedup (csr.cpp:82-108) */
int mg_graph_symmetrize(const mg_graph* g, mg_graph** out);
/* assign_random_weights (generate.cpp:64-79) */
int mg_graph_assign_weights(const mg_graph* g, uint32_t lo, uint32_t hi, uint64_t seed,
                            mg_graph** out);
/* grid_edges / path_edges (generate.cpp:81-97) -> build_csr -> symmetrize_dedup */
int mg_graph_grid(uint32_t rows, uint32_t cols, mg_graph** out);
int mg_graph_path(uint32_t n, mg_graph** out);
int mg_graph_info(const mg_graph* g, uint32_t* num_vertices, uint64_t* num_edges,
                  int* has_weights);
int mg_graph_arrays(const mg_graph* g, const uint32_t** row_offsets, const uint32_t** col_indices,
                    const uint32_t** edge_values);
void mg_graph_destroy(mg_graph* g);

/* counter-based R-MAT generator used for the large benchmark graphs
 * (SURVEY §8(f)-1): edge i, bit k draws from mix64(seed, i, k); the host and
 * device versions produce bit-identical symmetrized CSRs. */
int mg_graph_rmat_hashed(int scale, int edge_factor, uint64_t seed, int threads, mg_graph** out);

/* --------------------------------------------------------------------------
 * partitioners (kept from the reference, partition.cpp:31-85) */
int mg_partition_random(uint32_t num_vertices, uint32_t n, uint64_t seed, uint32_t* owner_out);
int mg_partition_biased_random(const mg_graph* g, uint32_t n, uint64_t seed, double bias,
                               uint32_t* owner_out);

/* --------------------------------------------------------------------------
 * device partition plan: build_partition_plan (partition.cpp:121-209) on the
 * host, then every partition's sub-CSR + owner map + border lists uploaded
 * to its device.  devices[p] = CUDA ordinal of worker p (repeats allowed: a
 * partition per worker, workers may share a GPU for testing). */
typedef struct mg_plan mg_plan;

enum { MG_DUP_ALL = 0, MG_DUP_ONEHOP = 1 };

int mg_plan_create(const mg_graph* g, const uint32_t* owner, uint32_t num_partitions,
                   int duplication, const int* devices /* nullable => all on device 0 */,
                   mg_plan** out);
/* device-generated graph (hashed R-MAT, optional mirrored weights), partitioned
 * on the device with partition_random semantics by `owner` (host array, may be
 * NULL for n == 1).  Avoids the host round trip for scale-24/26 graphs. */
int mg_plan_create_rmat_device(int scale, int edge_factor, uint64_t seed, int with_weights,
                               uint32_t w_lo, uint32_t w_hi, uint64_t w_seed,
                               const uint32_t* owner, uint32_t num_partitions,
                               const int* devices, mg_plan** out);
/* device-generated random geometric graph:
 * n_vertices points uniform in the unit square, edge iff distance <
 * 0.55*sqrt(ln n / n); vertex IDs in generation order */
int mg_plan_create_rgg_device(uint32_t n_vertices, uint64_t seed, const uint32_t* owner,
                              uint32_t num_partitions, const int* devices, mg_plan** out);
void mg_plan_destroy(mg_plan* plan);
int mg_plan_info(const mg_plan* plan, uint32_t* num_vertices, uint64_t* num_edges,
                 uint32_t* num_partitions);
/* BorderMetrics (partition.cpp:211-242): pair_border n*n (nullable), edge_cut */
int mg_plan_border_metrics(const mg_plan* plan, uint64_t* pair_border, uint64_t* edge_cut);
/* copy the global CSR of a device-built plan back to the host (for the CPU
 * baseline / oracle on the same graph) */
int mg_plan_download_graph(const mg_plan* plan, mg_graph** out);
/* device->host bytes the last primitive call / fetch actually copied for its
 * results (e.g. the split u32 / 8-bit / 4-bit label download) */
int mg_plan_last_d2h_bytes(const mg_plan* plan, uint64_t* bytes);
/* time the primitive's dominant kernel with CUDA events on its stream */
int mg_plan_set_profiling(mg_plan* plan, int enable);

/* --------------------------------------------------------------------------
 * engine configuration (EngineConfig, engine.hpp:308-315; AllocationPolicy,
 * frontier.hpp:63-69) */
enum { MG_POLICY_JUST = 0, MG_POLICY_FIXED = 1, MG_POLICY_MAX = 2, MG_POLICY_FUSED = 3 };
enum { MG_FUSED_AUTO = 0, MG_FUSED_ON = 1, MG_FUSED_OFF = 2 };
enum { MG_COMM_DEFAULT = -1, MG_COMM_SELECTIVE = 0, MG_COMM_BROADCAST = 1 };
enum {
  MG_ROLE_ADVANCE_OUTPUT = 0,
  MG_ROLE_FILTER_OUTPUT = 1,
  MG_ROLE_INPUT_FRONTIER = 2,
  MG_ROLE_OUTBOX = 3,
  MG_ROLE_INBOX = 4,
  MG_NUM_ROLES = 5
};

typedef struct mg_config {
  int policy;                     /* MG_POLICY_*                                   */
  int fused;                      /* MG_FUSED_*                                    */
  int comm_override;              /* MG_COMM_*                                     */
  uint32_t h_inflation;           /* >= 1                                          */
  int drop_enabled;               /* DropPackage fault injection (engine.hpp:302)  */
  uint32_t drop_src, drop_dst;
  uint64_t drop_iteration;
  uint64_t max_supersteps;        /* default 1000000                               */
  uint64_t hard_cap_bytes;        /* per-worker budget, 0 = unlimited              */
  double factors[MG_NUM_ROLES];   /* sizing factors (FixedPrealloc / PreallocFused) */
  /* DOBFS (any number of partitions) and BFS (single partition): run a
   * logically-forward superstep with the pull kernels when the exact frontier
   * degree sum exceeds 3x the unvisited list (Beamer's exact cost rule; summed
   * over all partitions so every worker takes the same direction).  The
   * output set is the same; labels, direction log, S and the reported W
   * follow the reference rule (BFS: every superstep forward); the records
   * sent (H) can only shrink.  0 = off. */
  int dobfs_exact_cost;
} mg_config;

void mg_config_default(mg_config* cfg);

/* RunStats (engine.hpp:261-298), scalar part */
enum {
  MG_STOP_FRONTIERS_EMPTY = 0,
  MG_STOP_CONDITION = 1,
  MG_STOP_MAX_SUPERSTEPS = 2,
  MG_STOP_WORKER_ERROR = 3
};
typedef struct mg_stats {
  uint32_t n;
  int stop_reason;
  int communication;              /* MG_COMM_SELECTIVE / MG_COMM_BROADCAST */
  int policy;
  uint64_t supersteps;            /* S */
  uint64_t edges_examined;        /* W */
  uint64_t combine_ops;           /* C */
  uint64_t h_total;               /* sum of H matrix */
  uint64_t wire_records;
  uint64_t peak_bytes;
  uint64_t reallocs;
  double wall_ms;                 /* host wall clock of the superstep loop (engine.hpp:951-964) */
  double exchange_ms;             /* device time of pack+deliver kernels                        */
  double device_ms;               /* CUDA-event time of the superstep loop incl. per-run init   */
  uint64_t gpu_launches;          /* kernels launched by the run                                */
  uint64_t exchange_bytes;        /* bytes written into peer inboxes                           */
  /* dominant kernel of the primitive, filled when profiling is on
   * (mg_plan_set_profiling): CUDA-event time, launches, algorithmic bytes */
  double kernel_ms;
  uint64_t kernel_launches;
  double kernel_bytes;
  /* second timed kernel class (DOBFS: kernel_* = pull step, kernel2_* = the
   * load-balanced push advance) */
  double kernel2_ms;
  uint64_t kernel2_launches;
  double kernel2_bytes;
  /* 1 when the supersteps ran as one CUDA-graph launch (device-driven loop,
   * DobfsGraphRunner), 0 for the host-driven enactor loop */
  int device_loop;
} mg_stats;

/* per-run arrays of the last run on this plan:
 *   MG_ARR_H_MATRIX n*n, MG_ARR_H_PER_ITER S*n ([iter][src]),
 *   MG_ARR_OUT_PER_ITER S, MG_ARR_EDGES_PER_ITER S, MG_ARR_COMBINE_PER_ITER S,
 *   MG_ARR_DIRECTION_LOG S (DOBFS: 0 forward / 1 backward per superstep).
 * Returns the full length in *len; copies min(len, cap) values. */
enum {
  MG_ARR_H_MATRIX = 0,
  MG_ARR_H_PER_ITER = 1,
  MG_ARR_OUT_PER_ITER = 2,
  MG_ARR_EDGES_PER_ITER = 3,
  MG_ARR_COMBINE_PER_ITER = 4,
  MG_ARR_DIRECTION_LOG = 5
};
int mg_plan_last_array(const mg_plan* plan, int which, uint64_t* buf, uint64_t cap,
                       uint64_t* len);
/* BufferStats per worker and role (frontier.hpp:71-81) of the last run */
int mg_plan_last_buffer_stats(const mg_plan* plan, uint32_t worker, int role,
                              uint64_t* realloc_count, uint64_t* peak_items,
                              uint64_t* peak_bytes);

/* --------------------------------------------------------------------------
 * primitives (primitives.hpp) */
int mg_bfs(mg_plan* plan, uint32_t source, int mark_preds, const mg_config* cfg,
           uint32_t* labels, uint32_t* preds, mg_stats* stats);

/* DirectionState (primitives.hpp:50-65) */
typedef struct mg_direction_state {
  int current;                    /* 0 forward, 1 backward */
  uint64_t q_size, u_size, p_size;
  double fv, bv, do_a, do_b;
  int switched_to_backward_once;
} mg_direction_state;
void mg_make_direction_state(int current, uint64_t q, uint64_t u, uint64_t p, uint64_t edges,
                             uint64_t vertices, double do_a, double do_b, int switched_once,
                             mg_direction_state* out);
int mg_direction_decide(const mg_direction_state* s);

int mg_dobfs(mg_plan* plan, uint32_t source, double do_a, double do_b, int mark_preds,
             const mg_config* cfg, uint32_t* labels, uint32_t* preds, int32_t* direction_log,
             uint64_t direction_log_cap, uint64_t* direction_log_len, uint64_t* forward_edges,
             uint64_t* backward_edges, mg_stats* stats);

int mg_sssp(mg_plan* plan, uint32_t source, int mark_preds, const mg_config* cfg,
            uint64_t* dists, uint32_t* preds, mg_stats* stats);

int mg_cc(mg_plan* plan, const mg_config* cfg, uint32_t* components, mg_stats* stats);

int mg_bc(mg_plan* plan, uint32_t source, const mg_config* cfg, double* bc, double* sigma,
          uint32_t* labels, mg_stats* stats);

int mg_pagerank(mg_plan* plan, double damping, double epsilon, uint64_t max_iter,
                const mg_config* cfg, double* ranks, uint64_t* iterations, double* rank_sums,
                uint64_t rank_sums_cap, uint64_t* rank_sums_len, mg_stats* stats);

/* fetch the device-resident result of the last run (labels / dists / comps
 * as raw words; values as f64) into a host buffer of |V| entries */
enum { MG_RES_LABELS = 0, MG_RES_PREDS = 1, MG_RES_DISTS = 2, MG_RES_COMPONENTS = 3,
       MG_RES_BC = 4, MG_RES_SIGMA = 5, MG_RES_RANKS = 6 };
int mg_plan_fetch(mg_plan* plan, int which, void* host_out);

/* --------------------------------------------------------------------------
 * multi-process fabric (one process per GPU on one node, e.g. torchrun).
 * Every rank calls the same constructor with the same partition map and the
 * same job-unique `fabric_key`; rank r uploads only partition r to `device`.
 * The ranks rendezvous through a POSIX shared-memory segment named after the
 * key (host barrier + WorkerReport all-gather, the reference's Barrier and
 * completion callback, engine.hpp:449-473/784-820) and map each other's inbox
 * arenas with CUDA IPC, so the pack kernels store records straight into the
 * peer GPU's HBM over NVLink.  Result buffers of a multi-process run receive
 * this rank's hosted vertices only. */
int mg_plan_create_mp(const mg_graph* g, const uint32_t* owner, uint32_t num_partitions,
                      int duplication, uint32_t rank, int device, const char* fabric_key,
                      mg_plan** out);
int mg_plan_create_rmat_device_mp(int scale, int edge_factor, uint64_t seed, int with_weights,
                                  uint32_t w_lo, uint32_t w_hi, uint64_t w_seed,
                                  const uint32_t* owner, uint32_t num_partitions, uint32_t rank,
                                  int device, const char* fabric_key, mg_plan** out);
/* host protocol self-test (no GPU): `rounds` barriers + all-gathers among
 * `world` processes; returns MG_OK when every gathered value checks out */
int mg_fabric_selftest(const char* fabric_key, uint32_t rank, uint32_t world, uint32_t rounds);

/* number of kernels this library has launched since load (evidence counter) */
uint64_t mg_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* MGRAPH_B200_H */
