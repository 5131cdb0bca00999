/*
 * cad.h -- C-ABI of the B200-native core-attention (CA) hot path.
 *
 * Drop-in boundary for DistCA's CA path. The reference (`cadsim`, C++20) has
 * a value-type C++ API and no FFI; every entry point below replaces one
 * reference function (cited as P/<file>:<line>, P = /root/reference/proj) or
 * one modeled device operation that the reference only simulates
 * (P/src/sim.cpp:22-30 for the CA kernel, P/src/sim.cpp:69-125 for the
 * dispatch/return windows).
 *
 * Conventions
 *  - POD structs only; no C++ or torch types cross this boundary.
 *  - Every function returns int status: CAD_OK (0) or a negative code. The
 *    reference's C++ exceptions map to codes: ConfigError -> CAD_ERR_CONFIG,
 *    DomainError -> CAD_ERR_DOMAIN (P/include/cadsim/types.hpp:18-27). The
 *    message of the last error on the calling thread is cad_last_error().
 *  - Nothing throws across the ABI.
 *  - Scheduler calls are re-entrant and thread-safe (the reference's types
 *    are immutable values, P/include/cadsim/types.hpp:30-31). Device calls
 *    take an explicit cudaStream_t (passed as void*) and caller-owned
 *    device buffers; one comm context per GPU and per thread.
 */
#ifndef CAD_H_
#define CAD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CAD_OK 0
#define CAD_ERR_CONFIG (-1)
#define CAD_ERR_DOMAIN (-2)
#define CAD_ERR_CUDA (-3)
#define CAD_ERR_NCCL (-4)
#define CAD_ERR_CAPACITY (-5) /* caller buffer too small; *n holds the need */

/* Layout, P/include/cadsim/types.hpp:99 */
#define CAD_LAYOUT_CONTIGUOUS 0
#define CAD_LAYOUT_HEAD_TAIL 1

/* DistKind, P/include/cadsim/workload.hpp:13-19 */
#define CAD_DIST_PRETRAIN_UPSAMPLED 0
#define CAD_DIST_PROLONG_LIKE 1
#define CAD_DIST_UNIFORM 2
#define CAD_DIST_FIXED 3
#define CAD_DIST_CUSTOM_HISTOGRAM 4

/* ---------------------------------------------------------------------- */
/* Descriptors                                                             */
/* ---------------------------------------------------------------------- */

/* cadsim::Item, P/include/cadsim/types.hpp:112-124. A CA-task extent:
 * queries [q_begin,q_end) of document `doc` with causal context
 * [0,kv_extent), kv_extent == q_end. */
typedef struct cad_item {
  int64_t doc;
  int64_t q_begin;
  int64_t q_end;
  int64_t kv_extent;
  int64_t ht_mirror;
  int32_t home_device;
  uint8_t layout; /* CAD_LAYOUT_* */
  uint8_t pad_[3];
} cad_item;

/* cadsim::CATask, P/include/cadsim/types.hpp:131-137 */
typedef struct cad_task {
  cad_item item;
  int32_t source_device;
  int32_t assigned_server;
  int64_t comm_bytes;   /* Q/KV dispatch bytes, 0 when served at home */
  int64_t output_bytes; /* O return bytes, 0 when served at home */
} cad_task;

/* cadsim::SchedulerConfig, P/include/cadsim/scheduler.hpp:12-21 */
typedef struct cad_sched_cfg {
  double epsilon;
  double e_threshold;
  int64_t tile_size;
  double alpha_ca;
  int64_t size_q;
  int64_t size_kv;
  uint8_t double_query_head_tail;
  uint8_t pad_[7];
  int64_t max_moves;
} cad_sched_cfg;

/* cadsim::ServerLoad, P/include/cadsim/scheduler.hpp:23-30 (items are
 * returned separately by cad_plan_server). */
typedef struct cad_server_load {
  int32_t device;
  int32_t pad_;
  double assigned_flops;
  int64_t assigned_core;
  int64_t n_items;
  int64_t sent_bytes;
  int64_t received_bytes;
} cad_server_load;

/* Scalar fields of cadsim::SchedulePlan, P/include/cadsim/scheduler.hpp:32-45 */
typedef struct cad_plan_stats {
  double target;
  double max_load;
  double min_load;
  double epsilon_used;
  int64_t total_comm_bytes;
  int64_t total_output_bytes;
  int64_t migrations;
  int64_t splits;
  int64_t rejected_small;
  int64_t n_tasks;
  int64_t n_servers;
  int32_t tolerance_met;
  int32_t pad_;
} cad_plan_stats;

/* cadsim::MigrationProposal, P/include/cadsim/scheduler.hpp:60-67 */
typedef struct cad_proposal {
  double delta_f_max;
  cad_item shard;
  cad_item remainders[2];
  int32_t n_remainders;
  int32_t whole_item;
  int64_t v_comm;
  double priority;
} cad_proposal;

/* cadsim::CommQuery / ShardChoice, P/include/cadsim/comm.hpp:41-60 */
typedef struct cad_comm_query {
  double delta_f_max;
  double f_item;
  int64_t L_q;
  int64_t L_kv;
  int64_t size_q;
  int64_t size_kv;
  uint8_t layout;
  uint8_t pad_[7];
  int64_t ht_mirror;
} cad_comm_query;

typedef struct cad_shard_choice {
  int64_t n_q;
  int64_t n_kv;
  int64_t bytes;
  int64_t core;
} cad_shard_choice;

/* cadsim::LengthDistribution, P/include/cadsim/workload.hpp:28-43 */
typedef struct cad_length_dist {
  int32_t kind; /* CAD_DIST_* */
  int32_t pad_;
  int64_t max_doc_len;
  int64_t min_len_threshold;
  uint64_t seed;
  double log_mu;
  double log_sigma;
  double upsample_drop_prob;
  double long_mix_weight;
  double long_log_mu;
  double long_log_sigma;
  int64_t fixed_len;
  int64_t uniform_min;
  const int64_t* hist_len; /* custom_histogram: lengths */
  const double* hist_p;    /* custom_histogram: weights */
  int64_t hist_n;
} cad_length_dist;

/* cadsim::ServedTask, P/include/cadsim/sim.hpp:30-35, by task index. */
typedef struct cad_served_task {
  int64_t task_index; /* index into cad_plan_tasks() */
  int64_t in_bytes;
  int64_t out_bytes;
  int32_t half; /* 0 = ping, 1 = pong */
  int32_t pad_;
} cad_served_task;

typedef struct cad_plan cad_plan; /* opaque SchedulePlan */

/* ---------------------------------------------------------------------- */
/* Host: workload, cost, scheduler                                         */
/* ---------------------------------------------------------------------- */

const char* cad_last_error(void);
const char* cad_version(void);

void cad_sched_cfg_default(cad_sched_cfg* cfg); /* scheduler.hpp:12-21 defaults */
void cad_length_dist_default(cad_length_dist* d); /* workload.hpp:28-43 defaults */

/* validate_item, P/src/types.cpp:58-74 */
int cad_validate_item(const cad_item* item);
/* ca_flops_core, P/src/cost.cpp:32-44 */
int cad_ca_flops_core(const cad_item* item, int64_t* core);
/* exact_causal_pairs, P/src/oracle.cpp:50-54 (closed form) */
int64_t cad_causal_pairs(int64_t n_q, int64_t n_kv);
/* item_bytes / shard_bytes, P/src/scheduler.cpp:53-60, P/src/comm.cpp:35-42 */
int cad_item_bytes(const cad_item* item, const cad_sched_cfg* cfg, int64_t* bytes);

/* sample_batch, P/src/workload.cpp:67-84. Two-call: lengths may be NULL with
 * cap 0 to learn *n_docs. */
int cad_sample_batch(const cad_length_dist* dist, int64_t total_tokens,
                     int64_t* lengths, int64_t cap, int64_t* n_docs);
/* place_sequential + chunk_items, P/src/workload.cpp:86-124 and
 * P/src/types.cpp:117-132: the contiguous items of every device chunk, in
 * chunk order. */
int cad_place_sequential(const int64_t* lengths, int64_t n_docs,
                         int64_t n_devices, int64_t tokens_per_device,
                         cad_item* items, int64_t cap, int64_t* n_items);

/* target_load, P/src/scheduler.cpp:13-19 */
int cad_target_load(const cad_item* items, int64_t n, int64_t n_servers,
                    double alpha_ca, double* target);
/* classify_servers, P/src/scheduler.cpp:21-34. Output arrays hold n entries. */
int cad_classify_servers(const double* loads, int64_t n, double target,
                         int32_t* surplus_dev, double* surplus_gap,
                         int64_t* n_surplus, int32_t* deficit_dev,
                         double* deficit_gap, int64_t* n_deficit);
/* one_tile_slack, P/src/scheduler.cpp:36-49 */
int cad_one_tile_slack(const cad_item* items, int64_t n,
                       const cad_sched_cfg* cfg, double* slack);
/* v_min_comm, P/src/comm.cpp:98-178 */
int cad_v_min_comm(const cad_comm_query* q, int64_t tile, cad_shard_choice* out);
/* propose_migration, P/src/scheduler.cpp:109-194. *has_value = 0 plays
 * std::nullopt. */
int cad_propose_migration(const cad_server_load* source,
                          const cad_server_load* dest, const cad_item* item,
                          double target, const cad_sched_cfg* cfg,
                          cad_proposal* out, int32_t* has_value);

/* schedule, P/src/scheduler.cpp:196-357 (bit-exact) */
int cad_schedule(const cad_item* items, int64_t n, int64_t n_servers,
                 const cad_sched_cfg* cfg, cad_plan** plan);
/* schedule_pp_tick, P/src/scheduler.cpp:359-373: items[i] belongs to stage
 * stage_of[i]; n_stages stages. */
int cad_schedule_pp_tick(const cad_item* items, const int32_t* stage_of,
                         int64_t n, int64_t n_stages, int64_t n_servers,
                         const cad_sched_cfg* cfg, cad_plan** plan);
int cad_plan_get_stats(const cad_plan* plan, cad_plan_stats* stats);
int cad_plan_tasks(const cad_plan* plan, const cad_task** tasks, int64_t* n);
int cad_plan_server(const cad_plan* plan, int64_t server, cad_server_load* load,
                    const cad_item** items);
/* plan_to_stream, P/src/scheduler.cpp:375-385. *needed = strlen + 1. */
int cad_plan_to_text(const cad_plan* plan, char* buf, size_t cap, size_t* needed);
void cad_plan_free(cad_plan* plan);

/* Pipeline tick table of simulate_pp_iteration (P/src/sim.cpp:297-353):
 * out[tick * n_stages + stage] for n_ticks ticks (two-call: out may be NULL
 * with cap 0 to learn *n_ticks; CAD_ERR_CAPACITY then). Errors as the
 * reference: n_stages < 1, n_microbatches < n_stages -> CAD_ERR_CONFIG. */
#define CAD_PP_1F1B 0       /* PPSchedule::vanilla_1f1b */
#define CAD_PP_PHASE_SYNC 1 /* PPSchedule::cad_phase_sync */
typedef struct cad_tick_work {
  int32_t active;
  int32_t backward;
  int64_t microbatch;
} cad_tick_work;
int cad_pp_tick_table(int64_t n_microbatches, int64_t n_stages, int32_t kind,
                      cad_tick_work* out, int64_t cap, int64_t* n_ticks);

/* device_plans_from_schedule (served/sent + assign_halves),
 * P/src/sim.cpp:34-46,129-157 */
int cad_device_plan(const cad_plan* plan, int32_t device,
                    cad_served_task* served, int64_t cap_served,
                    int64_t* n_served, cad_served_task* sent, int64_t cap_sent,
                    int64_t* n_sent);

/* ---------------------------------------------------------------------- */
/* Device: the CA kernels (replace task_layer_seconds, P/src/sim.cpp:22-30) */
/* ---------------------------------------------------------------------- */

/* One CA task as the server's kernel sees it: q rows [q_off, q_off+n_q) of
 * the packed Q/O/dO buffers attend to kv rows [kv_off, kv_off+kv_len) of the
 * packed K/V buffers with a bottom-right causal mask: query i sees keys
 * 0 .. kv_len-n_q+i (P/src/oracle.cpp:50-54). Requires kv_len >= n_q >= 1. */
typedef struct cad_ca_task {
  int64_t q_off;
  int64_t n_q;
  int64_t kv_off;
  int64_t kv_len;
} cad_ca_task;

/* Packed THD layouts: Q/O/dO [q_rows][h_q][head_dim] bf16, K/V/dK/dV
 * [kv_rows][h_kv][head_dim] bf16, LSE [h_q][q_rows] fp32 (natural log),
 * all accumulation fp32 (in TMEM), outputs written bf16. head_dim must be 128.
 * softmax_scale <= 0 selects 1/sqrt(head_dim). */
typedef struct cad_ca_shape {
  int32_t h_q;
  int32_t h_kv;
  int32_t head_dim;
  float softmax_scale;
  int64_t q_rows;
  int64_t kv_rows;
} cad_ca_shape;

typedef struct cad_ca_plan cad_ca_plan; /* device work list for a task set */

typedef struct cad_ca_plan_info {
  int64_t n_fwd_units;
  int64_t n_bwd_units;
  int64_t causal_pairs;   /* sum over tasks of exact causal pairs */
  double fwd_flops;       /* 4 * d * h_q * pairs */
  double bwd_flops;       /* 10 * d * h_q * pairs */
  size_t workspace_bytes; /* bytes cad_ca_bwd needs (+ an fp32 dQ accumulator
                             when CAD_BWD_FUSED=1 selects the experimental
                             fused backward) */
} cad_ca_plan_info;

int cad_ca_plan_create(const cad_ca_task* tasks, int64_t n_tasks,
                       const cad_ca_shape* shape, cad_ca_plan** plan);
int cad_ca_plan_info_get(const cad_ca_plan* plan, cad_ca_plan_info* info);
int cad_ca_plan_destroy(cad_ca_plan* plan);
/* Caps the persistent CTAs of this plan's launches (0 = one per SM), e.g.
 * to leave SMs to NCCL kernels that overlap the CA kernel. */
int cad_ca_plan_set_max_ctas(cad_ca_plan* plan, int max_ctas);

/* Forward: O = softmax(scale * Q K^T + causal mask) V, LSE per (head, row). */
int cad_ca_fwd(const cad_ca_plan* plan, const void* q, const void* k,
               const void* v, void* o, float* lse, void* stream);

/* Backward: dQ, dK, dV from Q, K, V, O, dO, LSE. Deterministic (no atomics).
 * dQ rows of every task and dK/dV rows of every KV group (tasks sharing one
 * kv_off, e.g. shards of one document) are overwritten; the group's rows
 * receive the sum over all of its tasks. Tasks must have disjoint Q rows and
 * groups disjoint KV rows (CAD_ERR_DOMAIN at plan creation otherwise).
 * workspace >= workspace_bytes. */
int cad_ca_bwd(const cad_ca_plan* plan, const void* q, const void* k,
               const void* v, const void* o, const float* lse, const void* dout,
               void* dq, void* dk, void* dv, void* workspace, size_t ws_bytes,
               void* stream);

/* The backward's launches, separately: D = rowsum(dO*O) (+ log2 LSE) into the
 * workspace, then dK/dV and dQ, which only depend on the workspace and may
 * run on different streams once DELTA has completed. With CAD_BWD_FUSED=1
 * (experimental, not deterministic) CAD_BWD_DKDV also adds the dQ partials
 * into the workspace's fp32 accumulator and CAD_BWD_DQ converts it. */
#define CAD_BWD_DELTA 1
#define CAD_BWD_DKDV 2
#define CAD_BWD_DQ 4
#define CAD_BWD_ALL 7
int cad_ca_bwd_parts(const cad_ca_plan* plan, const void* q, const void* k,
                     const void* v, const void* o, const float* lse,
                     const void* dout, void* dq, void* dk, void* dv,
                     void* workspace, size_t ws_bytes, int parts, void* stream);

/* ---------------------------------------------------------------------- */
/* Device: dispatch / return (replace layer_windows, P/src/sim.cpp:69-125)  */
/* ---------------------------------------------------------------------- */

/* One layer's data movement for one rank (the real counterpart of
 * device_plans_from_schedule + layer_windows, P/src/sim.cpp:69-157). Built
 * from a schedule and the pre-schedule home items (cad_place_sequential
 * output); all ranks build it deterministically. Two halves (ping = 0,
 * pong = 1, the assign_halves split). Per half, four row exchanges: */
#define CAD_XFER_Q 0      /* Q (and dO) rows: home -> server            */
#define CAD_XFER_KV 1     /* K/V rows: owner -> server (KV once per doc) */
#define CAD_XFER_O_RET 2  /* O/LSE (and dQ) rows: server -> home         */
#define CAD_XFER_KV_RET 3 /* dK/dV partial rows: server -> owner (summed) */

typedef struct cad_layer_plan cad_layer_plan;

typedef struct cad_layer_half_info {
  int64_t home_rows;  /* rows of this rank's home buffers */
  int64_t q_rows;     /* rows of the server Q/O/dO buffers of the half */
  int64_t kv_rows;    /* rows of the server K/V buffers of the half */
  int64_t n_tasks;
  const cad_ca_task* tasks;   /* server CA-tasks (plan for cad_ca_plan_create) */
  const int64_t* task_index;  /* index into cad_plan_tasks() per server task */
  int64_t remote_send_bytes[4]; /* bytes this rank puts on the wire per xfer */
} cad_layer_half_info;

/* Row lists of one exchange as seen by this rank: send_idx lists source
 * rows grouped by destination peer (send_counts[p] each), recv_idx lists
 * destination rows grouped by source peer. Peer == rank is a local copy. */
typedef struct cad_xfer {
  int64_t n_peers;
  const int64_t* send_counts;
  const int64_t* send_idx;
  const int64_t* recv_counts;
  const int64_t* recv_idx;
  int64_t n_send;
  int64_t n_recv;
} cad_xfer;

int cad_layer_plan_create(const cad_plan* plan, const cad_item* home_items,
                          int64_t n_items, int32_t rank, int64_t q_row_bytes,
                          int64_t kv_row_bytes, cad_layer_plan** out);
/* Same, with balance = 1: each server's halves evened out in causal pairs
 * (to within 1 %) by moving the query tail of the heavier half's largest
 * contiguous CA-task into the other half; balance = 2: one half (every task
 * in the ping half, the pong half empty: no ping-pong, half the launches,
 * for batches whose transfers are negligible). The reference's halves
 * (assign_halves, P/src/sim.cpp:34-46) balance nothing per server; served
 * tasks, residency and results are unchanged, only the ping/pong split
 * moves. balance = 0 is cad_layer_plan_create. */
int cad_layer_plan_create_ex(const cad_plan* plan, const cad_item* home_items,
                             int64_t n_items, int32_t rank, int64_t q_row_bytes,
                             int64_t kv_row_bytes, int32_t balance,
                             cad_layer_plan** out);
int cad_layer_plan_info(const cad_layer_plan* lp, int32_t half,
                        cad_layer_half_info* info);
int cad_layer_plan_xfer(const cad_layer_plan* lp, int32_t half, int32_t which,
                        cad_xfer* x);
void cad_layer_plan_destroy(cad_layer_plan* lp);

typedef struct cad_comm cad_comm; /* one NCCL communicator per GPU */

#define CAD_UNIQUE_ID_BYTES 128
int cad_comm_unique_id(uint8_t id[CAD_UNIQUE_ID_BYTES]);
int cad_comm_init(const uint8_t id[CAD_UNIQUE_ID_BYTES], int32_t rank,
                  int32_t world, cad_comm** comm);
int cad_comm_destroy(cad_comm* comm);

/* Row gather: dst[i] = src[idx[i]] for rows of row_bytes (16-byte multiple). */
int cad_gather_rows(const void* src, const int64_t* idx_dev, int64_t n_rows,
                    int64_t row_bytes, void* dst, void* stream);
/* Row scatter: dst[idx[i]] = src[i]. */
int cad_scatter_rows(const void* src, const int64_t* idx_dev, int64_t n_rows,
                     int64_t row_bytes, void* dst, void* stream);
/* Row scatter-add of bf16 rows into fp32 rows: dst[idx[i]] += src[i]
 * (row_elems elements per row); rows may repeat (partials are summed). */
int cad_scatter_add_bf16(const void* src, const int64_t* idx_dev,
                         int64_t n_rows, int64_t row_elems, float* dst,
                         void* stream);
/* Column gather/scatter of a [heads][rows] fp32 matrix (LSE):
 * dst[i][h] = src[h][idx[i]] and its inverse. */
int cad_gather_cols_f32(const float* src, int64_t src_rows, int32_t heads,
                        const int64_t* idx_dev, int64_t n, float* dst,
                        void* stream);
int cad_scatter_cols_f32(const float* src, const int64_t* idx_dev, int64_t n,
                         int32_t heads, float* dst, int64_t dst_rows,
                         void* stream);
/* fp32 -> bf16 elementwise (dK/dV accumulators to output). */
int cad_f32_to_bf16(const float* src, int64_t n, void* dst, void* stream);

/* ---- copy-engine transport (CUDA IPC + stream memory operations) ------ */
/* The export handle of the allocation holding `ptr` and ptr's offset in it. */
int cad_ipc_handle(const void* ptr, uint8_t handle[64], int64_t* offset);
/* Maps a peer allocation (cudaIpcOpenMemHandle, lazy peer access). */
int cad_ipc_open(const uint8_t handle[64], void** base);
int cad_ipc_close(void* base);

/* A run of consecutive rows: rows [src_row, src_row+n_rows) -> [dst_row, ...). */
typedef struct cad_run {
  int64_t src_row;
  int64_t dst_row;
  int64_t n_rows;
} cad_run;
/* One cudaMemcpyAsync per run (copy engines; dst may be a peer mapping). */
int cad_copy_runs(const cad_run* runs, int64_t n, const void* src, void* dst,
                  int64_t row_bytes, void* stream);
/* Runs of a [heads][rows] fp32 matrix (LSE): one 2-D copy per run. */
int cad_copy_runs_cols(const cad_run* runs, int64_t n, const float* src,
                       int64_t src_rows, float* dst, int64_t dst_rows,
                       int32_t heads, void* stream);
/* SM-driven copy of a list of byte ranges (device array of cad_span; dst
 * may be a peer mapping, written over NVLink by loads/stores): one launch of
 * n_ctas CTAs for the whole list, 16-byte vectors where src, dst and size
 * are 16-byte aligned, 4-byte words otherwise (sizes must be multiples of
 * 4). Used instead of copy-engine memcpys when the CA kernels' L2 traffic
 * starves the copy engines. */
typedef struct cad_span {
  const void* src;
  void* dst;
  int64_t bytes;
} cad_span;
int cad_copy_spans(const cad_span* spans_dev, int64_t n, int32_t n_ctas, void* stream);
/* GPU-side flags: write a 32-bit value once prior stream work is done, and
 * make a stream wait until a (local) flag is >= value. */
int cad_stream_write_u32(void* addr, uint32_t value, void* stream);
int cad_stream_wait_u32(const void* addr, uint32_t value, void* stream);

/* All-to-allv over the communicator (grouped ncclSend/ncclRecv), byte
 * counts and displacements per peer, on `stream`. */
int cad_alltoallv(cad_comm* comm, const void* send, const int64_t* send_bytes,
                  const int64_t* send_displ, void* recv,
                  const int64_t* recv_bytes, const int64_t* recv_displ,
                  void* stream);

/* ---------------------------------------------------------------------- */
/* Device: the per-layer executor -- "run this device's layer: dispatch, CA, */
/* return" (the real counterpart of simulate_layer_pingpong / layer_windows, */
/* P/include/cadsim/sim.hpp:88, P/src/sim.cpp:69-125,176-221)               */
/* ---------------------------------------------------------------------- */

/* How rows move between ranks. */
#define CAD_TRANSPORT_LOCAL 0 /* every rank's context lives in this process
                                 (one GPU, or GPUs with peer access): peers'
                                 buffers are addressed directly; the same
                                 copy/flag code path as IPC. Driven phase by
                                 phase in dependency order across the ranks
                                 (cad_layer_step refuses: CAD_ERR_CONFIG) */
#define CAD_TRANSPORT_IPC 1   /* one process per GPU: each rank pushes its
                                 rows into the peers' buffers (CUDA IPC
                                 mappings, copy engines) and signals arrival
                                 with GPU-side flags; no host synchronisation */
#define CAD_TRANSPORT_NCCL 2  /* gather -> grouped ncclSend/ncclRecv
                                 all-to-allv -> scatter on the caller's stream */

typedef struct cad_layer_cfg {
  int32_t rank;
  int32_t world;
  int32_t h_q;
  int32_t h_kv;
  int32_t head_dim;      /* 128 */
  float softmax_scale;   /* <= 0: 1/sqrt(head_dim) */
  int32_t transport;     /* CAD_TRANSPORT_* */
  int32_t layers;        /* server activation sets. 1 = one CA layer. L > 1 is
                            a benchmark mode: L stacked CA layers per step with
                            the identity between them (every layer sees the
                            step's inputs; O/LSE/dQ are the last layer's, dK/dV
                            the SUM over the L layers) */
  int32_t balance_halves; /* 0: the reference's assign_halves split; 1: halves
                            evened out per server; 2: one half (see
                            cad_layer_plan_create_ex) */
  int32_t reserve_sms;   /* CA kernels leave this many SMs free (NCCL) */
  int32_t pad_[2];
} cad_layer_cfg;

typedef struct cad_layer_ctx cad_layer_ctx;

typedef struct cad_layer_ctx_info {
  int64_t home_rows;          /* rows of this rank's home buffers */
  int64_t q_rows[2];          /* server Q rows per half */
  int64_t kv_rows[2];         /* server K/V rows per half */
  int64_t n_tasks[2];         /* CA-tasks served per half */
  int64_t served_pairs;       /* exact causal pairs this rank computes */
  int64_t wire_bytes[2][4];   /* bytes this rank puts on the wire per half and
                                 CAD_XFER_* of one layer (remote peers only;
                                 Q/KV count one tensor: x2 for K+V / Q+dO) */
  int64_t blob_bytes;         /* size of cad_layer_ctx_export's blob */
  int64_t launches;           /* kernels this context launched so far */
} cad_layer_ctx_info;

/* Caller buffers of one step on this rank's HOME rows (packed THD, the row
 * order of the rank's home items): inputs q/dout [home_rows][h_q][d], k/v
 * [home_rows][h_kv][d] bf16 (NULL: already in cad_layer_ctx_home's
 * buffers); outputs o/dq bf16 and lse [h_q][home_rows] fp32 (copied out of
 * the home buffers when non-NULL and not those buffers), dk/dv bf16 and/or
 * their fp32 sums dk_acc/dv_acc [home_rows][h_kv][d] (each written when
 * non-NULL). A backward-only step (CAD_PASS_BWD) reads o/lse as inputs. */
typedef struct cad_layer_io {
  const void* q;
  const void* k;
  const void* v;
  const void* dout;
  void* o;
  float* lse;
  void* dq;
  void* dk;
  void* dv;
  float* dk_acc;
  float* dv_acc;
} cad_layer_io;

/* Builds every rank's row plan (deterministic; cad_layer_plan_create_ex for
 * each rank), the server CA plans of both halves and the server buffers on
 * the current device. */
int cad_layer_ctx_create(const cad_plan* plan, const cad_item* home_items,
                         int64_t n_items, const cad_layer_cfg* cfg,
                         cad_layer_ctx** out);
int cad_layer_ctx_info_get(const cad_layer_ctx* ctx, cad_layer_ctx_info* info);
/* The home buffers of a layer, INSIDE the context's server buffers (zero-copy
 * own rows: a rank's own tasks read Q/K/V/dO and write O/dQ there in place,
 * and the peers push their returns there). Callers that produce inputs or
 * consume outputs in place use these pointers (and may pass NULL inputs in
 * cad_layer_io); other caller buffers are copied in at the start of a step and
 * out at its finish. With stacked benchmark layers, layer l >= 1 reads its
 * own home inputs unless cad_layer_io gives buffers (then copied into every
 * layer). */
int cad_layer_ctx_home(const cad_layer_ctx* ctx, int32_t layer, cad_layer_io* io);
/* Kept for the earlier contract (outputs bound up front): now a no-op; the
 * outputs live in the context and cad_layer_io's o/lse/dq receive copies. */
int cad_layer_ctx_bind_outputs(cad_layer_ctx* ctx, void* o, float* lse, void* dq);
/* LOCAL/IPC: this rank's buffer references (blob of info.blob_bytes). Gather
 * every rank's blob (any host collective), then connect with the
 * concatenation in rank order. */
int cad_layer_ctx_export(cad_layer_ctx* ctx, void* blob, size_t cap, size_t* need);
int cad_layer_ctx_connect(cad_layer_ctx* ctx, const void* blobs, size_t blob_bytes);
/* NCCL: the communicator of this rank (not owned). */
int cad_layer_ctx_set_comm(cad_layer_ctx* ctx, cad_comm* comm);
int cad_layer_ctx_destroy(cad_layer_ctx* ctx);

/* The per-layer entry points (cad_dispatch / cad_return).
 * A step is: cad_layer_begin, then in dependency order per (layer, half)
 * dispatch(QKV) -> compute(fwd) -> return(O), dispatch(DO) ->
 * compute(bwd) -> return(GRAD), then cad_layer_finish. Cross-rank ordering
 * is the context's job (GPU flags for LOCAL/IPC, the collective for NCCL);
 * ordering between the caller's streams on one rank is the caller's
 * (cad_layer_step does both). NCCL: every transport call of one context must
 * go to one stream. */
#define CAD_DISPATCH_QKV 0 /* Q, K, V rows: home -> servers (forward)  */
#define CAD_DISPATCH_DO 1  /* dO rows: home -> servers (backward)      */
#define CAD_DISPATCH_FWD_STATE 2 /* O rows + LSE: home -> servers, for a
                                    backward whose forward ran under another
                                    plan (a pipeline tick, sim.cpp:326-353);
                                    issue before the DO dispatch */
#define CAD_RETURN_O 0     /* O rows + LSE: servers -> home            */
#define CAD_RETURN_GRAD 1  /* dQ rows -> home, dK/dV partials -> owners */
int cad_layer_begin(cad_layer_ctx* ctx, void* stream);
/* Passes of a step: forward and backward (the default), or one of them (a
 * pipeline tick runs one pass per tick; layers == 1). A forward-only step
 * ends once the O/LSE returns arrived; a backward-only step dispatches Q/K/V,
 * the forward state (O, LSE) and dO, and sums the dK/dV partials. */
#define CAD_PASS_FWD 1
#define CAD_PASS_BWD 2
#define CAD_PASS_BOTH 3
int cad_layer_begin_ex(cad_layer_ctx* ctx, int32_t passes, void* stream);
int cad_dispatch(cad_layer_ctx* ctx, int32_t layer, int32_t half, int32_t what,
                 const cad_layer_io* io, void* stream);
/* Same, with this rank's own rows (tasks it serves itself) copied on
 * local_stream (LOCAL/IPC; cad_layer_step puts them on the compute stream). */
int cad_dispatch_ex(cad_layer_ctx* ctx, int32_t layer, int32_t half, int32_t what,
                    const cad_layer_io* io, void* stream, void* local_stream);
int cad_layer_compute(cad_layer_ctx* ctx, int32_t layer, int32_t half,
                      int32_t backward, void* stream);
int cad_return(cad_layer_ctx* ctx, int32_t layer, int32_t half, int32_t what,
               const cad_layer_io* io, void* stream);
/* Waits for every return addressed to this rank and sums, per home KV row,
 * the dK/dV partials of every server that used it (fp32, no atomics) into
 * dk/dv (bf16) and/or dk_acc/dv_acc (fp32). */
int cad_layer_finish(cad_layer_ctx* ctx, const cad_layer_io* io, void* stream);

/* One whole step (all layers, forward + backward) on `stream` (compute) and
 * the context's comm stream, in the reference's ping-pong windows. IPC and
 * NCCL transports (one process per rank); LOCAL only in COMPUTE mode. */
#define CAD_STEP_PINGPONG 0 /* comm of one half under CA of the other */
#define CAD_STEP_SERIAL 1   /* everything on `stream`, no overlap */
#define CAD_STEP_COMPUTE 2  /* CA kernels only (server buffers as resident) */
#define CAD_STEP_COMM 3     /* exchanges only, no CA kernels */
#define CAD_STEP_SIGNAL 4   /* ping-pong with every flag, the rank's own
                               rows and the dK/dV reduction, but every
                               transfer to a peer shrunk to its flag (the
                               reference's signal mode, sim.hpp:14-18;
                               IPC only) */
#define CAD_STEP_COMM_LOCAL 5 /* COMM without the transfers to peers: the
                                 rank's own rows and the reduction only */
int cad_layer_step(cad_layer_ctx* ctx, const cad_layer_io* io, int32_t mode,
                   void* stream);
int cad_layer_step_ex(cad_layer_ctx* ctx, const cad_layer_io* io, int32_t mode,
                      int32_t passes, void* stream);

/* Timeline of the last cad_layer_step (tracing on): one record per phase,
 * times in ms from the step's start on its compute stream. For FWD/BWD,
 * t_ready is when the inputs had arrived (flags/events satisfied). */
#define CAD_TRACE_DISPATCH_QKV 0
#define CAD_TRACE_DISPATCH_DO 1
#define CAD_TRACE_FWD 2
#define CAD_TRACE_BWD 3
#define CAD_TRACE_RETURN_O 4
#define CAD_TRACE_RETURN_GRAD 5
#define CAD_TRACE_FINISH 6
typedef struct cad_trace_rec {
  int32_t kind;
  int32_t layer;
  int32_t half;
  int32_t pad_;
  float t_begin;
  float t_ready;
  float t_end;
  float pad2_;
} cad_trace_rec;
int cad_layer_ctx_set_trace(cad_layer_ctx* ctx, int32_t on);
int cad_layer_ctx_trace(cad_layer_ctx* ctx, cad_trace_rec* recs, int64_t cap, int64_t* n);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* CAD_H_ */
