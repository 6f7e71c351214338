/* csg_engine.h — C ABI of the B200 trace-analysis engine.
 *
 * The engine is the device half of the drop-in for the reference collsight
 * analyzer (Mycroft Coll-level trigger + root-cause analysis). Everything here
 * is plain C: opaque handles, plain structs, pointers and sizes. No C++ or
 * torch types cross this boundary and no exception escapes it; every call
 * returns a csg_status and csg_last_error() explains a failure.
 *
 * Status codes mirror collsight_status (reference
 * proj/include/collsight/collsight.h:17-23): the reference maps ConfigError
 * to 2, TraceParseError to 3 and every other std::exception (DataError
 * included) to 4 (proj/src/c_api.cpp:34-45).
 *
 * Reference entry point each call replaces is cited per declaration; paths
 * are relative to the reference tree (proj/...).
 */
#ifndef CSG_ENGINE_H_
#define CSG_ENGINE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum csg_status {
  CSG_OK = 0,
  CSG_ERR_CONFIG = 2,  /* ConfigError (proj/include/collsight/types.hpp:46) */
  CSG_ERR_PARSE = 3,   /* TraceParseError (types.hpp:52) */
  CSG_ERR_RUNTIME = 4, /* DataError / CUDA failure / any other error */
  CSG_ERR_ARG = 5      /* null or invalid argument */
} csg_status;

/* ---------------------------------------------------------------------------
 * Packed trace record (48 bytes), the device wire format.
 *
 * A lossless re-encoding of every field the analyzer reads from the
 * reference's CompletionRecord / StateRecord
 * (proj/include/collsight/trace.hpp:19-46): the timestamp() accessor value
 * (end_ms | window_end_ms, proj/src/trace.cpp:35-37), comm_id, rank, channel,
 * op_seq, the record kind, and the kind's payload. node, stuck_ms and
 * total_chunks are validated at parse time but never read by the analyzer
 * and are not carried. State counters travel as u32 (range-checked by the
 * packer; a counter >= 2^32 is rejected with CSG_ERR_RUNTIME).
 * ------------------------------------------------------------------------- */
enum { CSG_KIND_COMPLETION = 0, CSG_KIND_STATE = 1 };
/* OpName order of proj/include/collsight/types.hpp:35-41 */
enum {
  CSG_OP_ALLGATHER = 0,
  CSG_OP_REDUCESCATTER = 1,
  CSG_OP_ALLREDUCE = 2,
  CSG_OP_SEND = 3,
  CSG_OP_RECV = 4
};

typedef struct csg_packed_record {
  double ts;        /* end_ms (completion) | window_end_ms (state) */
  int64_t op_seq;
  int32_t rank;
  int32_t comm_id;
  int32_t channel;
  uint8_t kind;     /* CSG_KIND_* */
  uint8_t op_name;  /* CSG_OP_* for completions, 0 for states */
  uint16_t reserved;
  union {
    struct {
      double start_ms;
      uint64_t msg_bytes;
    } c;
    struct {
      uint32_t gpu_ready;
      uint32_t rdma_transmitted;
      uint32_t rdma_done;
      uint32_t reserved;
    } s;
  } u;
} csg_packed_record;

/* ---------------------------------------------------------------------------
 * Layout + program tables (the read-only tables the RCA walks).
 * Mirrors Topology::groups (proj/include/collsight/topology.hpp:15-55) and
 * OpProgram (proj/include/collsight/program.hpp:14-30). Groups are indexed
 * by comm_id (comm_id == index, as in the reference). Members are in ring
 * order.
 * ------------------------------------------------------------------------- */
enum { CSG_GROUP_DP = 0, CSG_GROUP_PP = 1, CSG_GROUP_TP = 2 };

typedef struct csg_topology_desc {
  int32_t world_size;        /* Topology::world_size() = tp*pp*dp */
  int32_t n_groups;
  const uint8_t* group_kind; /* [n_groups] CSG_GROUP_* */
  const int64_t* member_off; /* [n_groups+1] */
  const int32_t* members;    /* [member_off[n_groups]] ring order */
} csg_topology_desc;

typedef struct csg_program_desc {
  int32_t n_ops;           /* ops_per_iteration; op_seq == index */
  const uint8_t* op_name;  /* [n_ops] CSG_OP_* */
  const int32_t* group;    /* [n_ops] comm_id */
  const int32_t* src;      /* [n_ops] Send/Recv endpoints, -1 otherwise */
  const int32_t* dst;      /* [n_ops] */
  const int64_t* dep_off;  /* [n_ops+1] */
  const int64_t* deps;     /* [dep_off[n_ops]] depends_on, earlier seqs */
} csg_program_desc;

/* TriggerConfig (proj/include/collsight/trigger.hpp:15-25) */
typedef struct csg_trigger_config {
  double delta_ms;
  double detect_interval_ms;
  double throughput_drop_factor;
  double interval_inflation_factor;
  int32_t max_sampled_ranks;
  int32_t warmup_windows;
  double ema_alpha;
} csg_trigger_config;

/* AnalysisConfig (proj/include/collsight/rca.hpp:42-49) */
typedef struct csg_analysis_config {
  double straggler_threshold_ms;
  double delta_ms;
  double flow_skew_factor;
  int32_t consecutive_iterations_k;
  int32_t reserved;
} csg_analysis_config;

void csg_trigger_config_default(csg_trigger_config* out);
void csg_analysis_config_default(csg_analysis_config* out);

/* ---------------------------------------------------------------------------
 * Reports. Enum values follow proj/include/collsight/rca.hpp:16-37 and
 * trigger.hpp:37.
 * ------------------------------------------------------------------------- */
enum { CSG_TRIGGER_FAILURE = 0, CSG_TRIGGER_STRAGGLER = 1 };
enum {
  CSG_RC_UNINITIALIZED_OR_BLOCKED = 0,
  CSG_RC_RDMA_ISSUE_OR_RECEIVER_NOT_READY = 1,
  CSG_RC_RDMA_ISSUE_OR_RECEIVER_FAILED = 2,
  CSG_RC_GPU_ISSUE = 3,
  CSG_RC_STRAGGLER_LATE_START = 4,
  CSG_RC_STRAGGLER_LATE_END = 5,
  CSG_RC_FLOW_INCOMPLETE = 6,
  CSG_RC_FLOW_SKEWED = 7
};
enum { CSG_SIDE_LOCAL = 0, CSG_SIDE_REMOTE = 1, CSG_SIDE_UNDETERMINED = 2 };
enum {
  CSG_VERDICT_SUSPECTS = 0,
  CSG_VERDICT_UNDETERMINED = 1,
  CSG_VERDICT_FALSE_TRIGGER = 2,
  CSG_VERDICT_INSUFFICIENT_HISTORY = 3,
  CSG_VERDICT_NO_STRAGGLER = 4
};

typedef struct csg_trigger_event { /* TriggerEvent, trigger.hpp:39-43 */
  int32_t kind;
  int32_t suspect_rank;
  double time_ms;
} csg_trigger_event;

typedef struct csg_suspect { /* SuspectEntry, rca.hpp:58-65 */
  int32_t rank;
  uint8_t category;
  uint8_t side;
  uint16_t reserved;
  int32_t group;
  int32_t reserved2;
  int64_t stuck_op;
  double onset_ms;
} csg_suspect;

typedef struct csg_evidence { /* EvidenceRef, rca.hpp:67-72 */
  int32_t rank;
  int32_t channel;
  double time_ms;
  int64_t op_seq;
} csg_evidence;

typedef struct csg_report_view { /* RootCauseReport, rca.hpp:74-82 */
  int32_t verdict;
  csg_trigger_event trigger;
  const csg_suspect* suspects;
  size_t n_suspects;
  const csg_suspect* exonerated;
  size_t n_exonerated;
  const int32_t* affected_groups;
  size_t n_affected;
  const csg_evidence* evidence;
  size_t n_evidence;
  uint64_t records_scanned;
} csg_report_view;

typedef struct csg_progress { /* ProgressTriple, rca.hpp:85-89 */
  uint64_t gpu_ready;
  uint64_t rdma_transmitted;
  uint64_t rdma_done;
} csg_progress;

/* ---------------------------------------------------------------------------
 * Handles
 * ------------------------------------------------------------------------- */
typedef struct csg_ctx csg_ctx;         /* one device + stream */
typedef struct csg_store csg_store;     /* device-resident TraceStore */
typedef struct csg_model csg_model;     /* device topology/program tables */
typedef struct csg_trigger_state csg_trigger_state; /* TriggerState */
typedef struct csg_results csg_results; /* one or more RootCauseReports */

const char* csg_version(void);
/* Message for the most recent failing call on this thread. */
const char* csg_last_error(void);

/* Device context. `device` is a CUDA ordinal. The context owns one stream;
 * calls on one context are serialized, distinct contexts are independent. */
csg_status csg_ctx_create(int device, csg_ctx** out);
void csg_ctx_free(csg_ctx* ctx);
/* Milliseconds of device time spent in the engine's kernels since the last
 * reset, measured with CUDA events on the context stream; and the number of
 * kernel launches issued. */
csg_status csg_ctx_stats(csg_ctx* ctx, double* device_ms, uint64_t* launches);
void csg_ctx_reset_stats(csg_ctx* ctx);
/* Per-kernel CUDA-event timing on the context stream (off by default).
 * csg_ctx_kernel_stats writes {"kernel": [total_ms, launches], ...} as JSON
 * (NUL-terminated, truncated to cap) and the byte counters of the
 * host<->device copies the engine issued since the last reset. */
csg_status csg_ctx_profile(csg_ctx* ctx, int enable);
csg_status csg_ctx_kernel_stats(csg_ctx* ctx, char* json, size_t cap,
                                uint64_t* h2d_bytes, uint64_t* d2h_bytes);
/* Marks the store's device index stale so the next analysis rebuilds it
 * (the benchmark re-times ingest + index every step). */
csg_status csg_store_invalidate(csg_store* store);

/* Sharded mode: one context per GPU, each store holding
 * the records of a rank range (store order preserved inside a rank). After
 * csg_ctx_comm_init every analysis call on the context combines the shards
 * with NCCL collectives on the context stream and returns the same results
 * on every rank. csg_comm_unique_id is called on one rank and its 128 bytes
 * broadcast to the others (the Python driver uses torch.distributed). */
csg_status csg_comm_unique_id(unsigned char* out, size_t cap);
csg_status csg_ctx_comm_init(csg_ctx* ctx, const unsigned char* id, size_t len,
                             int nranks, int rank);
csg_status csg_ctx_comm_info(csg_ctx* ctx, int* nranks, int* rank,
                             uint64_t* collectives);

/* TraceStore (proj/include/collsight/trace.hpp:101-124).
 * append copies `n` packed records from HOST memory (pinned or pageable)
 * into HBM, in emission order; append_device takes records already in HBM on
 * the context's device. Like TraceStore::append (proj/src/trace.cpp:99) it
 * does not validate the records' invariants. */
csg_status csg_store_create(csg_ctx* ctx, csg_store** out);
csg_status csg_store_reserve(csg_store* store, size_t capacity);
csg_status csg_store_append(csg_store* store, const csg_packed_record* host,
                            size_t n);
csg_status csg_store_append_device(csg_store* store,
                                   const csg_packed_record* device, size_t n);
/* JSONL trace text -> records, parsed on the device (the reference's
 * load_trace_file / parse_trace_text, proj/src/trace.cpp:241-346: one record
 * per non-empty line, in line order). The text streams through pinned
 * staging into HBM and is parsed there. *accepted = 1: the records were
 * appended. *accepted = 0 (status still CSG_OK): some line is outside what
 * the device parser vouches for — invalid input, JSON escapes, unknown or
 * duplicate fields, more than 19 significant digits (see csrc/jsonl.cuh) —
 * or the file cannot be read; the store is unchanged and the caller parses
 * the text with the exact host parser, which raises the reference's error
 * (TraceParseError with its line number) or accepts the trace. */
csg_status csg_store_append_jsonl(csg_store* store, const char* text, size_t len,
                                  int* accepted);
csg_status csg_store_append_jsonl_file(csg_store* store, const char* path,
                                       int* accepted);
/* Known-answer hooks: the host instantiation of the device line parser and
 * of its decimal -> binary64 conversion (1 = accepted, 0 = left to the exact
 * parser). */
int csg_jsonl_parse_line(const char* line, size_t len, csg_packed_record* out);
int csg_jsonl_parse_double(const char* tok, size_t len, double* out);
/* Copies the store's first n packed records back to host memory. */
csg_status csg_store_records(const csg_store* store, csg_packed_record* host, size_t n);
csg_status csg_store_clear(csg_store* store);
size_t csg_store_size(const csg_store* store);
/* Builds the device indices now (otherwise built lazily on first use). */
csg_status csg_store_build_index(csg_store* store);
void csg_store_free(csg_store* store);

/* TraceStore::query (proj/src/trace.cpp:101-119): store indices of the
 * records of `ranks` with t0 <= timestamp <= t1, ordered by (timestamp, rank)
 * and stable on store order. *n_out receives the match count; at most `cap`
 * indices are written. t0 > t1 fails with "query: t0 > t1" (status 4). */
csg_status csg_store_query(csg_store* store, const int32_t* ranks,
                           size_t n_ranks, double t0, double t1,
                           uint64_t* out_idx, size_t cap, size_t* n_out);

/* TraceStore::last_log_per_rank (proj/src/trace.cpp:121-144): per member in
 * order, the max-timestamp record at or before t (the later append wins
 * ties); members with none are omitted. */
csg_status csg_store_last_log_per_rank(csg_store* store,
                                       const int32_t* members,
                                       size_t n_members, double t,
                                       int32_t* out_rank, uint64_t* out_idx,
                                       size_t* n_out);

/* Layout + program tables, uploaded once. */
csg_status csg_model_create(csg_ctx* ctx, const csg_topology_desc* topo,
                            const csg_program_desc* program, csg_model** out);
void csg_model_free(csg_model* model);

/* sample_ranks (proj/src/trigger.cpp:29-55). Host-side: O(G log G). */
csg_status csg_sample_ranks(const csg_model* model, int32_t max_sampled_ranks,
                            uint64_t seed, int32_t* out, size_t cap,
                            size_t* n_out);

/* evaluate (proj/src/trigger.cpp:57-136): one detection tick at t over
 * [t - delta, t] for the sampled ranks, updating `state`. *tripped is 1 and
 * *event filled when a rank tripped. */
csg_status csg_trigger_state_create(csg_ctx* ctx, csg_trigger_state** out);
void csg_trigger_state_free(csg_trigger_state* state);
csg_status csg_evaluate(csg_store* store, const int32_t* sampled,
                        size_t n_sampled, double t, csg_trigger_state* state,
                        const csg_trigger_config* cfg, int* tripped,
                        csg_trigger_event* event);

/* Root-cause analysis of one trigger: analyze / analyze_failure /
 * analyze_straggler (proj/src/rca.cpp:540-884). `mode` selects dispatch:
 * 0 = analyze (by trigger kind), 1 = force failure, 2 = force straggler. */
csg_status csg_analyze(csg_store* store, const csg_model* model,
                       const csg_analysis_config* cfg,
                       const csg_trigger_event* trigger, int mode,
                       csg_results** out);

/* affected_groups (proj/src/rca.cpp:400-461). Sorted comm_ids. */
csg_status csg_affected_groups(csg_store* store, const csg_model* model,
                               const csg_analysis_config* cfg,
                               const csg_trigger_event* trigger,
                               int32_t* out, size_t cap, size_t* n_out,
                               uint64_t* scanned);

/* run_detection (proj/src/runner.cpp:47-81): ticks t = I, 2I, ... <= the
 * store's last timestamp, skipping t < delta; every tripped tick is analyzed.
 * `seed` drives sample_ranks exactly as cfg.sim.seed does in the reference
 * (runner.cpp:63-64). The sampled ranks are written to sampled_out when
 * non-NULL (cap entries at most). */
csg_status csg_run_detection(csg_store* store, const csg_model* model,
                             const csg_trigger_config* tcfg,
                             const csg_analysis_config* acfg, uint64_t seed,
                             csg_results** out, int32_t* sampled_out,
                             size_t sampled_cap, size_t* n_sampled);

size_t csg_results_count(const csg_results* res);
csg_status csg_results_get(const csg_results* res, size_t i,
                           csg_report_view* out);
void csg_results_free(csg_results* res);

/* Pure table functions, shared with the device RCA code
 * (proj/src/rca.cpp:249-316). Host-callable for known-answer tests.
 * check_min_op: returns 1 and fills out (sorted) when a strict minimum
 * exists, 0 when every rank sits on the same op. */
csg_status csg_check_min_op(const int32_t* ranks, const int64_t* ops,
                            size_t n, int32_t* out, size_t* n_out,
                            int* has_min);
csg_status csg_check_min_data(const int32_t* ranks, const csg_progress* prog,
                              size_t n, int32_t* out, size_t* n_out);
csg_status csg_check_rc_table(const csg_progress* counters,
                              const csg_progress* peer, int* category,
                              int* side);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* CSG_ENGINE_H_ */
