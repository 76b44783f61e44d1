/*
 * rlx.h — C-ABI of the B200 look-ahead candidate evaluator.
 *
 * The reference (`rlmux`, pure Python) has no FFI; its de-facto seam for
 * this hot path is the chooser callable handed to `_drive`
 * (rlmux/scheduler.py:925-950, chooser at :963-972) together with the
 * module-global `enumerate_actions` (:648-703) it scores through
 * `candidate_cost` (:902-918) and `action_finish_estimate` (:773-789).
 * These entry points replace exactly that seam:
 *
 *   rlx_open / rlx_close           handle + device buffers (one handle per GPU / rank)
 *   rlx_load_instance              static per-instance data: pipelines, knobs, slowdown
 *                                  LUT (replaces SlowdownModel.slowdown, slowdown.py:129-156)
 *   rlx_decide                     one chooser call: enumerate + score + argmin over a
 *                                  serial range (replaces scheduler.py:939-940 and :963-972)
 *   rlx_decode                     serial -> action (so every rank can materialise the
 *                                  global winner after the cross-GPU min-loc)
 *   rlx_set_stream                 order the handle's work on a caller stream
 *   rlx_last_error                 text of the last failure
 *   rlx_drive                      the whole decision loop `_drive` (:925-950) behind
 *                                  the ABI: plan -> score -> apply winner -> advance
 *   rlx_plan_info                  host-only planning of one decision (candidate counts,
 *                                  capacity checks) — no device needed
 *
 * and the reference's mutable execution state `ExecState` (:339-634), held
 * natively (one RlxState per simulated run; no device needed):
 *
 *   rlx_state_create / _clone / _destroy   ExecState(instance, record) / clone()
 *   rlx_state_apply                 ExecState.apply (:486-515, merge surgery :517-581)
 *   rlx_state_advance               ExecState.advance(until) (:593-627)
 *   rlx_state_info / _node / _events / _completion   queries
 *   rlx_state_snapshot              the RlxStateDesc view rlx_decide consumes
 *
 * All arrays are plain host pointers owned by the caller and only read
 * during the call. Times are IEEE-754 binary64 seconds; every cost/finish
 * value is bit-identical to the reference's Python float arithmetic.
 */
#ifndef RLX_H
#define RLX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RLX_ABI_VERSION 4

/* Kind codes = declaration order of rlmux SubStageKind (graph.py:69-76). */
enum {
  RLX_KIND_PREFILL_BURST = 0,
  RLX_KIND_DECODE_LARGE = 1,
  RLX_KIND_DECODE_MEDIUM = 2,
  RLX_KIND_DECODE_SMALL = 3,
  RLX_KIND_REFERENCE = 4,
  RLX_KIND_TRAINING = 5,
  RLX_KIND_TOOL_WAIT = 6,
  RLX_NKIND = 7
};

/* Allocation index space of the slowdown LUT.
 *   0            FULL_ALLOCATION (1.0, 0.8)                       slowdown.py:52
 *   1 + 4*i + j  Multiplex alloc (MUX_SM_GRID[i], MEM_GRID[j])    scheduler.py:46, :671-675
 *   13 + 4*i + j complement_allocation of the above                slowdown.py:169-175
 * LUT layout: lut[(kind * 8 + partner) * RLX_NALLOC + alloc], partner 0 = None,
 * partner k+1 = kind k. A NaN entry marks a (kind, partner) pair missing from
 * the table (the reference raises KeyError on use, slowdown.py:143-147). */
#define RLX_NALLOC 25
#define RLX_NPARTNER 8

/* Candidate classes = reference priorities (scheduler.py:644). */
enum { RLX_CLASS_MULTIPLEX = 0, RLX_CLASS_MERGE = 1, RLX_CLASS_EXCLUSIVE = 2 };

/* Status codes. */
enum {
  RLX_OK = 0,
  RLX_ERR_ARG = 1,         /* bad argument / malformed state                       */
  RLX_ERR_CUDA = 2,        /* CUDA runtime / device failure                        */
  RLX_ERR_SCHEDULING = 3,  /* reference SchedulingError (e.g. window guard, :866) */
  RLX_ERR_KEY = 4,         /* reference KeyError (missing slowdown row / latency)  */
  RLX_ERR_LIMIT = 5,       /* outside this build's compiled limits                 */
  RLX_ERR_VALUE = 6        /* reference ValueError                                 */
};

#define RLX_MAX_MEMBERS 64

typedef struct RlxInstanceDesc {
  int32_t abi_version;           /* = RLX_ABI_VERSION */
  int32_t n_pipes;
  const char* pipe_names;        /* NUL-separated pipeline ids, pipe p at pipe_name_off[p] */
  const int32_t* pipe_name_off;
  const double* latency;         /* [n_pipes*3] latency_model[bucket] for buckets 0..2     */
  const uint8_t* latency_ok;     /* [n_pipes*3] 1 if that bucket key exists              */
  const uint8_t* has_spec;       /* [n_pipes] PipelineSpec present                        */
  const double* model_params;    /* [n_pipes]                                             */
  const double* peak_flops;      /* [n_pipes]                                             */
  const double* prefill_mfu;     /* [n_pipes]                                             */
  int32_t n_workers;
  const int32_t* worker_ids;     /* [n_workers] ascending (Instance.workers(), :135-139)  */
  double headroom;
  double realloc_penalty;
  double default_migration_cost;
  int32_t merge_enabled;
  int32_t _pad;
  const double* lut;             /* [RLX_NKIND * RLX_NPARTNER * RLX_NALLOC]               */
  const double* alloc_sm;        /* [RLX_NALLOC] sm share of each allocation index        */
  const double* alloc_mem;       /* [RLX_NALLOC] mem share of each allocation index       */
} RlxInstanceDesc;

/* Snapshot of ExecState (scheduler.py:339-366) at a decision point.
 * Nodes are the alive sub-stages (completed ones included); node index =
 * position in these arrays. */
typedef struct RlxStateDesc {
  double now;
  int32_t n_nodes;
  int32_t n_edges;
  const int32_t* pipe;           /* [n] pipeline index                                    */
  const int32_t* worker;         /* [n] dense worker index into worker_ids                */
  const int32_t* kind;           /* [n] RLX_KIND_*                                        */
  const double* duration;        /* [n]                                                   */
  const double* mem;             /* [n] mem_fraction                                      */
  const int64_t* remaining;      /* [n] remaining_decode_tokens                           */
  const int64_t* active;         /* [n] active_requests                                   */
  const int64_t* context;        /* [n] context_tokens                                    */
  const uint8_t* completed;      /* [n]                                                   */
  const double* merge_prefix;    /* [n] pending merge prefix (0 if none)                  */
  const char* ids;               /* NUL-separated node ids                                */
  const int32_t* id_off;         /* [n]                                                   */
  const int32_t* edge_src;       /* [n_edges]                                             */
  const int32_t* edge_dst;       /* [n_edges]                                             */
  int32_t n_running;
  int32_t n_toolwaits;
  const int32_t* run_node;       /* [n_running]                                           */
  const int32_t* run_partner;    /* [n_running] node index of the partner, -1 if none     */
  const double* run_rate;
  const double* run_prefix;
  const double* run_work;
  const int32_t* tw_node;        /* [n_toolwaits] running tool waits                      */
  const double* tw_end;
  int32_t n_grants;              /* last_mem_grant entries (realloc penalty)              */
  int32_t _pad;
  const int32_t* grant_worker;   /* dense worker index                                    */
  const int32_t* grant_pipe;
  const double* grant_mem;
} RlxStateDesc;

typedef struct RlxDecideArgs {
  int32_t window;                /* look-ahead depth W >= 1                               */
  int32_t max_merge;             /* merge-set size cap; <= 0 means uncapped (reference)   */
  int64_t serial_begin;          /* shard [begin, end) of the global serial range;        */
  int64_t serial_end;            /*   end < 0 means "to the last candidate"               */
  double* keys_out;              /* optional host [2*(end-begin)]: (cost, finish) per     */
                                 /*   candidate, for parity tests                         */
  void* dev_key_out;             /* optional DEVICE pointer to 5 x uint64 that receives   */
                                 /*   the shard's packed best key (RlxKey) and, in word 4, */
                                 /*   its lowest failing candidate (serial << 8 | device  */
                                 /*   error code; ~0: none) — the row of the NCCL min-loc */
  int32_t flags;                 /* RLX_F_*                                               */
  int32_t _pad;
} RlxDecideArgs;

#define RLX_F_NO_SYNC_STATS 1     /* skip the stats readback */
#define RLX_F_REUSE_PLAN 2        /* re-score the plan already resident on the device   */
                                  /*   (state may be NULL; no planning, no H2D copy)     */
#define RLX_F_SHARD 4             /* serial_begin/serial_end = part index r / part count w: */
                                  /*   score every w-th block of 32 serials of each class */
                                  /*   (multiplex, merges, exclusive), starting at block r */
                                  /*   — cost-balanced multi-GPU shards (dist.part_serials) */

/* Packed key: cost and finish are non-negative doubles, so their bit
 * patterns order as uint64; word 2 = priority << 61 | serial; word 3 = 1 if
 * valid. Lexicographic order over words 0..2 == the reference's
 * (cost, finish, priority, serial) tuple order (scheduler.py:969). */
typedef struct RlxKey {
  uint64_t cost_bits;
  uint64_t finish_bits;
  uint64_t prio_serial;
  uint64_t valid;
} RlxKey;

typedef struct RlxAction {
  int32_t cls;                   /* RLX_CLASS_*                                           */
  int32_t node_a;                /* Exclusive node / Multiplex first                      */
  int32_t node_b;                /* Multiplex second                                      */
  int32_t alloc;                 /* alloc index of node_a (0 for Exclusive)               */
  int32_t target_worker;         /* Merge target (dense worker index)                     */
  int32_t n_members;             /* Merge members, node indices in sorted-id order        */
  int32_t members[RLX_MAX_MEMBERS];
} RlxAction;

typedef struct RlxDecision {
  int64_t n_candidates;          /* total candidates at this decision (all shards)        */
  int32_t found;                 /* shard had >= 1 candidate                              */
  int32_t priority;
  int64_t serial;
  double cost;
  double finish;
  RlxAction action;              /* decoded winner of this shard                          */
  RlxKey key;
  /* measurement */
  int64_t passes;                /* list-scheduling passes run                            */
  double alg_bytes;              /* SURVEY §8(d) algorithmic bytes of the scored shard    */
  double kernel_ms;              /* device time of the scoring kernel (CUDA events)       */
  double plan_ms;                /* host planning time                                    */
  int64_t n_merge, n_multiplex, n_exclusive;
  double device_ms;              /* device time from plan upload to the reduced key       */
  int64_t h2d_bytes;             /* plan bytes copied host -> device by this call         */
  int64_t d2h_bytes;             /* result bytes copied device -> host                    */
  int64_t shard_begin, shard_end;/* serial range actually scored                          */
  int64_t events;                /* simulated events (advances) over all passes           */
  int64_t err_key;               /* lowest failing candidate of the shard: serial << 8 |  */
                                 /*   device error code, or -1 (rlx_error_text)           */
} RlxDecision;

/* ---- native execution state (ExecState) ------------------------------ */

/* Static sub-stage graph of an instance: every pipeline graph's nodes in
 * Instance.graphs order, then each graph's node insertion order (the
 * reference's ExecState dict order, scheduler.py:348-356). */
typedef struct RlxGraphDesc {
  int32_t n_nodes;
  int32_t n_edges;
  const int32_t* pipe;           /* [n] pipeline index                                    */
  const int32_t* worker;         /* [n] dense worker index                                */
  const int32_t* kind;           /* [n] RLX_KIND_*                                        */
  const double* duration;
  const double* mem;
  const int64_t* remaining;
  const int64_t* active;
  const int64_t* context;
  const int64_t* token_total;
  const int64_t* span_lo;        /* step_span                                             */
  const int64_t* span_hi;
  const char* ids;               /* NUL-separated node ids                                */
  const int32_t* id_off;
  const int32_t* edge_src;
  const int32_t* edge_dst;
} RlxGraphDesc;

/* One action to apply (node indices are RlxState node indices). Rates are
 * the slowdown factors of the allocation (SlowdownModel.slowdown); NaN
 * marks a missing table row, reported as RLX_ERR_KEY after validation, in
 * the reference's order (scheduler.py:486-505). */
typedef struct RlxApply {
  int32_t cls;                   /* RLX_CLASS_*                                           */
  int32_t node_a, node_b;
  int32_t target_worker;         /* Merge: dense worker index                             */
  int32_t n_members;
  int32_t _pad;
  int32_t members[RLX_MAX_MEMBERS];
  double rate_a, rate_b;
  double sm_a, mem_a, sm_b, mem_b;
} RlxApply;

typedef struct RlxStateInfo {
  double now;
  double makespan;
  int32_t n_total;               /* node slots (dead merge members included)              */
  int32_t n_alive;
  int32_t n_done;
  int32_t done;
  int32_t has_events;
  int32_t n_running;
  int32_t n_toolwaits;
  int32_t _pad;
  int64_t revision;              /* bumped by every merge (structure change)              */
  int64_t n_events;              /* recorded events (record=1)                            */
} RlxStateInfo;

typedef struct RlxNodeInfo {
  int32_t pipe, worker, kind, alive, completed, running;
  double duration, mem, completion_time;
  int64_t remaining, active, context, token_total, span_lo, span_hi;
  const char* id;                /* owned by the state                                    */
} RlxNodeInfo;

/* Recorded event (scheduler.py:389-391; kinds as rlmux/sim.py:45). */
enum { RLX_EV_START = 0, RLX_EV_FINISH = 1, RLX_EV_RERATE = 2, RLX_EV_MERGE = 3, RLX_EV_MIGRATION = 4,
       RLX_EV_TOOLWAIT_START = 5 };
typedef struct RlxEvent {
  double time;
  int32_t worker;                /* dense worker index                                    */
  int32_t kind;                  /* RLX_EV_*                                              */
  int32_t node;
  int32_t _pad;
  double sm, mem;                /* allocation of start / rerate events (NaN otherwise)   */
} RlxEvent;

int rlx_state_create(const RlxInstanceDesc* inst, const RlxGraphDesc* graph, int record, void** state);
int rlx_state_clone(const void* state, void** out);
void rlx_state_destroy(void* state);
const char* rlx_state_error(const void* state);
int rlx_state_apply(void* state, const RlxApply* action);
int rlx_state_advance(void* state, int has_until, double until);
int rlx_state_info(const void* state, RlxStateInfo* out);
/* Fills `out` with views of the state's own arrays, valid until the next
 * mutation of the state. */
int rlx_state_snapshot(void* state, RlxStateDesc* out);
int rlx_state_node(const void* state, int32_t node, RlxNodeInfo* out);
int rlx_state_events(const void* state, int64_t first, int64_t count, RlxEvent* out);
int rlx_state_completion(const void* state, uint8_t* completed /* [n_total] */, double* times /* [n_total] */);

/* ---- the whole decision loop behind the ABI --------------------------- */

typedef struct RlxDriveArgs {
  int32_t window;
  int32_t max_merge;             /* <= 0: uncapped                                        */
  int64_t max_decisions;         /* stop after this many chooser calls (<= 0: run to done) */
  int64_t max_steps;             /* capacity of the `steps` array                         */
} RlxDriveArgs;

/* One applied action of the schedule (TimedAction) plus its decision. */
typedef struct RlxStep {
  double start;                  /* state.now when the action was applied                 */
  RlxAction action;              /* node indices = RlxState node indices                  */
  double cost, finish;           /* winning key                                           */
  int32_t priority;
  int32_t _pad;
  int64_t serial;
  int64_t n_candidates;
  double decision_ms;            /* host state in -> winner applied (wall clock)          */
  double kernel_ms;              /* scoring kernel (CUDA events)                          */
} RlxStep;

/* `_drive(instance, chooser, ...)` (scheduler.py:925-950) with the device
 * chooser: repeat { plan + score + argmin on the GPU; apply the winner to
 * `state` } until no candidate, then advance; until the state is done.
 * Writes the applied actions to `steps` (*n_steps of them) and the number
 * of chooser calls (decisions with >= 1 candidate) to *n_decisions. On a
 * failure the steps applied so far stay valid. */
int rlx_drive(void* handle, void* state, const RlxDriveArgs* args, RlxStep* steps, int64_t* n_steps,
              int64_t* n_decisions);

/* Host-only planning of one decision (no device, no handle): candidate
 * counts and the plan's sizes, or the capacity error the device path would
 * report (RLX_ERR_LIMIT) with its text in `err`. */
typedef struct RlxPlanInfo {
  int64_t n_candidates, n_multiplex, n_merge, n_exclusive;
  int32_t window_nodes;          /* |window| (N_w)                                        */
  int32_t local_nodes;           /* window + auxiliary tool waits                         */
  int32_t max_worker_order;      /* longest per-worker ready order (ready-mask bits)      */
  int32_t hot_bytes;             /* plan bytes staged into shared memory                  */
  int64_t blob_bytes;            /* plan bytes copied host -> device                      */
} RlxPlanInfo;
int rlx_plan_info(const RlxInstanceDesc* inst, const RlxStateDesc* state, int32_t window, int32_t max_merge,
                  RlxPlanInfo* out, char* err, int32_t err_len);

/* ---- Sub-Stage Graph construction from rollout length tables ---------- */

/* One pipeline's sample batch (rlmux PipelineSpec.samples, workload.py:59-110):
 * per sample its prompt and turns (prefill tokens injected at the turn,
 * decode tokens, tool latency after the turn); samples are assigned to
 * workers round-robin (workload.py round_robin_assignment) unless
 * `worker_of` is given. Replaces expand_to_trace + construct_graph's
 * rollout part (workload.py:275-392, graph.py:206-362). */
typedef struct RlxRolloutTables {
  int32_t n_samples;
  int32_t n_workers;             /* dp workers                                            */
  const int32_t* worker_of;      /* [n_samples] or NULL (sample i -> worker i % n_workers) */
  const int64_t* prompt;         /* [n_samples]                                           */
  const int32_t* turn_off;       /* [n_samples + 1] CSR into the turn arrays              */
  const int64_t* turn_prefill;   /* [n_turns]                                             */
  const int64_t* turn_decode;    /* [n_turns]                                             */
  const double* turn_tool;       /* [n_turns] tool latency after the turn (0: none)       */
  double latency[5];             /* per-step latency: buckets 0..2, reference, training   */
} RlxRolloutTables;

/* One rollout sub-stage: worker `worker`, sequence `seq` (id
 * "<pipeline>/w<worker>/r<seq:03d>"), in worker order then sequence order. */
typedef struct RlxSegment {
  int32_t worker, seq;
  int32_t kind;                  /* RLX_KIND_* (PrefillBurst / Decode* / ToolWait)        */
  int32_t bucket;                /* stable token bucket, -1 for a tool wait               */
  int64_t step_lo, step_hi;      /* step_span                                             */
  int64_t decode;                /* remaining_decode_tokens                               */
  int64_t active0;               /* active_requests (first step)                          */
  int64_t context0;              /* context_tokens (first step; 0 for a tool wait)        */
  int64_t tokens;                /* token_total                                           */
  double duration;               /* steps x latency[bucket] (tool wait: x latency[0])     */
} RlxSegment;

/* Replay every (pipeline, worker) cohort and segment its step records on
 * `device` (stability window L_s = `window`, bucket lower bounds
 * `bucket_bounds[0..n_buckets)` starting at 0, n_buckets <= 5). The result
 * handle holds each pipeline's segments (rlx_graph_segments). */
int rlx_graph_build(int device, int32_t n_pipes, const RlxRolloutTables* tables, const int32_t* bucket_bounds,
                    int32_t n_buckets, int32_t window, void** result);
int rlx_graph_segments(void* result, int32_t pipe, RlxSegment* out, int64_t cap, int64_t* n_out);
int rlx_graph_stats(void* result, double* kernel_ms, int64_t* n_records);
const char* rlx_graph_error(void* result);
void rlx_graph_free(void* result);

/* ---- batched replay of schedules into metrics (rlmux/sim.py:69-173) ---- */

/* One timed action of a schedule: node ids are NUL-terminated strings in a
 * shared blob (`n_ids` consecutive ones from `id_off`: Exclusive 1,
 * Multiplex 2, Merge the members); `sm`/`mem` the allocation of node a;
 * `target_worker` the Merge target (external worker id). */
typedef struct RlxSimAction {
  double start;
  double sm, mem;
  int32_t cls;                   /* RLX_CLASS_*                                           */
  int32_t target_worker;
  int32_t n_ids;
  int32_t id_off;
} RlxSimAction;

typedef struct RlxSimResult {
  int32_t status;                /* RLX_OK, or the status simulate() raises with          */
  int32_t action_index;          /* failing action (n: the final drain), -1 if none       */
  double makespan;
  double throughput;             /* aggregate_throughput                                  */
  int64_t total_tokens;
  char error[192];               /* the reference's message                               */
} RlxSimResult;

/* Replay schedules [s] = actions [sched_off[s], sched_off[s+1]) on copies of
 * the instance's initial ExecState, over `n_threads` host threads (<= 0: all).
 * Outputs per schedule: result, per-pipeline latency / tokens [n_sched * P]
 * (pipelines in instance order) and per-worker average utilisation
 * [n_sched * W] (dense worker order). Allocations must be in the instance's
 * LUT (RLX_ERR_LIMIT otherwise). */
int rlx_simulate_batch(const RlxInstanceDesc* inst, const RlxGraphDesc* graph, int32_t n_sched,
                       const int64_t* sched_off, const RlxSimAction* actions, const char* ids, int32_t n_threads,
                       RlxSimResult* results, double* pipe_latency, int64_t* pipe_tokens, double* util_avg);

/* ---- brute-force oracle (rlmux/scheduler.py:1086-1226) ------------------ */

/* enumerate_actions (:648-703) on a native state, in serial order: node
 * indices in the state's index space, `alloc` = allocation index. */
int rlx_enumerate(const RlxInstanceDesc* inst, const void* state, RlxAction* out, int64_t cap, int64_t* n_out);
/* brute_force_schedule's search (:1172-1218) from the instance's initial
 * state, seeded with the best seed makespan: depth-first over the
 * deduplicated candidates and one advance, pruned by the bound and the
 * state memo, in the reference's visiting order. `*n_out` = -1 when no
 * schedule beats the seeds by more than EPS, else the winning actions in
 * `out` (node indices of the replayed state, as rlx_drive's steps). */
int rlx_branch_and_bound(const RlxInstanceDesc* inst, const RlxGraphDesc* graph, double best_makespan, int32_t cap,
                         RlxStep* out, int32_t* n_out, double* best_out, int64_t* visited);

int rlx_abi_version(void);
int rlx_open(int device, void** handle);
int rlx_load_instance(void* handle, const RlxInstanceDesc* inst);
int rlx_decide(void* handle, const RlxStateDesc* state, const RlxDecideArgs* args, RlxDecision* out);
int rlx_decode(void* handle, int64_t serial, RlxAction* out);
/* Issue all further work of this handle on `cuda_stream` (a cudaStream_t of
 * the handle's device, e.g. the caller's torch stream, so CUDA events and
 * NCCL calls on that stream order with the scoring kernel); NULL restores
 * the handle's private (non-blocking) stream. To order with the legacy
 * default stream pass cudaStreamLegacy, not NULL. */
int rlx_set_stream(void* handle, void* cuda_stream);
const char* rlx_last_error(void* handle);
/* Status and the reference's message for a device error code (the low byte
 * of RlxDecision.err_key), so every rank of a multi-GPU decision can raise
 * the same exception for the globally lowest failing candidate. */
int rlx_error_text(int32_t device_code, char* buf, int32_t buf_len);
void rlx_close(void* handle);

#ifdef __cplusplus
}
#endif

#endif /* RLX_H */
