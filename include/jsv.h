/*
 * jsv.h -- C ABI of libjsv.so, the sm_100a allocation planner.
 *
 * This is the drop-in boundary for the reference planner hot path
 * (reference pkg/src/sliceserve/planner.py).  The reference has no FFI: its
 * only boundary is the Python API, so every entry point below replaces one
 * Python function and is bound with ctypes by
 * paper_2603_08797_b200/_native.py:
 *
 *   jsv_plan_batch        <- plan()              planner.py:915-957  (T = on: _Search 731-912)
 *                         <- plan_uninformed()   planner.py:973-1110 (T = off)
 *   jsv_max_demand_batch  <- max_demand()        planner.py:1125-1175
 *   jsv_derive            <- derive_configuration() planner.py:243-315
 *                            + validate_configuration() planner.py:329-361
 *   jsv_validate          <- validate_configuration() on a caller-built Configuration
 *   jsv_brute_force       <- brute_force_plan()    planner.py:1191-1272
 *   jsv_pool_dump         <- _Search.pools (Stage 1, _candidate_pool 586-635) for parity tests
 *   jsv_pack              <- placement.pack()      placement.py:163-216 (+ _exact_pack 219-266)
 *   jsv_min_gpus          <- placement.min_gpus()  placement.py:269-290
 *
 * Conventions: plain C types only, caller-owned host buffers, integer status
 * codes (0 = ok) plus jsv_last_error() (thread-local message).  No C++
 * exception crosses this boundary.  All planner arithmetic happens on the GPU;
 * the planner entry points refuse to run without a CUDA device (there is no CPU
 * fallback).  The placement entry points (jsv_pack, jsv_min_gpus) are host
 * code: sequential bitmask tree walks over a plan's few MIG instances.
 *
 * Threading: a context serialises its calls (each entry point taking a
 * jsv_context holds the context's mutex for the whole call), so several host
 * threads may share one; contexts are independent of each other.  A problem
 * belongs to the context it was created on.
 */
#ifndef JSV_H
#define JSV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define JSV_MAX_TASKS 16
#define JSV_MAX_EDGES 32
#define JSV_MAX_PATHS 64
#define JSV_MAX_ITEMS 16   /* items per bundle (exhaustive mode is <= log2(exhaustive_limit)) */
#define JSV_MAX_MIX 8
#define JSV_NUM_SEGMENTS 24

#define JSV_SPACE_A 1u      /* accuracy scaling */
#define JSV_SPACE_S 2u      /* spatial partitioning */
#define JSV_SPACE_T 4u      /* task-graph-informed budgeting */

/* binding-constraint codes (reference planner.py:709 priority order) */
#define JSV_BIND_NONE (-1)
#define JSV_BIND_THROUGHPUT 0
#define JSV_BIND_LATENCY 1
#define JSV_BIND_RESOURCES 2
#define JSV_BIND_ACCURACY 3
#define JSV_BIND_COVERAGE 4

/* status codes */
#define JSV_OK 0
#define JSV_ERR_CUDA 1
#define JSV_ERR_ARG 2
#define JSV_ERR_CAPACITY 3
#define JSV_ERR_NODEV 4
#define JSV_ERR_CONFIG 5

typedef struct jsv_context jsv_context;
typedef struct jsv_problem jsv_problem;

/*
 * Lowered AppSpec + ProfileTable (reference model.py:84-333, profiles.py:39-219).
 * Tasks are indexed by their rank in Python string order of task ids; every
 * string ordering of the reference becomes an integer rank here.
 */
typedef struct {
  int32_t n_tasks, n_edges, n_paths, entry;
  const int32_t* topo;        /* [T] task indices in topological order (model.py:187-203) */
  const int32_t* decl;        /* [T] task indices in declaration order (graph.task_ids) */
  const int32_t* succ_off;    /* [T+1] edge e of task t = succ_off[t]+j, j-th id-sorted successor */
  const int32_t* edge_dst;    /* [E] */
  const int32_t* pred_off;    /* [T+1] */
  const int32_t* pred_edge;   /* [E] edges into t, sources id-sorted (model.py:180-185) */
  const int32_t* path_off;    /* [P+1] paths in graph.paths order (lexicographic) */
  const int32_t* path_task;   /* [sum |p|] */
  const double* path_frac;    /* [P] */
  const int32_t* var_off;     /* [T+1] variants of a task, id-sorted */
  const double* var_acc;      /* [V] */
  const int32_t* var_fac_off; /* [V] factors of variant v: var_fac[var_fac_off[v] + j] */
  const double* var_fac;      /* [sum outdeg] */
  const int32_t* most_acc;    /* [T] local index of Task.most_accurate (model.py:78-81) */
  const int32_t* key_off;     /* [T+1] profile keys of a task in (variant, mig, mps, batch) order */
  const int32_t* key_var;     /* [K] local variant index */
  const int32_t* key_seg;     /* [K] segment rank 0..23 in (mig, mps) order */
  const int32_t* key_batch;   /* [K] */
  const int32_t* key_cost;    /* [K] slice cost */
  const double* key_lat;      /* [K] */
  const double* key_thr;      /* [K] */
  /* sub-space tuple lists (planner.py:406-432), 4 per task, index t*4 + 2*A + S */
  const int32_t* sub_off;     /* [4T+1] */
  const int32_t* sub_key;     /* local key indices, ascending */
  /* per sub-space variant groups + representative tuples (planner.py:518-526) */
  const int32_t* grp_off;     /* [4T+1] */
  const int32_t* grp_rep;     /* [2 * groups] tuple indices into the sub-space list, -1 = none */
  double a_max;               /* max_system_accuracy (model.py:296-299), computed on host */
} jsv_problem_desc;

/* Request fields shared by every probe of one call (planner.py:122-149). */
typedef struct {
  int32_t budget;             /* slice_budget */
  uint32_t space;             /* JSV_SPACE_* bits */
  double slack;
  const uint8_t* has_override;/* [E] or NULL */
  const double* override_val; /* [E] or NULL */
  int32_t pareto_width;
  int32_t exhaustive_limit;
  double eps;
  int32_t n_mix;
  double mix[JSV_MAX_MIX];
  int32_t feasible_only;
} jsv_request;

/* One probe = one plan() call: demand + the SLO/objective scalars of its AppSpec. */
typedef struct {
  double demand;
  double slo_eff;             /* AppSpec.effective_latency_slo_ms */
  double acc_slo;
  double alpha, beta;
  /* plan_uninformed statics (planner.py:997-1067), computed on the host in
   * Python float order; the demand-dependent parts run on the GPU */
  double uni_lat_budget[JSV_MAX_TASKS];
  double uni_floor[JSV_MAX_TASKS];
  double uni_weight[JSV_MAX_TASKS];
  double uni_best_hput[JSV_MAX_TASKS];
  int32_t uni_best_slices[JSV_MAX_TASKS];
  int32_t uni_min_cost[JSV_MAX_TASKS];
} jsv_probe;

/* Result of one probe (PlanResult + Configuration + verdicts, lowered). */
typedef struct {
  int32_t feasible;
  int32_t has_config;
  int32_t binding;            /* JSV_BIND_* */
  int32_t dead;               /* reference _Search.dead short-circuit */
  double objective;
  double a_obj;
  int64_t nodes;              /* B&B nodes visited (not a parity field) */
  int64_t leaves;             /* candidate allocations fully evaluated */
  int32_t pool_size[JSV_MAX_TASKS];
  int32_t pool_present[JSV_MAX_TASKS]; /* plan_uninformed stops early: absent tasks = 0 */
  int32_t truncated[JSV_MAX_TASKS];
  /* configuration, per task index */
  int32_t n_items[JSV_MAX_TASKS];
  uint32_t items[JSV_MAX_TASKS][JSV_MAX_ITEMS]; /* (local key << 16) | count */
  double hput[JSV_MAX_TASKS][JSV_MAX_ITEMS];
  double latency[JSV_MAX_TASKS];
  double capacity[JSV_MAX_TASKS];
  double demand[JSV_MAX_TASKS];
  double accuracy[JSV_MAX_TASKS];
  int32_t slices[JSV_MAX_TASKS];
  double fanout[JSV_MAX_EDGES];
  double path_acc[JSV_MAX_PATHS];
  int32_t total_slices;
  uint32_t uncovered_mask;
  /* verdict margins (validate_configuration order) */
  double lat_margin[JSV_MAX_PATHS];
  double thr_margin[JSV_MAX_TASKS];
  double res_margin;
  double acc_margin;
} jsv_plan_out;

typedef struct {
  double demand;              /* MaxDemandResult.demand_rps */
  int32_t probes;             /* sequential probe count of the reference bisection */
  int32_t status;             /* 0 ok, 1 zero (tiny probe infeasible), 2 diverged */
  int64_t gpu_probes;         /* probes actually evaluated (speculation included) */
} jsv_demand_out;

typedef struct {
  float ms_stage1, ms_stage2, ms_total; /* device time of the last call (CUDA events) */
  int64_t candidates_generated;         /* Stage-1 bundles generated */
  int64_t leaves;                       /* Stage-2 candidates evaluated */
  int64_t nodes;
  int32_t kernel_launches;
  int32_t dims;                         /* skyline row width D (padded) */
  int64_t pair_tests_a;                 /* sum over jobs of n^2 (Stage-1 skyline pairs) */
  int64_t pair_tests_b;                 /* sum over jobs of F^2 (frontier ranking pairs) */
  int64_t leaf_work;                    /* (prefix, bundle) items at the last level */
  int64_t exh_candidates;               /* mixed-radix candidates swept by the exhaustive kernel */
  int32_t exh_probes;                   /* probes solved by the exhaustive kernel */
  int32_t exh_pad_;
  int64_t swept;                        /* candidates the exhaustive register sweep compared
                                           one by one (live prefixes x sink pool); the rest of
                                           exh_candidates were decided by their prefix's
                                           throughput verdicts */
  int64_t live_prefixes;                /* prefixes the exhaustive sweep derived in full (the
                                           others failed a prefix task's throughput verdict) */
  int64_t s1_shadow_tests;              /* fused Stage 1: skyline pair tests on the float shadow */
  int64_t s1_exact_tests;               /* ... and exact double tests behind them */
} jsv_stats;

const char* jsv_last_error(void);
int jsv_version(void);
int jsv_device_count(void);

int jsv_context_create(int device, jsv_context** out);
void jsv_context_destroy(jsv_context* ctx);

int jsv_problem_create(jsv_context* ctx, const jsv_problem_desc* desc, jsv_problem** out);
void jsv_problem_destroy(jsv_problem* prob);

/* plan() over n independent probes (same request, per-probe demand/SLOs). */
int jsv_plan_batch(jsv_context* ctx, const jsv_problem* prob, const jsv_request* req,
                   int32_t n, const jsv_probe* probes, jsv_plan_out* out);

/* max_demand() for n points (probe.demand ignored); runs the doubling +
 * bisection of planner.py:1152-1173 with speculative batched probes and
 * replays it exactly.  The final plans (planner.py:1155, 1174) are written
 * to plans[n]. */
int jsv_max_demand_batch(jsv_context* ctx, const jsv_problem* prob, const jsv_request* req,
                         int32_t n, const jsv_probe* points, double rel_tol,
                         jsv_demand_out* out, jsv_plan_out* plans);

/* derive_configuration + validate_configuration of one explicit assignment:
 * n_items[t] items per task, items[t][k] = (local key << 16) | count, canonical order. */
int jsv_derive(jsv_context* ctx, const jsv_problem* prob, const jsv_request* req,
               const jsv_probe* probe, const int32_t* n_items, const uint32_t* items,
               jsv_plan_out* out);

/* brute_force_plan() (planner.py:1191-1272) over the request space's profile keys:
 * every instance-count map with counts 0..min(max_count, left / cost) and total
 * slices <= budget, each derived + validated on the GPU; argmax (objective,
 * -total_slices), ties on the smaller canonical m.  *assignments = number of maps
 * (SolverStats.nodes); more than max_assignments -> JSV_ERR_CONFIG "oracle refuses:
 * assignment cap exceeded".  *found = 0: no feasible map (out is then unused);
 * else out = derive + validate of the winner.  The task/variant/segment/batch caps
 * of OracleCaps are checked by the caller (planner.py:1205-1227). */
int jsv_brute_force(jsv_context* ctx, const jsv_problem* prob, const jsv_request* req,
                    const jsv_probe* probe, int32_t max_count, int64_t max_assignments,
                    int64_t* assignments, int32_t* found, jsv_plan_out* out);

/* validate_configuration on caller-supplied derived fields (per task index). */
int jsv_validate(jsv_context* ctx, const jsv_problem* prob, const jsv_request* req,
                 const jsv_probe* probe, const double* latency, const double* capacity,
                 const double* demand, int32_t total_slices, double a_obj,
                 uint32_t uncovered_mask, jsv_plan_out* out);

/* Stage-1 pool of one task for one probe, in frontier order (parity tests).
 * stats[k*(4+outdeg) + {0,1,2,3,4+j}] = slices, capacity, accuracy, latency, fanout_j;
 * items[k*JSV_MAX_ITEMS + i]. */
int jsv_pool_dump(jsv_context* ctx, const jsv_problem* prob, const jsv_request* req,
                  const jsv_probe* probe, int32_t task, int32_t cap, int32_t* n_out,
                  int32_t* n_items, uint32_t* items, double* stats, int32_t* truncated);

int jsv_last_stats(jsv_context* ctx, jsv_stats* out);

/* Page-locked host memory (cudaHostAlloc, portable).  An output array of
 * jsv_plan_batch in such memory receives the device-to-host copy directly (no
 * staging copy); any host memory works.  jsv_host_alloc returns NULL on failure
 * (jsv_last_error).  No reference counterpart: a transfer-path knob. */
void* jsv_host_alloc(size_t bytes);
void jsv_host_free(void* p);

/*
 * Stage-2 strategy of a context (no reference counterpart: the reference has
 * one CPU branch-and-bound, planner.py:731-912; every strategy returns its
 * exact result).
 *   JSV_STRATEGY_SEARCH      level-synchronous branch-and-bound (reference filters)
 *   JSV_STRATEGY_EXHAUSTIVE  mixed-radix sweep of the whole Stage-1 cross-product
 *                            (every candidate derived + validated) for probes whose
 *                            cross-product is <= max_candidates; search otherwise
 *   JSV_STRATEGY_AUTO        exhaustive when the cross-product is <= max_candidates
 *                            (default, limit 2^31 ~ 1 ms of sweep), search otherwise
 */
#define JSV_STRATEGY_SEARCH 0
#define JSV_STRATEGY_EXHAUSTIVE 1
#define JSV_STRATEGY_AUTO 2
int jsv_set_strategy(jsv_context* ctx, int strategy, int64_t max_candidates);

/*
 * Shard the exhaustive sweep of every probe across `world` GPUs: this context
 * evaluates prefix range [Q*rank/world, Q*(rank+1)/world) of each probe's
 * candidate space and returns its local argmax (jsv_plan_out of the local best,
 * or the replicated infeasibility diagnosis).  Ranks combine the outputs with
 * one all-gather (paper_2603_08797_b200/shard.py).  Search-strategy probes are
 * replicated on every rank.
 */
int jsv_set_shard(jsv_context* ctx, int rank, int world);

/* jsv_plan_batch with shard (rank, world) for this call only (the context's
 * own shard setting is untouched, so concurrent callers do not see it). */
int jsv_plan_batch_shard(jsv_context* ctx, const jsv_problem* prob, const jsv_request* req,
                         int32_t n, const jsv_probe* probes, int32_t rank, int32_t world,
                         jsv_plan_out* out);

/* Per-kernel CUDA-event timing on the library stream (bench roofline).
 * jsv_profile(on) resets the accumulators; on = 0 off, 1 every kernel, or
 * (1 << 30) | mask for only the kernels whose id bit is set.  jsv_kernel_times fills
 * ms[k] / count[k] for kernel ids 0..n-1 (see JSV_KERNEL_NAMES) and returns the id count. */
int jsv_profile(jsv_context* ctx, int on);
int jsv_kernel_times(jsv_context* ctx, int n, double* ms, int64_t* count);
#define JSV_KERNEL_NAMES \
  "generate", "stats", "pairs_a", "compact", "pairs_b", "truncate", "mrank", "s2_prep", \
  "s2_level", "s2_leaf", "s2_reduce", "finalize", "uninformed", "bucket", "s2_prefix", "s2_exh", \
  "s2_xreduce", "s2_xsort", \
  "fo_prep", "fo_enum", "fo_eval"

/*
 * Placement of MIG instances onto GPUs (reference placement.py).  A geometry
 * lists per MIG profile p its allowed (start, footprint width) pairs
 * [start_off[p], start_off[p+1]) and its first-fit-decreasing rank
 * order_rank[p] (the reference sorts instances by (-max width, -compute cost,
 * profile name, index); ranks are that order over profiles, computed by the
 * caller).  Instances are given as profile indices (MPS never affects packing).
 */
typedef struct jsv_geometry {
  int32_t n_profiles;
  int32_t slices_per_gpu;      /* <= 30 */
  const int32_t* start_off;    /* [n_profiles + 1] */
  const int32_t* start_pos;    /* allowed start offsets */
  const int32_t* start_width;  /* footprint width per start */
  const int32_t* order_rank;   /* [n_profiles] */
} jsv_geometry;

/* pack(instances, gpu_count, geometry, node_budget): per input instance i,
 * placed[i] = 1 with (gpu[i], start[i], width[i]), or 0 (unplaced).
 * gpu_count < 0 -> JSV_ERR_CONFIG (GeometryError "gpu_count must be non-negative"). */
int jsv_pack(const jsv_geometry* geometry, const int32_t* inst_profile, int32_t n,
             int32_t gpu_count, int64_t node_budget, int32_t* gpu, int32_t* start,
             int32_t* width, int32_t* placed);

/* min_gpus(instances, geometry, node_budget): *out = the smallest count that
 * fits every instance, or -1 - i when instance i fits no empty GPU
 * (GeometryError "instance ... does not fit an empty GPU"). */
int jsv_min_gpus(const jsv_geometry* geometry, const int32_t* inst_profile, int32_t n,
                 int64_t node_budget, int32_t* out);

#ifdef __cplusplus
}
#endif
#endif /* JSV_H */
