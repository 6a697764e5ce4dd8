// jsv_kernels.h -- kernel argument blocks and launchers shared by the host runtime.
#pragma once
#include <vector>
#include "jsv_internal.cuh"

// Per-kernel CUDA-event timing on the launching stream (bench.py roofline).
enum KernelId {
  K_GENERATE, K_STATS, K_PAIRS_A, K_COMPACT, K_PAIRS_B, K_TRUNCATE, K_MRANK, K_S2_PREP,
  K_S2_LEVEL, K_S2_LEAF, K_S2_REDUCE, K_FINALIZE, K_UNINFORMED, K_BUCKET, K_S2_PREFIX, K_S2_EXH, K_S2_XREDUCE, K_S2_XSORT, K_FO_PREP, K_FO_ENUM, K_FO_EVAL, K_X_LIVE, K_COUNT_
};

struct Prof {
  bool on = false;
  unsigned mask = ~0u;  // kernels (bit = K_ id) that get an event pair
  bool cur = false;     // the open begin_on was recorded
  cudaStream_t st = nullptr;
  std::vector<cudaEvent_t> ev;
  std::vector<int> ids;
  size_t used = 0;
  void begin(int id) { begin_on(id, st); }
  void end() { end_on(st); }
  // events on the kernel's own stream (kernels of a side stream overlap the main one:
  // their times are their own, not a share of a serial step)
  void begin_on(int id, cudaStream_t s) {
    cur = on && ((mask >> id) & 1u);
    if (!cur) return;
    if (used + 2 > ev.size()) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ev.push_back(e);
      }
    }
    ids.resize(ev.size() / 2 + 1);
    ids[used / 2] = id;
    cudaEventRecord(ev[used], s);
  }
  void end_on(cudaStream_t s) {
    if (!cur) return;
    cur = false;
    cudaEventRecord(ev[used + 1], s);
    used += 2;
  }
};

extern thread_local Prof* g_prof;

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel, size):
// the call costs microseconds of host time on every launch otherwise
#include <map>
#include <mutex>
// (one process-wide memo: the attribute belongs to the function, not to a host
// thread, so a per-thread memo let a new thread lower a limit another thread's
// memo still believed raised -- the next larger launch then failed)
inline void jsv_smem_attr(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = done[{dev, fn}];
  if (bytes > cur) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) ==
        cudaSuccess)
      cur = bytes;  // (only ever raised; a failed raise is reported by the launch)
  }
}
#define PROF_BEGIN(id) \
  do {                 \
    if (g_prof) g_prof->begin(id); \
  } while (0)
#define PROF_END()     \
  do {                 \
    if (g_prof) g_prof->end(); \
  } while (0)
#define PROF_BEGIN_ON(id, s) \
  do {                       \
    if (g_prof) g_prof->begin_on(id, s); \
  } while (0)
#define PROF_END_ON(s)       \
  do {                       \
    if (g_prof) g_prof->end_on(s); \
  } while (0)

struct S1Args {
  const DGraph* g;
  DTables tb;
  const DReq* rq;
  const DProbe* probes;
  int n_probes, T, maxi, D, W, maxout;
  long long C_probe;
  long long task_base[MAXT + 1];
  long long task_cap[MAXT];
  const GenDesc* desc;
  int n_desc, U;
  const unsigned* ways;
  uint32_t* items;
  int* nitems;
  double* arr;
  int* sl;
  unsigned* flag;
  int* cnt;
  int* front;
  int* fcnt;
  int* fpos;
  int* fcr;
  int* sorted;
  int* scr;
  int* pool_cand;
  int* pool_n;
  int* pool_trunc;
  int* p_sl;
  double* p_cap;
  double* p_acc;
  double* p_lat;
  double* p_fan;
  double* pool_min_lat2;
  int* pool_min_sl;
  double* pool_acc_ub;
  int* err;
  int S;          // slice budget
  int* order;     // [Ctot] per-job candidate order by slices
  int* bstart;    // [jobs * (S+2)] slice bucket starts
  int* surv;      // [Ctot] survivors of the same-bucket skyline pass, slices order
  int* pcnt;      // [Ctot] survivors before each sorted position
  int* sbst;      // [jobs * (S+2)] survivor bucket starts
  int* scnt;      // [jobs] survivors
  double* arrl;   // [D * Ctot] coordinates in list order (slices order, then survivor order)
  int* fsorted;   // [jobs] 1: k_front_sort computed the job's frontier ranks
  float4* arrf;   // [Ctot] float shadow of coordinates 1..4 in bucket order (D >= 5)
  int wl_mask;    // bit k: the launch consumes work list k (set by launch_stage1)
  int4* wl[3];    // pair-pass work lists {job, i0, j0}: same-bucket, survivors, frontier
  int* wn;        // [3] their lengths (zeroed per batch)
  int desc_t0[MAXT + 1];  // fused Stage 1: first descriptor of each task (descriptors by task)
  int fused_cap;  // fused Stage 1: candidates whose working lists fit shared memory
  unsigned long long* stamps;  // JSV_S1_PHASES: [jobs x 10] phase timestamps (else null)
  unsigned long long* tests;   // fused Stage 1: [2] skyline pair tests (float shadow, exact)
  int tma;        // fused Stage 1: stage the task's tables with cp.async.bulk (JSV_NO_TMA: loops)
  // fused Stage 1 split launch: block b of the launch runs job job_map[job_off + b]
  // (null: job = b).  Heavy jobs (largest demand) get a whole SM of 1024 threads,
  // the rest share SMs two by two at 512 threads, all in one wave.
  const int* job_map;
  int job_off;
};

struct S1Launch {
  const int* tile_task;   // device [tiles_pp]
  const int* tile_start;  // device [tiles_pp]
  int tiles_pp;
  int jchunks_a, jchunk_a;
  int jchunks_b, jchunk_b;
  long long max_items;  // capacity of each work list
  long long grid;       // blocks of the grid-stride pair kernels
};

int stage1_padded_dims(int D);
int launch_stage1(const S1Args& a, const S1Launch& L, cudaStream_t st);
int launch_stage1_expand(const S1Args& a, const int* rep, int n_s1, int n, cudaStream_t st);
size_t s1_fused_smem(int D, int NB, int cap);
int launch_stage1_fused(const S1Args& a, size_t smem, int n_heavy, cudaStream_t st, cudaStream_t st2,
                        cudaEvent_t fork, cudaEvent_t join);

// ------------------------------------------------------------------ stage 2

struct S2Args {
  const DGraph* g;
  const DReq* rq;
  const DProbe* probes;
  int n_probes, T, W, maxout;
  // pools (job = probe*T + task, entry = job*W + k)
  const int* pool_n;
  const int* p_sl;
  const double* p_cap;
  const double* p_acc;
  const double* p_lat;
  const double* p_fan;
  // candidate items, for the m tie-break (planner.py:852)
  const uint32_t* items;
  const int* nitems;
  const int* pool_cand;
  long long C_probe;
  long long task_base[MAXT + 1];
  int maxi;
  // m order of the pool bundles (k_m_rank; exhaustive full plans): [job * W + k] =
  // rank | ext << 16 | empty << 31 -- rank = #bundles of the pool with a smaller item
  // list, ext = rank + #bundles having this list as a proper prefix
  const uint32_t* mrank;
  // packed m keys (XArgs::mkey): [job * W + k] = key0 | key1 << 16 -- the rank of the
  // bundle's item list among every list and every list followed by a later task's
  // entry (key1: that continuation); mnone[job]: the same for "no instances"
  const uint32_t* mkey;
  const uint32_t* mnone;
  const double* min_lat2;  // [jobs] (0 for could_zero tasks, set by stage2 prep)
  const int* min_sl;
  const double* acc_ub;
  const int* future;       // [n_probes*(T+1)] future_slices by topo position
  BestRec* best;
  int* active;             // [n_probes] 1 = search this probe
  // level expansion
  int level, last, diag, want_config;
  long long n_slots;            // frontier slots of this level (all probes, with gaps)
  const long long* foff;        // [n_probes] first slot of each probe
  const long long* fcap;        // [n_probes] slot capacity of each probe
  const unsigned long long* fcnt;  // [n_probes] live prefixes of each probe (device)
  const uint16_t* cur;          // frontier choices [slot, T] (topo positions)
  int* cur_flag;                // [slot] bit0 = r > 0, bit1 = some child survived (diag)
  // per-slot prefix state (k_s2_prefix)
  long long* pr_width;           // 64-bit so the work scan cannot overflow (> 2^31 items)
  int* pr_flag;
  int* pr_probe;
  double* pr_r;
  int* pr_used;
  double* pr_lat;               // [slot * P] partial path latency before t
  double* pr_acc;               // [slot * P] partial path accuracy product
  unsigned long long* ptot;     // [n_probes] work items of each probe
  long long* pfx;               // [n_slots + 1] exclusive scan of pr_width
  const long long* pstart;      // [n_probes] first work item of each probe
  uint16_t* nxt;
  double* nxt_key;              // [slot of nxt] objective upper bound of the child (LEAF_FULL;
                                // orders a frontier best-first before it is split)
  unsigned long long* nxt_cnt;  // [n_probes]
  const long long* nxt_off;     // [n_probes]
  const long long* nxt_cap;     // [n_probes]
  int* err;
  // leaf level: blocks own (probe, chunk); per-block partial best, then a per-probe reduce
  int mode;                 // LEAF_FULL / LEAF_FIRST / LEAF_ANY
  const long long* boff;    // [n_probes+1] leaf-block offsets
  int ipt;                  // work items per thread in the leaf kernel
  struct LeafPart* part;    // [total leaf blocks]
  unsigned long long* inc;  // [n_probes] incumbent objective (order-preserving bits)
  int dbg;
};

#define LEAF_FULL 0
#define LEAF_FIRST 1
#define LEAF_ANY 2

struct LeafPart {
  int has;        // feasible candidate
  int sl;
  double obj;
  long long code; // (prefix << 16) | choice-at-last-level (0xFFFF = empty)
  int has_leaf;   // reached leaf (diagnostics)
  int pad_;
  long long leaf; // max reached leaf code
  unsigned long long leaves;
};

// exhaustive Stage 2 (jsv_exhaustive.cuh)
#define XBLOCK 256

struct XPart {
  int has, sl;
  double obj;
  long long idx;
  unsigned long long leaves;
  unsigned long long swept;  // candidates the register sweep compared (live prefixes x pool)
  unsigned long long mk;     // packed m key of the best (XArgs::mkey)
};

// per-probe decomposition (host-computed after Stage 1)
struct XProbe {
  int radix[MAXT];      // digit radix by topo position (pool_n + could_zero)
  int pn[MAXT];         // pool size by topo position ("no instances" digit value)
  long long q0, nq;     // prefix range of this shard
  long long loff;       // first slot of this probe's live list (prefix sum of nq)
  int glog;             // lanes per prefix group = 1 << glog
  int R;                // radix of the last position
  int rounds;           // 1: exhaustive probe (0: not swept)
  int rpl;              // register sweep: sink records per lane, ceil(pool / 32) (0: loop)
};

struct XArgs {
  S2Args s;
  const XProbe* xp;
  const long long* boff;  // [2 (n_probes + 1)]: part slots [boff[i], boff[n_probes + 1 + i]) of probe i
  const long long* roff;  // [n_probes + 1] first warp-round of each probe (concatenated rounds)
  const long long* cstart;  // [n_chunks + 1] first warp-round of each chunk
  long long n_chunks;
  unsigned long long* work; // chunk counter of the persistent blocks (zeroed per launch)
  XPart* part;            // [blocks]
  int mode;               // LEAF_FULL / LEAF_FIRST / LEAF_ANY
  int tma;                // stage the sink pool with cp.async.bulk (alignment holds)
  int fast;               // jsv_problem::lat_fast (non-negative bounded latencies)
  double lat2_max;        // 2 x the largest profile latency of the sink task
  // rank space (fast != 0), per probe [n_probes * W]: records and sorted columns
  uint4* xrank;           // {rank(capacity), rank(accuracy), rank(2 L), slices} per bundle
  uint2* xpack;           // the same as two SWAR words of 15-bit fields (rpl > 0)
  double* scap;           // sink-pool capacities sorted ascending
  double* sacc;           // sink-pool accuracies sorted ascending
  double* slat2;          // sink-pool 2 L sorted ascending
  int max_pn_last;        // largest sink pool of the batch
  int rpl;                // rank space: 1 = sink records kept in registers (XProbe::rpl per
                          // lane), 0 = loop over the shared-memory records
  int prune;              // prefixes failing a prefix task's throughput verdict are decided
                          // by k_x_live without the full derivation or a sweep
  const long long* uoff;  // [n_probes + 1] first upper prefix of each probe (k_x_live's
                          // work units: every prefix digit but the fastest)
  unsigned* live;         // live prefixes (local index - q0) of probe i at [xp[i].loff, ...)
  int* live_cnt;          // [n_probes] live prefixes per probe
  long long* roff_w;      // = roff, written by k_x_sched
  int mkey;               // full plans, T <= 5: m tie-breaks compare packed 55-bit keys
  int* xr_done;           // [n_probes] column blocks of k_x_rank finished
  int xr_zeroed;          // xr_done arrives zeroed (else launch_x_rank clears it)
  const long long* dev_totals;  // device-planned batches (k_x_plan): [0] upper prefixes
  int round;              // prefixes per round (<= x_slots(P))
};

// k_x_plan: XProbe construction on the device (no host round trip between Stage 1
// and the exhaustive Stage 2)
struct XPlanArgs {
  long long exh_limit;   // largest cross-product swept
  long long fo_budget;   // feasibility probes: candidates scanned from the front (0: all)
  long long live_cap;    // capacity of the live lists (entries)
  int shard_rank, shard_world;
  int reg;               // register sweep (XProbe::rpl)
  XProbe* xp;            // [n] out
  int* handled;          // [n] out: probe taken by the exhaustive sweep
  int* trunc;            // [n] out: feasibility scan truncated to fo_budget
  long long* uoff;       // [n + 1] out: first upper prefix of each probe
  long long* totals;     // [4] out: upper prefixes, live capacity used, candidates, probes
  int* err;              // capacity exceeded -> 4
};
int launch_x_plan(const XArgs& a, const XPlanArgs& pa, cudaStream_t st);
// rounds per chunk of the exhaustive kernel's persistent blocks
#define X_CHUNK 8
#ifndef JSV_XMINB
#define JSV_XMINB 2
#endif

// prefix-state slots per warp of the exhaustive kernel for a graph with P paths
__host__ __device__ constexpr int x_slots(int pm) { return pm <= 8 ? 32 : (pm <= 16 ? 8 : 2); }
// sink-pool records padded to a whole number of 4 x 32-lane sweeps
__host__ __device__ constexpr int x_pad(int n) { return ((n > 0 ? n : 1) + 127) & ~127; }
size_t x_smem_bytes(int max_pn_last, int P, bool rank);
long long x_resident_blocks(const XArgs& a, int P, size_t smem);
int launch_x_rank(const XArgs& a, cudaStream_t st);
int launch_stage2_exhaustive(const XArgs& a, long long grid, int P, size_t smem, cudaStream_t st,
                             cudaStream_t st2, cudaEvent_t fork, cudaEvent_t join,
                             long long n_upper, cudaStream_t st3 = nullptr,
                             cudaEvent_t join2 = nullptr);

// fan-out graphs (jsv_fanout.cuh)
#define FO_DELTA_W 1e-9   // slack on real-valued accuracy sums (>> float error)
#define FO_EPS_OBJ 1e-11  // |float objective - real objective| bound used for convergence

struct FoCls {
  double acc;  // accuracy of the class (bundle accuracy)
  int s;       // slices
  int pad_;
};

struct FoCand {
  int probe, b0;
  uint16_t cls[MAXT];  // class index per leaf position (0xFFFF: no instances)
};

struct FoArgs {
  S2Args s;
  int k;                   // leaves
  int entry;               // entry task index
  int leaf[MAXT];          // leaf task index per path (graph.paths order)
  int edge[MAXT];          // edge entry -> leaf
  int P0max;               // largest entry pool of the batch
  int SB;                  // slice budget (DP range 0..SB)
  const int* act;          // [n_probes] 1 = solve with this path
  FoCls* cls;              // [probe][b0][leafpos][W]
  int* ncls;               // [probe][b0][leafpos]
  double* F;               // [probe][b0][leafpos + 1][SB + 1]
  double* b0best;          // [probe][b0] best real objective (-inf: none)
  double* tau;             // [n_probes]
  FoCand* cand;            // candidate buffer
  unsigned long long* ncand;
  long long cand_cap;
  int* overflow;
  int shard_rank, shard_world;  // entry bundles b0 in [P0 r / W, P0 (r + 1) / W) only
};

int launch_fanout_prep(const FoArgs& a, cudaStream_t st);
int launch_fanout_tau(const FoArgs& a, double delta, cudaStream_t st);
int launch_fanout_round(const FoArgs& a, long long* n_cand_host, cudaStream_t st);

int launch_stage2_leaf(const S2Args& a, long long n_blocks, cudaStream_t st);
int launch_stage2_reduce(const S2Args& a, cudaStream_t st);

int launch_stage2_prep(const S2Args& a, double* min_lat2, int* min_sl, double* acc_ub, int* future,
                       cudaStream_t st);
int launch_stage2_prefix(const S2Args& a, cudaStream_t st);
int launch_stage2_level(const S2Args& a, long long total, cudaStream_t st);
int launch_stage2_blocked(const S2Args& a, cudaStream_t st);
// order each probe's frontier rows by the children's objective bound, descending
// (sort_tmp == nullptr: *sort_bytes <- the scratch size; returns a cudaError_t)
int launch_frontier_best_first(const double* key, uint16_t* rows, uint16_t* rows_tmp, double* k_tmp,
                               double* k_out, int* perm, int* perm_out, void* sort_tmp,
                               size_t* sort_bytes, const long long* foff, const long long* fcap,
                               const long long* seg_end, const unsigned long long* fcnt, int n,
                               long long n_slots, long long max_cap, int T, cudaStream_t st);

struct FinArgs {
  const DGraph* g;
  DTables tb;
  const DReq* rq;
  const DProbe* probes;
  int n_probes, T, W, maxi, maxout;
  long long C_probe;
  long long task_base[MAXT + 1];
  const int* pool_n;
  const int* pool_trunc;
  const int* pool_cand;
  const uint32_t* items;
  const int* nitems;
  const int* p_sl;
  const double* p_cap;
  const double* p_acc;
  const double* p_lat;
  const double* p_fan;
  const BestRec* best;
  const int* dead;         // [n_probes]
  const int* pick;         // [n_probes*T] plan_uninformed picks (-1 none), or null
  const int* uni_kills;    // [n_probes*T*5]
  int uninformed;
  jsv_plan_out* out;
};

int launch_finalize(const FinArgs& a, cudaStream_t st);
int launch_uninformed(const S2Args& a, const FinArgs& f, int* pick, int* kills, cudaStream_t st);

// explicit assignment (derive_configuration) and verdicts on given fields
struct DeriveArgs {
  const DGraph* g;
  DTables tb;
  const DReq* rq;
  const DProbe* probe;
  const int* n_items;      // [T]
  const uint32_t* items;   // [T*MAXI]
  jsv_plan_out* out;
};
int launch_derive(const DeriveArgs& a, cudaStream_t st);

struct ValidateArgs {
  const DGraph* g;
  const DReq* rq;
  const DProbe* probe;
  const double* lat;
  const double* cap;
  const double* dem;
  int total_sl;
  double a_obj;
  uint32_t uncovered;
  jsv_plan_out* out;
};
int launch_validate(const ValidateArgs& a, cudaStream_t st);

// brute_force_plan (jsv_brute.cu): ranked enumeration of instance-count maps
#define BF_MAXK 64
struct BruteBest {
  int has, sl;
  double obj;
  long long idx;
};
struct BruteArgs {
  const DGraph* g;
  DTables tb;
  const DReq* rq;
  const DProbe* probe;
  int K, S, maxc;
  const int* key_task;    // [K] task index, ascending
  const int* key_local;   // [K] local key index within the task
  const int* key_cost;    // [K] slice cost
  const long long* ways;  // [(K+1) x (S+1)] count suffixes of keys i.. within `left` slices
  long long total;        // ways[0][S] = maps to evaluate
  BruteBest* part;        // [blocks]
  int* found;
  long long* win;
  int* n_items;           // [T]   winner, for k_derive
  uint32_t* items;        // [T*MAXI]
};
int launch_brute(const BruteArgs& a, int blocks, cudaStream_t st);
