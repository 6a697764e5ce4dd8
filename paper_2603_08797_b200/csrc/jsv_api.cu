// jsv_api.cu -- host runtime of libjsv.so: context, lowered problems, batch
// orchestration of the Stage-1 / Stage-2 kernels, and the max_demand driver.
//
// Host-side scalar set-up (demand upper bounds, could_zero, exhaustive vs
// structured decision, plan_uninformed slice budgets) mirrors the reference's
// Python float order exactly; the file is compiled with -ffp-contract=off so
// no host expression is contracted into an FMA.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>
#include <algorithm>

#include <cub/device/device_scan.cuh>

#include "jsv_internal.cuh"
#include "jsv_kernels.h"

static thread_local std::string g_err;

#include <chrono>
// JSV_TIMING=1: host-side timestamps of the batch pipeline on stderr (diagnostics)
static double host_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}
static bool timing_on() {
  static const bool on = getenv("JSV_TIMING") != nullptr;
  return on;
}
// (timestamps are buffered and printed when the batch ends, so the printing
// does not stretch the gaps it measures)
struct TMark { double t; const char* label; };
static thread_local std::vector<TMark> g_tmarks;
static void jsv_t(const char* label) {
  g_tmarks.push_back({host_ms(), label});
  if (strcmp(label, "finalize done") == 0 || g_tmarks.size() > 4096) {
    for (const TMark& m : g_tmarks) fprintf(stderr, "[jsv t] %10.3f %s\n", m.t, m.label);
    g_tmarks.clear();
  }
}
#define JSV_T(label)                 \
  do {                               \
    if (timing_on()) jsv_t(label);   \
  } while (0)

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      return fail(JSV_ERR_CUDA, std::string(#x) + " (jsv_api.cu:" + std::to_string(__LINE__) + "): " + cudaGetErrorString(e_)); \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    size_t want = bytes + bytes / 4 + 256;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) n = want;
    return e;
  }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(p); }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

enum BufId {
  B_REQ, B_PROBES, B_DESC, B_WAYS, B_TILE_TASK, B_TILE_START, B_ITEMS, B_NITEMS, B_ARR, B_SL, B_FLAG,
  B_CNT, B_FRONT, B_FCNT, B_FPOS, B_FCR, B_SORTED, B_SCR, B_POOLC, B_POOLN, B_POOLT, B_PSL,
  B_PCAP, B_PACC, B_PLAT, B_PFAN, B_S1LAT2, B_S1SL, B_S1ACC, B_S2LAT2, B_S2SL,
  B_XLIVE, B_MRANK, B_XRDONE, B_STAMPS, B_S1TESTS, B_S2ACC, B_FUT, B_BEST, B_FR0, B_FR1, B_FLAGS, B_NXTCNT, B_NXTOFF, B_NXTCAP, B_WOFF, B_FOFF,
  B_WIDTH, B_PPROBE, B_DEAD, B_PICK, B_UKILL, B_OUT, B_ERR, B_DITEMS, B_DN, B_VAL, B_ACTIVE,
  B_BOFF, B_PART, B_INC, B_ORDER, B_BSTART, B_PFX, B_PFXOFF, B_SCAN, B_CNT2, B_FCAP,
  B_PWIDTH, B_PFLAG, B_PR, B_PUSED, B_PLATS, B_PACCS, B_PTOT, B_PSTART, B_XPROBE, B_XBOFF,
  B_XPART, B_XSACC, B_XRANK, B_XSCAP, B_XSLAT, B_XPACK, B_FOACT,
  B_FOCLS, B_FONCLS, B_FOF, B_FOB0, B_FOTAU, B_FOCAND, B_FONCAND, B_FOOVF, B_SURV, B_PCNT, B_SBST, B_SCNT, B_WL0, B_WL1, B_WL2, B_WN, B_ARRL, B_REP, B_FSORT, B_ARRF,
  B_BFKEY, B_BFWAYS, B_BFPART, B_BFOUT, B_SRT_KTMP, B_SRT_KOUT, B_SRT_PERM, B_SRT_PERMO,
  B_SRT_TMP, B_SRT_ROWS, B_SRT_SEGE, B_JOBMAP, B_COUNT
};

struct jsv_context {
  // one call at a time per context: entry points lock it (ctypes releases the GIL,
  // and every call reuses the context's device scratch, pinned staging and stats)
  std::recursive_mutex mu;
  int device = 0;
  cudaStream_t st = nullptr;
  cudaStream_t st2 = nullptr;               // side stream for independent kernels of a call
  cudaEvent_t fork = nullptr, join = nullptr;  // st -> st2 -> st ordering (no timing)
  cudaStream_t st3 = nullptr;                  // second side stream (exhaustive m keys)
  cudaEvent_t join2 = nullptr;
  cudaEvent_t ev[4] = {};
  DevBuf buf[B_COUNT];
  jsv_stats stats{};
  Prof prof;
  double kms[K_COUNT_] = {};
  long long kcnt[K_COUNT_] = {};
  int strategy = JSV_STRATEGY_AUTO;
  long long exh_limit = 1LL << 31;
  // branch-and-bound per-level frontier / live-count buffers (reused call to call:
  // cudaMalloc / cudaFree per call would serialise the device)
  std::vector<std::unique_ptr<DevBuf>> bb_fr, bb_cnt, bb_key;
  int shard_rank = 0, shard_world = 1;
  // the Stage-1 plan whose descriptor / ways / tile tables are on the device now (and
  // the buffers they were copied into): the next batch of the same plan skips them
  unsigned long long s1_up_id = 0;
  const void* s1_up_ptr[4] = {nullptr, nullptr, nullptr, nullptr};
  // pinned host staging for per-solve tables (one async copy instead of several
  // pageable ones); reused call to call -- every call synchronises before returning
  // (slot 1: the exhaustive probes' records, in flight together with slot 0's
  // chunk tables)
  void* hpin[3] = {nullptr, nullptr, nullptr};
  size_t hpin_cap[3] = {0, 0, 0};
  void* pinned(size_t bytes, int slot = 0) {
    if (bytes > hpin_cap[slot]) {
      if (hpin[slot]) cudaFreeHost(hpin[slot]);
      hpin[slot] = nullptr;
      hpin_cap[slot] = 0;
      if (cudaHostAlloc(&hpin[slot], bytes * 2, cudaHostAllocDefault) != cudaSuccess) return nullptr;
      hpin_cap[slot] = bytes * 2;
    }
    return hpin[slot];
  }
};

thread_local Prof* g_prof = nullptr;

// fold the per-kernel event pairs recorded since the last collection (stream is idle)
static void collect_prof(jsv_context& c) {
  Prof& P = c.prof;
  if (!P.on) return;
  for (size_t i = 0; i + 1 < P.used; i += 2) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, P.ev[i], P.ev[i + 1]) == cudaSuccess) {
      c.kms[P.ids[i / 2]] += ms;
      c.kcnt[P.ids[i / 2]] += 1;
    }
  }
  P.used = 0;
}

struct ProfScope {
  explicit ProfScope(jsv_context* c) {
    c->prof.st = c->st;
    g_prof = c->prof.on ? &c->prof : nullptr;
  }
  ~ProfScope() { g_prof = nullptr; }
};

extern "C" int jsv_profile(jsv_context* ctx, int on) {
  if (!ctx) return fail(JSV_ERR_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
  // on: 0 off, 1 every kernel, or (1 << 30) | mask -- only the kernels whose K_ id
  // bit is set (fewer event records inside a timed region)
  ctx->prof.on = on != 0;
  ctx->prof.mask = (on & (1 << 30)) ? (unsigned)(on & ((1 << 30) - 1)) : ~0u;
  ctx->prof.st = ctx->st;
  for (int k = 0; k < K_COUNT_; ++k) {
    ctx->kms[k] = 0.0;
    ctx->kcnt[k] = 0;
  }
  return JSV_OK;
}

extern "C" int jsv_kernel_times(jsv_context* ctx, int n, double* ms, int64_t* count) {
  if (!ctx || !ms || !count) return fail(JSV_ERR_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
  for (int k = 0; k < n && k < K_COUNT_; ++k) {
    ms[k] = ctx->kms[k];
    count[k] = ctx->kcnt[k];
  }
  return K_COUNT_;
}

struct S1Plan {
  unsigned long long id = 0;  // process-unique (the device copy of the tables is reused by id)
  std::vector<GenDesc> desc;
  std::vector<unsigned> ways;
  std::vector<long long> task_cap;
  std::vector<int> tile_task, tile_start;
  int U = 0, maxi = 2;
  long long C_probe = 0;
  long long max_cap = 0;
};

struct jsv_problem {
  jsv_context* ctx = nullptr;
  int T = 0, E = 0, P = 0, entry = 0, maxout = 0;
  std::vector<int> topo, decl, succ_off, edge_dst, edge_src, pred_off, pred_edge, path_off,
      path_task;
  std::vector<double> path_frac;
  std::vector<int> var_off, var_fac_off, most_acc;
  std::vector<double> var_acc, var_fac;
  std::vector<int> key_off, key_var, key_cost;
  std::vector<double> key_lat, key_thr;
  std::vector<int> sub_off, sub_key, grp_off, grp_rep;
  double a_max = 0.0;
  // every profile latency is +0 or positive and finite, and no path sum can
  // overflow: the exhaustive kernel's Neumaier step may then use max/min for the
  // |f| >= |x| ordering and skip the non-finite-compensation test (exact)
  // (capacities finite too: fl(a - b) >= 0 <=> a >= b for the verdicts)
  bool lat_fast = false;
  DGraph hg{};
  DevBuf dgraph, d_var_acc, d_var_fac_off, d_var_fac, d_key_var, d_key_cost, d_key_lat, d_key_thr,
      d_sub_off, d_sub_key, d_grp_off, d_grp_rep;
  DTables dt{};
  std::map<std::tuple<int, unsigned, int, int>, std::shared_ptr<S1Plan>> s1cache;
};

template <class T>
static cudaError_t upload(DevBuf& b, const std::vector<T>& v) {
  size_t bytes = sizeof(T) * (v.empty() ? 1 : v.size());
  cudaError_t e = b.ensure(bytes);
  if (e != cudaSuccess) return e;
  if (!v.empty()) e = cudaMemcpy(b.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice);
  return e;
}

extern "C" const char* jsv_last_error(void) { return g_err.c_str(); }

// error reporting for the other translation units (jsv_place.cu)
int jsv_fail_msg(int code, const std::string& msg) { return fail(code, msg); }
extern "C" int jsv_version(void) { return 1; }
extern "C" int jsv_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

extern "C" int jsv_context_create(int device, jsv_context** out) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    return fail(JSV_ERR_NODEV, "no CUDA device visible: the sm_100a planner has no CPU fallback");
  if (device < 0 || device >= n) return fail(JSV_ERR_ARG, "device index out of range");
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(JSV_ERR_NODEV, std::string("libjsv is built for sm_100a, device is ") + prop.name);
  // the leaf evaluator keeps per-task arrays on the thread stack; make room explicitly
  CK(cudaDeviceSetLimit(cudaLimitStackSize, 8192));
  auto* c = new jsv_context();
  c->device = device;
  CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
  {
    // (the m keys are the longest side chain into the exhaustive sweep: their stream
    // gets the highest priority, so its blocks are dispatched ahead of the live pass)
    int least = 0, greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CK(cudaStreamCreateWithPriority(&c->st3, cudaStreamNonBlocking,
                                    getenv("JSV_NO_PRIO") ? least : greatest));
  }
  CK(cudaEventCreateWithFlags(&c->join2, cudaEventDisableTiming));
  for (auto& e : c->ev) CK(cudaEventCreate(&e));
  *out = c;
  return JSV_OK;
}

extern "C" void jsv_context_destroy(jsv_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->fork) cudaEventDestroy(ctx->fork);
  if (ctx->join) cudaEventDestroy(ctx->join);
  if (ctx->st2) cudaStreamDestroy(ctx->st2);
  if (ctx->join2) cudaEventDestroy(ctx->join2);
  if (ctx->st3) cudaStreamDestroy(ctx->st3);
  if (ctx->st) cudaStreamDestroy(ctx->st);
  for (void* h : ctx->hpin)
    if (h) cudaFreeHost(h);
  delete ctx;
}

// ---------------------------------------------------------------- problems

extern "C" int jsv_problem_create(jsv_context* ctx, const jsv_problem_desc* d, jsv_problem** out) {
  if (!ctx || !d || !out) return fail(JSV_ERR_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
  const int T = d->n_tasks, E = d->n_edges, P = d->n_paths;
  if (T < 1 || T > MAXT) return fail(JSV_ERR_ARG, "task count outside [1, 16]");
  if (E < 0 || E > MAXE) return fail(JSV_ERR_ARG, "edge count outside [0, 32]");
  if (P < 1 || P > MAXP) return fail(JSV_ERR_ARG, "path count outside [1, 64]");
  CK(cudaSetDevice(ctx->device));
  auto pr = std::make_unique<jsv_problem>();
  jsv_problem& p = *pr;
  p.ctx = ctx;
  p.T = T; p.E = E; p.P = P; p.entry = d->entry;
  p.topo.assign(d->topo, d->topo + T);
  p.decl.assign(d->decl, d->decl + T);
  p.succ_off.assign(d->succ_off, d->succ_off + T + 1);
  p.edge_dst.assign(d->edge_dst, d->edge_dst + E);
  p.pred_off.assign(d->pred_off, d->pred_off + T + 1);
  p.pred_edge.assign(d->pred_edge, d->pred_edge + E);
  p.path_off.assign(d->path_off, d->path_off + P + 1);
  p.path_task.assign(d->path_task, d->path_task + p.path_off[P]);
  p.path_frac.assign(d->path_frac, d->path_frac + P);
  p.var_off.assign(d->var_off, d->var_off + T + 1);
  const int V = p.var_off[T];
  p.var_acc.assign(d->var_acc, d->var_acc + V);
  p.var_fac_off.assign(d->var_fac_off, d->var_fac_off + V);
  int nfac = 0;
  for (int t = 0; t < T; ++t)
    nfac += (p.var_off[t + 1] - p.var_off[t]) * (p.succ_off[t + 1] - p.succ_off[t]);
  p.var_fac.assign(d->var_fac, d->var_fac + nfac);
  p.most_acc.assign(d->most_acc, d->most_acc + T);
  p.key_off.assign(d->key_off, d->key_off + T + 1);
  const int K = p.key_off[T];
  p.key_var.assign(d->key_var, d->key_var + K);
  p.key_cost.assign(d->key_cost, d->key_cost + K);
  p.key_lat.assign(d->key_lat, d->key_lat + K);
  p.key_thr.assign(d->key_thr, d->key_thr + K);
  {
    double mx = 0.0;
    bool ok = true;
    for (double v : p.key_lat) {
      if (!(v >= 0.0) || std::signbit(v) || !std::isfinite(v)) ok = false;
      else mx = std::max(mx, v);
    }
    for (double v : p.key_thr) ok = ok && std::isfinite(v) && v < 1e290;
    // accuracy threshold monotonicity: accuracies and path fractions >= +0
    for (double v : p.var_acc) ok = ok && v >= 0.0 && !std::signbit(v) && std::isfinite(v);
    for (double v : p.path_frac) ok = ok && v >= 0.0 && !std::signbit(v) && std::isfinite(v);
    p.lat_fast = ok && mx * 2.0 * (double)(T + 1) < 1e300;
  }
  p.sub_off.assign(d->sub_off, d->sub_off + 4 * T + 1);
  p.sub_key.assign(d->sub_key, d->sub_key + p.sub_off[4 * T]);
  p.grp_off.assign(d->grp_off, d->grp_off + 4 * T + 1);
  p.grp_rep.assign(d->grp_rep, d->grp_rep + 2 * p.grp_off[4 * T]);
  p.a_max = d->a_max;
  for (int t = 0; t < T; ++t) {
    if (p.key_off[t + 1] - p.key_off[t] > 65535) return fail(JSV_ERR_ARG, "too many profile keys");
  }
  p.edge_src.assign(E, 0);
  for (int t = 0; t < T; ++t)
    for (int e = p.succ_off[t]; e < p.succ_off[t + 1]; ++e) p.edge_src[e] = t;
  p.maxout = 1;
  for (int t = 0; t < T; ++t) p.maxout = std::max(p.maxout, p.succ_off[t + 1] - p.succ_off[t]);
  if (p.path_off[P] > MAXP * MAXT) return fail(JSV_ERR_ARG, "paths too long");
  DGraph& g = p.hg;
  memset(&g, 0, sizeof(g));
  g.T = T; g.E = E; g.P = P; g.entry = p.entry; g.maxout = p.maxout; g.sum_path = p.path_off[P];
  for (int i = 0; i < T; ++i) {
    g.topo[i] = p.topo[i];
    g.pos_of[p.topo[i]] = i;
    g.decl[i] = p.decl[i];
    g.most_acc[i] = p.most_acc[i];
  }
  for (int i = 0; i <= T; ++i) {
    g.succ_off[i] = p.succ_off[i];
    g.pred_off[i] = p.pred_off[i];
    g.var_off[i] = p.var_off[i];
    g.key_off[i] = p.key_off[i];
  }
  for (int e = 0; e < E; ++e) {
    g.edge_dst[e] = p.edge_dst[e];
    g.edge_src[e] = p.edge_src[e];
    g.pred_edge[e] = p.pred_edge[e];
  }
  for (int i = 0; i <= P; ++i) g.path_off[i] = p.path_off[i];
  for (int i = 0; i < p.path_off[P]; ++i) g.path_task[i] = p.path_task[i];
  for (int q = 0; q < P; ++q) {
    g.path_frac[q] = p.path_frac[q];
    uint32_t m = 0;
    for (int k = p.path_off[q]; k < p.path_off[q + 1]; ++k) m |= 1u << p.path_task[k];
    g.path_mask[q] = m;
  }
  g.a_max = p.a_max;
  CK(p.dgraph.ensure(sizeof(DGraph)));
  CK(cudaMemcpy(p.dgraph.p, &g, sizeof(DGraph), cudaMemcpyHostToDevice));
  CK(upload(p.d_var_acc, p.var_acc));
  CK(upload(p.d_var_fac_off, p.var_fac_off));
  CK(upload(p.d_var_fac, p.var_fac));
  CK(upload(p.d_key_var, p.key_var));
  CK(upload(p.d_key_cost, p.key_cost));
  CK(upload(p.d_key_lat, p.key_lat));
  CK(upload(p.d_key_thr, p.key_thr));
  CK(upload(p.d_sub_off, p.sub_off));
  CK(upload(p.d_sub_key, p.sub_key));
  CK(upload(p.d_grp_off, p.grp_off));
  CK(upload(p.d_grp_rep, p.grp_rep));
  p.dt.var_acc = p.d_var_acc.as<double>();
  p.dt.var_fac_off = p.d_var_fac_off.as<int>();
  p.dt.var_fac = p.d_var_fac.as<double>();
  p.dt.key_var = p.d_key_var.as<int>();
  p.dt.key_cost = p.d_key_cost.as<int>();
  p.dt.key_lat = p.d_key_lat.as<double>();
  p.dt.key_thr = p.d_key_thr.as<double>();
  p.dt.sub_off = p.d_sub_off.as<int>();
  p.dt.sub_key = p.d_sub_key.as<int>();
  p.dt.grp_off = p.d_grp_off.as<int>();
  p.dt.grp_rep = p.d_grp_rep.as<int>();
  *out = pr.release();
  return JSV_OK;
}

extern "C" void jsv_problem_destroy(jsv_problem* prob) { delete prob; }

// ------------------------------------------------------ host scalar set-up

// propagate_demand (model.py:239-264) with per-edge factors
static void host_rates(const jsv_problem& p, double demand, const double* fac, double* out) {
  for (int i = 0; i < p.T; ++i) {
    const int t = p.topo[i];
    if (t == p.entry) {
      out[t] = demand;
      continue;
    }
    double s = 0.0;
    for (int k = p.pred_off[t]; k < p.pred_off[t + 1]; ++k) {
      const int e = p.pred_edge[k];
      s += out[p.edge_src[e]] * fac[e];
    }
    out[t] = s;
  }
}

// _max_factors / _min_factors (planner.py:638-671)
static void host_factors(const jsv_problem& p, const jsv_request& rq, bool a, bool want_max,
                         double* fac) {
  for (int t = 0; t < p.T; ++t) {
    for (int e = p.succ_off[t]; e < p.succ_off[t + 1]; ++e) {
      const int j = e - p.succ_off[t];
      if (rq.has_override && rq.has_override[e]) {
        fac[e] = rq.override_val[e];
        continue;
      }
      const int v0 = p.var_off[t], v1 = p.var_off[t + 1];
      double best = 0.0;
      bool first = true;
      for (int v = v0; v < v1; ++v) {
        if (!a && v - v0 != p.most_acc[t]) continue;
        const double f = p.var_fac[p.var_fac_off[v] + j];
        if (first || (want_max ? f > best : f < best)) best = f;
        first = false;
      }
      fac[e] = best;
    }
  }
}

// CPython 3.12 sum() of floats
static double host_pysum(const double* x, int n) {
  if (n == 0) return 0.0;
  double f = 0.0 + x[0], c = 0.0;
  for (int i = 1; i < n; ++i) {
    double t = f + x[i];
    if (std::fabs(f) >= std::fabs(x[i])) c += (f - t) + x[i];
    else c += (x[i] - t) + f;
    f = t;
  }
  if (c != 0.0 && std::isfinite(c)) f += c;
  return f;
}

// order-preserving keys of doubles (NaN excluded)
static inline unsigned long long h_key(double x) {
  unsigned long long b;
  memcpy(&b, &x, 8);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
static inline double h_unkey(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  double x;
  memcpy(&x, &b, 8);
  return x;
}
static inline bool h_acc_pass(double w, double a_max, double s) {
  const double a = w / a_max;  // a_obj (model.py:293)
  return a - s >= 0;           // accuracy verdict (planner.py:350-351)
}

// Smallest double W with h_acc_pass(W); ok = 0 when no exact threshold exists.
static void acc_threshold(double a_max, double s, double& thr, int& ok) {
  ok = 0;
  thr = 0.0;
  if (!(a_max > 0) || !std::isfinite(a_max) || !std::isfinite(s)) return;
  const double ninf = -INFINITY, pinf = INFINITY;
  if (h_acc_pass(ninf, a_max, s)) {
    thr = ninf;
    ok = 1;
    return;
  }
  if (!h_acc_pass(pinf, a_max, s)) return;
  unsigned long long lo = h_key(ninf), hi = h_key(pinf);  // lo fails, hi passes
  while (hi - lo > 1) {
    const unsigned long long mid = lo + (hi - lo) / 2;
    if (h_acc_pass(h_unkey(mid), a_max, s)) hi = mid;
    else lo = mid;
  }
  thr = h_unkey(hi);
  ok = 1;
}

// The factor products of a request (independent of demand): computed once per batch
struct ProbeFactors {
  double up[2][MAXE];  // _demand_upper_bound, A' off / on
  double cz[MAXE];     // could_zero (the request's own A)
  double uni[MAXE];    // plan_uninformed (A off, upper)
};

static void probe_factors(const jsv_problem& p, const jsv_request& rq, ProbeFactors& f) {
  host_factors(p, rq, false, true, f.up[0]);
  host_factors(p, rq, true, true, f.up[1]);
  host_factors(p, rq, (rq.space & JSV_SPACE_A) != 0, false, f.cz);
  host_factors(p, rq, false, true, f.uni);
}

static void fill_probe(const jsv_problem& p, const jsv_request& rq, const jsv_probe& in,
                       DProbe& o, const ProbeFactors* pf = nullptr, bool zeroed = false) {
  ProbeFactors own;
  if (!pf) {
    probe_factors(p, rq, own);
    pf = &own;
  }
  if (!zeroed) memset(&o, 0, sizeof(o));
  o.demand = in.demand;
  o.slo_eff = in.slo_eff;
  o.acc_slo = in.acc_slo;
  o.alpha = in.alpha;
  o.beta = in.beta;
  {
    // one bisection per distinct (a_max, acc_slo): probes of a sweep share them
    static thread_local double c_amax = NAN, c_slo = NAN, c_thr = 0.0;
    static thread_local int c_ok = 0;
    if (!(p.a_max == c_amax && in.acc_slo == c_slo)) {
      acc_threshold(p.a_max, in.acc_slo, c_thr, c_ok);
      c_amax = p.a_max;
      c_slo = in.acc_slo;
    }
    o.acc_thr = c_thr;
    o.acc_thr_ok = c_ok;
  }
  double r[MAXT];
  for (int a = 0; a < 2; ++a) {
    host_rates(p, in.demand, pf->up[a], r);
    for (int t = 0; t < p.T; ++t) o.r_upper[a][t] = r[t];
  }
  host_rates(p, in.demand, pf->cz, r);
  o.could_zero = 0;
  for (int t = 0; t < p.T; ++t)
    if (r[t] == 0.0) o.could_zero |= 1u << t;
  for (int t = 0; t < p.T; ++t) {
    o.lat_budget[t] = in.uni_lat_budget[t];
    o.floor_[t] = in.uni_floor[t];
    o.weight[t] = in.uni_weight[t];
    o.best_hput[t] = in.uni_best_hput[t];
    o.best_slices[t] = in.uni_best_slices[t];
    o.min_cost[t] = in.uni_min_cost[t];
  }
  if (!(rq.space & JSV_SPACE_T)) {
    // plan_uninformed demand-dependent budgets (planner.py:1014-1037)
    host_rates(p, in.demand, pf->uni, r);
    double est[MAXT], est_decl[MAXT];
    for (int t = 0; t < p.T; ++t) {
      o.star[t] = r[t];
      est[t] = r[t] / o.best_hput[t] * (double)o.best_slices[t];
    }
    for (int i = 0; i < p.T; ++i) est_decl[i] = est[p.decl[i]];
    const double tot = host_pysum(est_decl, p.T);
    for (int t = 0; t < p.T; ++t) {
      double sb = tot > 0 ? (double)rq.budget * est[t] / tot : (double)rq.budget / (double)p.T;
      if ((double)o.min_cost[t] > sb) sb = (double)o.min_cost[t];
      o.slice_budget[t] = sb;
    }
  }
}

static void fill_req(const jsv_problem& p, const jsv_request& rq, DReq& o) {
  memset(&o, 0, sizeof(o));
  o.S = rq.budget;
  o.space = rq.space;
  o.slack = rq.slack;
  o.eps = rq.eps;
  o.W = rq.pareto_width;
  o.n_mix = rq.n_mix;
  for (int i = 0; i < rq.n_mix && i < JSV_MAX_MIX; ++i) o.mix[i] = rq.mix[i];
  o.feasible_only = rq.feasible_only;
  for (int e = 0; e < p.E; ++e) {
    o.has_ov[e] = rq.has_override ? rq.has_override[e] : 0;
    o.ov[e] = (rq.has_override && rq.has_override[e]) ? rq.override_val[e] : 0.0;
  }
}

// _enumeration_size (planner.py:435-457): count vectors within budget, early exit
static long long enumeration_size(const std::vector<int>& costs, int S, int limit) {
  std::vector<long long> ways(S + 1, 0), nw(S + 1);
  ways[0] = 1;
  for (int cost : costs) {
    std::fill(nw.begin(), nw.end(), 0);
    for (int used = 0; used <= S; ++used) {
      if (!ways[used]) continue;
      for (int spent = used; spent <= S; spent += cost) nw[spent] += ways[used];
    }
    ways.swap(nw);
    long long s = 0;
    for (long long w : ways) s += w;
    if (s > limit) return (long long)limit + 1;
  }
  long long s = 0;
  for (long long w : ways) s += w;
  return s;
}

static int build_s1plan(const jsv_problem& p, const jsv_request& rq, S1Plan& pl) {
  const int S = rq.budget;
  const bool A = rq.space & JSV_SPACE_A, Sp = rq.space & JSV_SPACE_S;
  pl.task_cap.assign(p.T, 0);
  pl.maxi = 2;
  int unit = 0;
  for (int t = 0; t < p.T; ++t) {
    for (int a = 0; a <= (A ? 1 : 0); ++a) {
      for (int s = 0; s <= (Sp ? 1 : 0); ++s) {
        const int sub = t * 4 + 2 * a + s;
        const int n = p.sub_off[sub + 1] - p.sub_off[sub];
        if (n == 0) continue;
        GenDesc d{};
        d.task = t; d.sub = sub; d.a = a;
        d.n_tuples = n; d.key_base = p.sub_off[sub];
        d.grp_base = p.grp_off[sub];
        d.n_groups = p.grp_off[sub + 1] - p.grp_off[sub];
        d.unit_off = unit;
        std::vector<int> costs(n);
        for (int i = 0; i < n; ++i)
          costs[i] = p.key_cost[p.key_off[t] + p.sub_key[p.sub_off[sub] + i]];
        const long long size = enumeration_size(costs, S, rq.exhaustive_limit);
        if (size <= rq.exhaustive_limit) {
          d.mode = 0;
          d.w_off = (int)pl.ways.size();
          // suffix ways W[i][l] and max item count
          std::vector<unsigned> W((size_t)(n + 1) * (S + 1), 0);
          std::vector<int> mx((size_t)(n + 1) * (S + 1), 0);
          for (int l = 0; l <= S; ++l) W[(size_t)n * (S + 1) + l] = 1;
          for (int i = n - 1; i >= 0; --i)
            for (int l = 0; l <= S; ++l) {
              unsigned long long acc = 0;
              int best = 0;
              for (int c = 0; c * costs[i] <= l; ++c) {
                acc += W[(size_t)(i + 1) * (S + 1) + l - c * costs[i]];
                best = std::max(best, (c > 0) + mx[(size_t)(i + 1) * (S + 1) + l - c * costs[i]]);
              }
              W[(size_t)i * (S + 1) + l] = (unsigned)std::min<unsigned long long>(acc, 0xFFFFFFFFull);
              mx[(size_t)i * (S + 1) + l] = best;
            }
          if (W[S] != (unsigned)size) return fail(JSV_ERR_CONFIG, "enumeration size mismatch");
          const int items = mx[S];
          if (items > MAXI) return fail(JSV_ERR_CONFIG, "exhaustive bundles exceed 16 items");
          pl.maxi = std::max(pl.maxi, items);
          pl.ways.insert(pl.ways.end(), W.begin(), W.end());
          d.n_units = (int)size - 1;
          d.n_tuple_units = 0;
          d.n_mix_units = 0;
          pl.task_cap[t] += size - 1;
        } else {
          d.mode = 1;
          d.n_tuple_units = n;
          const int G = d.n_groups;
          d.n_mix_units = (G * (G - 1) / 2) * rq.n_mix * N_LEVELS * 4;
          d.n_units = d.n_tuple_units + d.n_mix_units;
          pl.task_cap[t] += (long long)n * (N_LEVELS + 1) + d.n_mix_units;
        }
        unit += d.n_units;
        pl.desc.push_back(d);
      }
    }
  }
  pl.U = unit;
  pl.C_probe = 0;
  pl.max_cap = 0;
  pl.tile_task.clear();
  pl.tile_start.clear();
  for (int t = 0; t < p.T; ++t) {
    pl.C_probe += pl.task_cap[t];
    pl.max_cap = std::max(pl.max_cap, pl.task_cap[t]);
    for (long long s0 = 0; s0 < pl.task_cap[t]; s0 += 256) {
      pl.tile_task.push_back(t);
      pl.tile_start.push_back((int)s0);
    }
  }
  if (pl.ways.empty()) pl.ways.push_back(0);
  return JSV_OK;
}

static int get_s1plan(jsv_problem& p, const jsv_request& rq, std::shared_ptr<S1Plan>& out) {
  auto key = std::make_tuple(rq.budget, rq.space & 3u, rq.exhaustive_limit, rq.n_mix);
  auto it = p.s1cache.find(key);
  if (it != p.s1cache.end()) {
    out = it->second;
    return JSV_OK;
  }
  auto pl = std::make_shared<S1Plan>();
  static std::atomic<unsigned long long> next_id{1};
  pl->id = next_id++;
  int rc = build_s1plan(p, rq, *pl);
  if (rc) return rc;
  p.s1cache[key] = pl;
  out = pl;
  return JSV_OK;
}

// ------------------------------------------------------------- batch solve

struct BatchState {
  int n = 0;
  int feasible_only = 0;
  std::shared_ptr<S1Plan> pl;
  S1Args s1{};
  std::vector<int> pool_n;
  std::vector<int> dead;
  std::vector<DProbe> probes;
  bool s1_pending = false;  // Stage-1 readbacks in flight (stage1_collect)
};

static int run_stage1(jsv_problem& p, const jsv_request& rq, int n, const DProbe* probes,
                      BatchState& bs, int n_s1, const std::vector<int>& rep) {
  jsv_context& c = *p.ctx;
  cudaStream_t st = c.st;
  int rc = get_s1plan(p, rq, bs.pl);
  if (rc) return rc;
  const S1Plan& pl = *bs.pl;
  const int T = p.T;
  const int W = rq.pareto_width;
  const int D = stage1_padded_dims(4 + p.maxout);
  const long long Ctot = (long long)n * pl.C_probe;
  const long long jobs = (long long)n * T;
  DReq hreq;
  fill_req(p, rq, hreq);
  auto& B = c.buf;
  CK(B[B_REQ].ensure(sizeof(DReq)));
  CK(B[B_PROBES].ensure(sizeof(DProbe) * n));
  CK(B[B_DESC].ensure(sizeof(GenDesc) * std::max<size_t>(1, pl.desc.size())));
  CK(B[B_WAYS].ensure(sizeof(unsigned) * std::max<size_t>(1, pl.ways.size())));
  CK(B[B_TILE_TASK].ensure(sizeof(int) * std::max<size_t>(1, pl.tile_task.size())));
  CK(B[B_TILE_START].ensure(sizeof(int) * std::max<size_t>(1, pl.tile_start.size())));
  // fused Stage 1 with more jobs than SMs but fewer than two per SM: every job on a
  // whole SM (1024 threads), the largest demands (the most candidates) first, so the
  // second wave holds the smallest jobs (measured: 192 XR jobs 346 -> ~200 us against
  // 512 threads two per SM; JSV_S1_SPLIT: the largest on 1024 threads and the rest
  // two per SM at 512, one wave -- 265 us)
  int n_sm = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  const long long jobs1 = (long long)n_s1 * T;
  std::vector<int> jmap;
  int n_heavy = 0;
  // (up to three jobs per SM: 384 XR jobs 0.525 -> 0.478 ms; at 768 the 512-thread
  // pairs are 2% faster)
  long long lpt_max = 3;  // (JSV_S1_LPT_MAX: the largest jobs-per-SM multiple scheduled LPT)
  if (const char* e = getenv("JSV_S1_LPT_MAX")) lpt_max = atoll(e);
  if (jobs1 > n_sm && jobs1 < lpt_max * n_sm && !getenv("JSV_NO_S1SPLIT")) {
    n_heavy = getenv("JSV_S1_SPLIT") ? (int)(2LL * n_sm - jobs1) : (int)jobs1;
    jmap.resize((size_t)jobs1);
    for (int j = 0; j < (int)jobs1; ++j) jmap[j] = j;
    std::stable_sort(jmap.begin(), jmap.end(),
                     [&](int x, int y) { return probes[x / T].demand > probes[y / T].demand; });
  }
  CK(B[B_JOBMAP].ensure(sizeof(int) * std::max<size_t>(1, jmap.size())));
  {
    // the batch's inputs staged in pinned memory: truly asynchronous copies
    // (pageable sources would each be a staged, host-blocking transfer)
    struct Up { void* dst; const void* src; size_t bytes; };
    // (the plan's tables only when another plan, or a reallocation, replaced them)
    const bool plan_resident = c.s1_up_id == pl.id && c.s1_up_ptr[0] == B[B_DESC].p &&
                               c.s1_up_ptr[1] == B[B_WAYS].p && c.s1_up_ptr[2] == B[B_TILE_TASK].p &&
                               c.s1_up_ptr[3] == B[B_TILE_START].p && !getenv("JSV_NO_S1CACHE");
    const size_t ps = plan_resident ? 0 : 1;
    const Up ups[] = {{B[B_REQ].p, &hreq, sizeof(DReq)},
                      {B[B_PROBES].p, probes, sizeof(DProbe) * n},
                      {B[B_DESC].p, pl.desc.data(), ps * sizeof(GenDesc) * pl.desc.size()},
                      {B[B_WAYS].p, pl.ways.data(), ps * sizeof(unsigned) * pl.ways.size()},
                      {B[B_TILE_TASK].p, pl.tile_task.data(), ps * sizeof(int) * pl.tile_task.size()},
                      {B[B_TILE_START].p, pl.tile_start.data(), ps * sizeof(int) * pl.tile_start.size()},
                      {B[B_JOBMAP].p, jmap.data(), sizeof(int) * jmap.size()}};
    c.s1_up_id = pl.id;
    c.s1_up_ptr[0] = B[B_DESC].p;
    c.s1_up_ptr[1] = B[B_WAYS].p;
    c.s1_up_ptr[2] = B[B_TILE_TASK].p;
    c.s1_up_ptr[3] = B[B_TILE_START].p;
    size_t total = 0;
    for (const Up& u : ups) total += (u.bytes + 15) & ~size_t(15);
    char* h = static_cast<char*>(c.pinned(total));
    if (!h) return fail(JSV_ERR_CUDA, "cudaHostAlloc failed");
    size_t off = 0;
    for (const Up& u : ups) {
      if (u.bytes == 0) continue;
      memcpy(h + off, u.src, u.bytes);
      CK(cudaMemcpyAsync(u.dst, h + off, u.bytes, cudaMemcpyHostToDevice, st));
      off += (u.bytes + 15) & ~size_t(15);
    }
  }
  const size_t C1 = (size_t)std::max<long long>(1, Ctot);
  JSV_T("s1: uploads issued");
  CK(B[B_ITEMS].ensure(sizeof(uint32_t) * C1 * pl.maxi));
  CK(B[B_NITEMS].ensure(sizeof(int) * C1));
  CK(B[B_ARR].ensure(sizeof(double) * C1 * D));
  CK(B[B_SL].ensure(sizeof(int) * C1));
  CK(B[B_FLAG].ensure(sizeof(unsigned) * C1));
  CK(B[B_FRONT].ensure(sizeof(int) * C1));
  CK(B[B_FPOS].ensure(sizeof(int) * C1));
  CK(B[B_FCR].ensure(sizeof(int) * C1));
  CK(B[B_SORTED].ensure(sizeof(int) * C1));
  CK(B[B_SCR].ensure(sizeof(int) * C1));
  CK(B[B_ORDER].ensure(sizeof(int) * C1));
  CK(B[B_BSTART].ensure(sizeof(int) * jobs * (rq.budget + 2)));
  CK(B[B_SURV].ensure(sizeof(int) * C1));
  CK(B[B_PCNT].ensure(sizeof(int) * C1));
  CK(B[B_SBST].ensure(sizeof(int) * jobs * (rq.budget + 2)));
  CK(B[B_SCNT].ensure(sizeof(int) * jobs));
  CK(B[B_CNT].ensure(sizeof(int) * jobs));
  CK(B[B_FCNT].ensure(sizeof(int) * jobs));
  CK(B[B_POOLC].ensure(sizeof(int) * jobs * W));
  CK(B[B_POOLN].ensure(sizeof(int) * jobs));
  CK(B[B_POOLT].ensure(sizeof(int) * jobs));
  CK(B[B_PSL].ensure(sizeof(int) * jobs * W));
  CK(B[B_PCAP].ensure(sizeof(double) * jobs * W));
  CK(B[B_PACC].ensure(sizeof(double) * jobs * W));
  CK(B[B_PLAT].ensure(sizeof(double) * jobs * W));
  CK(B[B_PFAN].ensure(sizeof(double) * jobs * W * p.maxout));
  CK(B[B_S1LAT2].ensure(sizeof(double) * jobs));
  CK(B[B_S1SL].ensure(sizeof(int) * jobs));
  CK(B[B_S1ACC].ensure(sizeof(double) * jobs));
  CK(B[B_ERR].ensure(sizeof(int)));
  // (the fused kernel stores every job's count itself: the zeroing is needed by the
  // chain's atomic counters and by duplicate probes only)
  const bool fused_path = D <= 8 && rq.budget + 2 <= 130 && !getenv("JSV_S1_LEGACY");
  if (!fused_path || n_s1 < n) CK(cudaMemsetAsync(B[B_CNT].p, 0, sizeof(int) * jobs, st));
  CK(cudaMemsetAsync(B[B_ERR].p, 0, sizeof(int), st));
  JSV_T("s1: memsets done");
  S1Args& a = bs.s1;
  memset(&a, 0, sizeof(a));
  a.g = p.dgraph.as<DGraph>();
  a.tb = p.dt;
  a.rq = B[B_REQ].as<DReq>();
  a.probes = B[B_PROBES].as<DProbe>();
  // Stage 1 runs on the first n_s1 probes (distinct Stage-1 inputs); k_s1_expand
  // copies their pools to the duplicate probes n_s1 .. n-1 afterwards
  a.n_probes = n_s1; a.T = T; a.maxi = pl.maxi; a.D = D; a.W = W; a.maxout = p.maxout;
  a.C_probe = pl.C_probe;
  long long acc = 0;
  for (int t = 0; t < T; ++t) {
    a.task_base[t] = acc;
    a.task_cap[t] = pl.task_cap[t];
    acc += pl.task_cap[t];
  }
  a.task_base[T] = acc;
  a.desc = B[B_DESC].as<GenDesc>();
  a.n_desc = (int)pl.desc.size();
  a.U = pl.U;
  a.ways = B[B_WAYS].as<unsigned>();
  a.items = B[B_ITEMS].as<uint32_t>();
  a.nitems = B[B_NITEMS].as<int>();
  a.arr = B[B_ARR].as<double>();
  a.sl = B[B_SL].as<int>();
  a.flag = B[B_FLAG].as<unsigned>();
  a.cnt = B[B_CNT].as<int>();
  a.front = B[B_FRONT].as<int>();
  a.fcnt = B[B_FCNT].as<int>();
  a.fpos = B[B_FPOS].as<int>();
  a.fcr = B[B_FCR].as<int>();
  a.sorted = B[B_SORTED].as<int>();
  a.scr = B[B_SCR].as<int>();
  a.pool_cand = B[B_POOLC].as<int>();
  a.pool_n = B[B_POOLN].as<int>();
  a.pool_trunc = B[B_POOLT].as<int>();
  a.p_sl = B[B_PSL].as<int>();
  a.p_cap = B[B_PCAP].as<double>();
  a.p_acc = B[B_PACC].as<double>();
  a.p_lat = B[B_PLAT].as<double>();
  a.p_fan = B[B_PFAN].as<double>();
  a.pool_min_lat2 = B[B_S1LAT2].as<double>();
  a.pool_min_sl = B[B_S1SL].as<int>();
  a.pool_acc_ub = B[B_S1ACC].as<double>();
  a.err = B[B_ERR].as<int>();
  a.S = rq.budget;
  a.order = B[B_ORDER].as<int>();
  a.bstart = B[B_BSTART].as<int>();
  a.surv = B[B_SURV].as<int>();
  a.pcnt = B[B_PCNT].as<int>();
  a.sbst = B[B_SBST].as<int>();
  a.scnt = B[B_SCNT].as<int>();
  // pair-pass work lists (filled on the device by the kernels that know each job's count)
  long long max_items = 0;
  for (int t = 0; t < T; ++t) {
    const long long cap = pl.task_cap[t];
    max_items += ((cap + 255) / 256) * std::max<long long>(1, (cap + 1023) / 1024);
  }
  max_items = std::max<long long>(1, max_items * n);
  CK(B[B_WL0].ensure(sizeof(int4) * max_items));
  CK(B[B_WL1].ensure(sizeof(int4) * max_items));
  CK(B[B_WL2].ensure(sizeof(int4) * max_items));
  CK(B[B_WN].ensure(sizeof(int) * 4));
  if (!fused_path) CK(cudaMemsetAsync(B[B_WN].p, 0, sizeof(int) * 4, st));
  a.wl[0] = B[B_WL0].as<int4>();
  a.wl[1] = B[B_WL1].as<int4>();
  a.wl[2] = B[B_WL2].as<int4>();
  a.wn = B[B_WN].as<int>();
  CK(B[B_ARRL].ensure(sizeof(double) * C1 * D));
  a.arrl = B[B_ARRL].as<double>();
  CK(B[B_FSORT].ensure(sizeof(int) * jobs));
  a.fsorted = B[B_FSORT].as<int>();
  CK(B[B_ARRF].ensure(sizeof(float4) * C1));
  a.arrf = B[B_ARRF].as<float4>();
  JSV_T("s1: args filled");
  S1Launch L{};
  L.max_items = max_items;
  {
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    L.grid = (long long)n_sm * 8;
  }
  L.tile_task = B[B_TILE_TASK].as<int>();
  L.tile_start = B[B_TILE_START].as<int>();
  L.tiles_pp = (int)pl.tile_task.size();
  L.jchunk_a = 1024;
  L.jchunks_a = (int)std::max<long long>(1, (pl.max_cap + L.jchunk_a - 1) / L.jchunk_a);
  L.jchunk_b = 1024;
  L.jchunks_b = L.jchunks_a;
  // fused Stage 1 (one block per job) unless rows are wider than 16 coordinates or
  // the budget's bucket tables are too large for shared memory
  {
    for (int t = 0, d = 0; t <= T; ++t) {
      while (d < (int)pl.desc.size() && pl.desc[d].task < t) ++d;
      a.desc_t0[t] = d;
    }
  }
  JSV_T("s1: before fused setup");
  const int NB = rq.budget + 2;
  // (measured: wide rows -- fan-out hubs -- and large budgets, whose jobs outgrow the
  // shared-memory lists, run faster through the multi-kernel chain)
  const bool fused = fused_path;
  if (fused) {
    const size_t smax = 100 * 1024;  // two blocks per SM (with the static shared memory)
    long long cap = pl.max_cap;
    if (s1_fused_smem(D, NB, (int)std::min<long long>(cap, 1 << 20)) > smax) {
      const size_t fixed = ((size_t)2 * NB * sizeof(int) + 15) & ~(size_t)15;
      cap = (long long)((smax - fixed - 64) / (5 * sizeof(int) + sizeof(float4) + 1));
    }
    a.fused_cap = (int)std::max<long long>(0, cap);
    const size_t smem = s1_fused_smem(D, NB, a.fused_cap);
    const bool phases = getenv("JSV_S1_PHASES") != nullptr;
    if (phases) {
      CK(B[B_STAMPS].ensure(sizeof(unsigned long long) * 10 * (size_t)n_s1 * T));
      a.stamps = B[B_STAMPS].as<unsigned long long>();
    }
    CK(B[B_S1TESTS].ensure(2 * sizeof(unsigned long long)));
    CK(cudaMemsetAsync(B[B_S1TESTS].p, 0, 2 * sizeof(unsigned long long), st));
    a.tests = B[B_S1TESTS].as<unsigned long long>();
    a.tma = getenv("JSV_NO_TMA") ? 0 : 1;
    a.job_map = n_heavy ? B[B_JOBMAP].as<int>() : nullptr;
    a.job_off = 0;
    c.stats.kernel_launches += launch_stage1_fused(a, smem, n_heavy, st, c.st2, c.fork, c.join);
    JSV_T("s1: launched");
    a.job_map = nullptr;
    if (phases) {
      // mean phase durations over the jobs (diagnostics on stderr)
      std::vector<unsigned long long> h(10 * (size_t)n_s1 * T);
      CK(cudaMemcpyAsync(h.data(), a.stamps, sizeof(unsigned long long) * h.size(),
                         cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      double acc[9] = {0};
      unsigned long long t0 = ~0ull, t1 = 0;
      for (size_t j = 0; j < (size_t)n_s1 * T; ++j) {
        for (int k = 0; k < 8; ++k) acc[k] += (double)(h[j * 10 + k + 1] - h[j * 10 + k]);
        t0 = std::min(t0, h[j * 10]);
        t1 = std::max(t1, h[j * 10 + 8]);
      }
      fprintf(stderr, "[jsv s1] jobs %d span %.1f us; mean us per phase:", n_s1 * T, (t1 - t0) / 1e3);
      for (int k = 0; k < 8; ++k) fprintf(stderr, " %.1f", acc[k] / (n_s1 * T) / 1e3);
      fprintf(stderr, "\n");
      if (atoi(getenv("JSV_S1_PHASES")) > 1)  // per job: task, start and end (us from t0)
        for (size_t j = 0; j < (size_t)n_s1 * T; ++j)
          fprintf(stderr, "[jsv s1 job] %zu %zu %.1f %.1f\n", j, j % T, (h[j * 10] - t0) / 1e3,
                  (h[j * 10 + 8] - t0) / 1e3);
      a.stamps = nullptr;
    }
  } else {
    c.stats.kernel_launches += launch_stage1(a, L, st);
  }
  CK(cudaGetLastError());
  if (n_s1 < n) {
    CK(B[B_REP].ensure(sizeof(int) * n));
    CK(cudaMemcpyAsync(B[B_REP].p, rep.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
    c.stats.kernel_launches += launch_stage1_expand(a, B[B_REP].as<int>(), n_s1, n, st);
    CK(cudaGetLastError());
  }
  bs.n = n;
  // pool sizes, pair-test counters and the error flag into pinned staging, read by
  // stage1_collect after the caller's next synchronisation (Stage 2 of exhaustive
  // probes is planned on the device, so no host round trip sits between the stages)
  {
    // (+ the generated and frontier counts per job: the batch statistics, read here
    // instead of by two synchronous copies after the batch)
    const size_t bytes = sizeof(long long) * 3 + 3 * sizeof(int) * (size_t)jobs;
    char* h = static_cast<char*>(c.pinned(bytes, 2));
    if (!h) return fail(JSV_ERR_CUDA, "cudaHostAlloc failed");
    memset(h, 0, sizeof(long long) * 3);
    if (a.tests) CK(cudaMemcpyAsync(h, a.tests, 2 * sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h + 2 * sizeof(long long), a.err, sizeof(int), cudaMemcpyDeviceToHost, st));
    char* hp = h + 3 * sizeof(long long);
    CK(cudaMemcpyAsync(hp, a.pool_n, sizeof(int) * jobs, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hp + sizeof(int) * jobs, a.cnt, sizeof(int) * jobs, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hp + 2 * sizeof(int) * jobs, a.fcnt, sizeof(int) * jobs, cudaMemcpyDeviceToHost,
                       st));
  }
  bs.s1_pending = true;
  JSV_T("s1: readbacks issued");
  return JSV_OK;
}

// After a synchronisation: Stage 1's readbacks -> pool sizes, dead probes, errors
static int stage1_collect(jsv_problem& p, BatchState& bs) {
  if (!bs.s1_pending) return JSV_OK;
  bs.s1_pending = false;
  jsv_context& c = *p.ctx;
  const int n = bs.n, T = p.T;
  const size_t jobs = (size_t)n * T;
  const char* h = static_cast<const char*>(c.hpin[2]);
  unsigned long long tests[2];
  int err = 0;
  memcpy(tests, h, sizeof(tests));
  memcpy(&err, h + 2 * sizeof(long long), sizeof(int));
  bs.pool_n.resize(jobs);
  memcpy(bs.pool_n.data(), h + 3 * sizeof(long long), sizeof(int) * jobs);
  c.stats.s1_shadow_tests += (long long)tests[0];
  c.stats.s1_exact_tests += (long long)tests[1];
  {
    const int* cnt = reinterpret_cast<const int*>(h + 3 * sizeof(long long)) + jobs;
    const int* fc = cnt + jobs;
    long long gen = 0;
    for (size_t i = 0; i < jobs; ++i) {
      gen += cnt[i];
      c.stats.pair_tests_a += (long long)cnt[i] * cnt[i];
      c.stats.pair_tests_b += (long long)fc[i] * fc[i];
    }
    c.stats.candidates_generated += gen;
    c.stats.dims = bs.s1.D;
  }
  if (err) return fail(JSV_ERR_CAPACITY, "stage-1 candidate capacity exceeded (code " +
                                             std::to_string(err) + ")");
  bs.dead.assign(n, 0);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < T; ++k) {
      const int t = p.topo[k];
      if (bs.pool_n[(size_t)i * T + t] == 0 && !((bs.probes[i].could_zero >> t) & 1u)) {
        bs.dead[i] = 1;
        break;
      }
    }
  return JSV_OK;
}

static void s2_base(jsv_problem& p, BatchState& bs, S2Args& a) {
  jsv_context& c = *p.ctx;
  auto& B = c.buf;
  memset(&a, 0, sizeof(a));
  a.g = p.dgraph.as<DGraph>();
  a.rq = B[B_REQ].as<DReq>();
  a.probes = B[B_PROBES].as<DProbe>();
  a.n_probes = bs.n;
  a.T = p.T;
  a.W = bs.s1.W;
  a.maxout = p.maxout;
  a.pool_n = bs.s1.pool_n;
  a.p_sl = bs.s1.p_sl;
  a.p_cap = bs.s1.p_cap;
  a.p_acc = bs.s1.p_acc;
  a.p_lat = bs.s1.p_lat;
  a.p_fan = bs.s1.p_fan;
  a.items = bs.s1.items;
  a.nitems = bs.s1.nitems;
  a.pool_cand = bs.s1.pool_cand;
  a.C_probe = bs.s1.C_probe;
  for (int t = 0; t <= p.T; ++t) a.task_base[t] = bs.s1.task_base[t];
  a.maxi = bs.s1.maxi;
  a.min_lat2 = B[B_S2LAT2].as<double>();
  a.min_sl = B[B_S2SL].as<int>();
  a.acc_ub = B[B_S2ACC].as<double>();
  a.future = B[B_FUT].as<int>();
  a.best = B[B_BEST].as<BestRec>();
  a.err = B[B_ERR].as<int>();
}

// Level-synchronous search over the active probes (T-informed plans).
//
// Frontier memory is bounded: when a level's children (an upper bound: every
// bundle passing the slices trim of every live prefix) would exceed
// JSV_BB_MAX_SLOTS (default 2^25), the level's frontier is split in two halves per
// probe and each half is expanded depth-first on its own (recursively, so deeper
// levels split the same way).  Every filter is admissible and the per-probe
// incumbent, kill counts, deepest blocked level and best leaf persist across the
// chunks (k_s2_reduce merges), so the result does not depend on the chunking.
struct BBState {
  jsv_problem* p;
  BatchState* bs;
  S2Args a;
  bool diag;
  long long max_slots;
  long long nodes = 0;
  std::vector<long long>* nodes_out;
};

static int bb_level(BBState& S, int L, DevBuf* cur, DevBuf* ccnt, const std::vector<long long>& foff,
                    const std::vector<long long>& fcap, DevBuf* ckey = nullptr) {
  jsv_problem& p = *S.p;
  BatchState& bs = *S.bs;
  jsv_context& c = *p.ctx;
  cudaStream_t st = c.st;
  auto& B = c.buf;
  S2Args& a = S.a;
  const int n = bs.n, T = p.T, P = p.P;
  const bool diag = S.diag;
  long long n_slots = 0;
  for (int i = 0; i < n; ++i) n_slots = std::max(n_slots, foff[i] + fcap[i]);
  std::vector<long long> pstart(n), nxt_off(n), nxt_cap(n), boff(n + 1);
  std::vector<unsigned long long> ptot(n), fcnt(n);
  JSV_T("s2 level begin");
  if (timing_on()) fprintf(stderr, "[jsv t] level %d slots %lld n %d\n", L, n_slots, n);
  const bool last = (L == T - 1);
  const size_t S1 = (size_t)std::max<long long>(1, n_slots);
  CK(B[B_FOFF].ensure(sizeof(long long) * n));
  CK(B[B_FCAP].ensure(sizeof(long long) * n));
  CK(cudaMemcpyAsync(B[B_FOFF].p, foff.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(B[B_FCAP].p, fcap.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, st));
  CK(B[B_PWIDTH].ensure(sizeof(long long) * (S1 + 1)));
  CK(B[B_PFLAG].ensure(sizeof(int) * S1));
  CK(B[B_PPROBE].ensure(sizeof(int) * S1));
  CK(B[B_PR].ensure(sizeof(double) * S1));
  CK(B[B_PUSED].ensure(sizeof(int) * S1));
  CK(B[B_PLATS].ensure(sizeof(double) * S1 * P));
  CK(B[B_PACCS].ensure(sizeof(double) * S1 * P));
  CK(B[B_PTOT].ensure(sizeof(unsigned long long) * n));
  CK(B[B_PFX].ensure(sizeof(long long) * (S1 + 1)));
  CK(cudaMemsetAsync(B[B_PTOT].p, 0, sizeof(unsigned long long) * n, st));
  if (diag) {
    CK(B[B_FLAGS].ensure(sizeof(int) * S1));
    CK(cudaMemsetAsync(B[B_FLAGS].p, 0, sizeof(int) * S1, st));
  }
  a.level = L;
  a.last = last ? 1 : 0;
  a.n_slots = n_slots;
  a.foff = B[B_FOFF].as<long long>();
  a.fcap = B[B_FCAP].as<long long>();
  a.fcnt = ccnt->as<unsigned long long>();
  a.cur = cur->as<uint16_t>();
  a.cur_flag = B[B_FLAGS].as<int>();
  a.pr_width = B[B_PWIDTH].as<long long>();
  a.pr_flag = B[B_PFLAG].as<int>();
  a.pr_probe = B[B_PPROBE].as<int>();
  a.pr_r = B[B_PR].as<double>();
  a.pr_used = B[B_PUSED].as<int>();
  a.pr_lat = B[B_PLATS].as<double>();
  a.pr_acc = B[B_PACCS].as<double>();
  a.ptot = B[B_PTOT].as<unsigned long long>();
  a.pfx = B[B_PFX].as<long long>();
  // (the scan's extra input slot n_slots: width 0)
  CK(cudaMemsetAsync(a.pr_width + n_slots, 0, sizeof(long long), st));
  c.stats.kernel_launches += launch_stage2_prefix(a, st);
  CK(cudaGetLastError());
  // exclusive scan of the per-slot widths (width 0 beyond the live prefixes)
  {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, a.pr_width, a.pfx, n_slots + 1, st));
    CK(B[B_SCAN].ensure(tmp));
    CK(cub::DeviceScan::ExclusiveSum(B[B_SCAN].p, tmp, a.pr_width, a.pfx, n_slots + 1, st));
  }
  CK(cudaMemcpyAsync(ptot.data(), a.ptot, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(fcnt.data(), a.fcnt, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  long long total = 0;
  for (int i = 0; i < n; ++i) {
    fcnt[i] = std::min<unsigned long long>(fcnt[i], (unsigned long long)fcap[i]);
    pstart[i] = total;
    total += (long long)ptot[i];
  }
  // ---- split: the children would not fit -> two halves of every probe's frontier
  if (!last && total > S.max_slots) {
    bool can = false;
    for (int i = 0; i < n; ++i) can = can || fcnt[i] >= 2;
    if (can) {
      if (timing_on()) fprintf(stderr, "[jsv t] level %d split (%lld children)\n", L, total);
      if (ckey) {
        // best-first: the frontier ordered by its children's objective bound (the
        // halves below are copied from the sorted rows and stay sorted: ckey = null)
        std::vector<long long> sege(n);
        long long max_cap = 0;
        for (int i = 0; i < n; ++i) {
          sege[i] = foff[i] + fcap[i];
          max_cap = std::max(max_cap, fcap[i]);
        }
        CK(B[B_SRT_SEGE].ensure(sizeof(long long) * n));
        CK(cudaMemcpyAsync(B[B_SRT_SEGE].p, sege.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, st));
        CK(B[B_SRT_KTMP].ensure(sizeof(double) * S1));
        CK(B[B_SRT_KOUT].ensure(sizeof(double) * S1));
        CK(B[B_SRT_PERM].ensure(sizeof(int) * S1));
        CK(B[B_SRT_PERMO].ensure(sizeof(int) * S1));
        CK(B[B_SRT_ROWS].ensure(sizeof(uint16_t) * S1 * T));
        size_t sb = 0;
        CK((cudaError_t)launch_frontier_best_first(nullptr, nullptr, nullptr, B[B_SRT_KTMP].as<double>(),
                                                   B[B_SRT_KOUT].as<double>(), B[B_SRT_PERM].as<int>(),
                                                   B[B_SRT_PERMO].as<int>(), nullptr, &sb, a.foff, a.fcap,
                                                   B[B_SRT_SEGE].as<long long>(), a.fcnt, n, n_slots,
                                                   max_cap, T, st));
        CK(B[B_SRT_TMP].ensure(std::max<size_t>(sb, 16)));
        CK(cudaGetLastError());  // (nothing pending before the sort)
        CK((cudaError_t)launch_frontier_best_first(
            ckey->as<double>(), cur->as<uint16_t>(), B[B_SRT_ROWS].as<uint16_t>(), B[B_SRT_KTMP].as<double>(),
            B[B_SRT_KOUT].as<double>(), B[B_SRT_PERM].as<int>(), B[B_SRT_PERMO].as<int>(), B[B_SRT_TMP].p,
            &sb, a.foff, a.fcap, B[B_SRT_SEGE].as<long long>(), a.fcnt, n, n_slots, max_cap, T, st));
        c.stats.kernel_launches += 3;
      }
      for (int half = 0; half < 2; ++half) {
        std::vector<long long> hoff(n), hcap(n);
        std::vector<unsigned long long> hcnt(n);
        long long rows = 0;
        for (int i = 0; i < n; ++i) {
          const long long m = (long long)fcnt[i], h = (m + 1) / 2;
          const long long lo = half ? h : 0, hi = half ? m : (m >= 2 ? h : m);
          hoff[i] = rows;
          hcap[i] = hi - lo;
          hcnt[i] = (unsigned long long)(hi - lo);
          rows += hi - lo;
        }
        auto fr = std::make_unique<DevBuf>();
        auto cn = std::make_unique<DevBuf>();
        CK(fr->ensure(sizeof(uint16_t) * std::max<long long>(1, rows) * T));
        CK(cn->ensure(sizeof(unsigned long long) * n));
        for (int i = 0; i < n; ++i) {
          const long long m = (long long)fcnt[i], h = (m + 1) / 2;
          const long long lo = half ? h : 0;
          if (hcap[i] > 0)
            CK(cudaMemcpyAsync(fr->as<uint16_t>() + hoff[i] * T, cur->as<uint16_t>() + (foff[i] + lo) * T,
                               sizeof(uint16_t) * hcap[i] * T, cudaMemcpyDeviceToDevice, st));
        }
        CK(cudaMemcpyAsync(cn->p, hcnt.data(), sizeof(unsigned long long) * n, cudaMemcpyHostToDevice, st));
        int rc = bb_level(S, L, fr.get(), cn.get(), hoff, hcap);
        if (rc) return rc;
        CK(cudaStreamSynchronize(st));  // (before the halves' buffers are freed)
      }
      return JSV_OK;
    }
  }
  for (int i = 0; i < n; ++i) {
    S.nodes += (long long)fcnt[i];
    if (S.nodes_out) (*S.nodes_out)[i] += (long long)fcnt[i];  // frontier prefixes of probe i
  }
  if (last && !diag) c.stats.leaf_work += total;
  DevBuf* nxt = nullptr;
  DevBuf* ncnt = nullptr;
  DevBuf* nkey = nullptr;
  std::vector<long long> noff(n), ncap(n);
  if (total > 0) {
    CK(B[B_PSTART].ensure(sizeof(long long) * n));
    CK(cudaMemcpyAsync(B[B_PSTART].p, pstart.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, st));
    a.pstart = B[B_PSTART].as<long long>();
    if (last) {
      long long nb = 0;
      const long long per_block = 256LL * a.ipt;
      for (int i = 0; i < n; ++i) {
        boff[i] = nb;
        nb += ((long long)ptot[i] + per_block - 1) / per_block;
      }
      boff[n] = nb;
      CK(B[B_BOFF].ensure(sizeof(long long) * (n + 1)));
      CK(cudaMemcpyAsync(B[B_BOFF].p, boff.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice,
                         st));
      CK(B[B_PART].ensure(sizeof(LeafPart) * std::max<long long>(1, nb)));
      a.boff = B[B_BOFF].as<long long>();
      a.part = B[B_PART].as<LeafPart>();
      c.stats.kernel_launches += launch_stage2_leaf(a, nb, st);
    } else {
      long long NO = 0;
      for (int i = 0; i < n; ++i) {
        nxt_off[i] = NO;
        nxt_cap[i] = (long long)ptot[i];
        NO += nxt_cap[i];
      }
      if ((int)c.bb_fr.size() <= L + 1) {
        c.bb_fr.resize(L + 2);
        c.bb_cnt.resize(L + 2);
      }
      if (!c.bb_fr[L + 1]) {
        c.bb_fr[L + 1] = std::make_unique<DevBuf>();
        c.bb_cnt[L + 1] = std::make_unique<DevBuf>();
      }
      if ((int)c.bb_key.size() <= L + 1) c.bb_key.resize(L + 2);
      if (!c.bb_key[L + 1]) c.bb_key[L + 1] = std::make_unique<DevBuf>();
      // children's objective bounds (full plans only: the order a later split uses)
      nkey = (a.mode == LEAF_FULL && !diag) ? c.bb_key[L + 1].get() : nullptr;
      if (nkey) CK(nkey->ensure(sizeof(double) * std::max<long long>(1, NO)));
      a.nxt_key = nkey ? nkey->as<double>() : nullptr;
      nxt = c.bb_fr[L + 1].get();
      ncnt = c.bb_cnt[L + 1].get();
      CK(B[B_NXTOFF].ensure(sizeof(long long) * n));
      CK(B[B_NXTCAP].ensure(sizeof(long long) * n));
      CK(ncnt->ensure(sizeof(unsigned long long) * n));
      CK(cudaMemcpyAsync(B[B_NXTOFF].p, nxt_off.data(), sizeof(long long) * n, cudaMemcpyHostToDevice,
                         st));
      CK(cudaMemcpyAsync(B[B_NXTCAP].p, nxt_cap.data(), sizeof(long long) * n, cudaMemcpyHostToDevice,
                         st));
      CK(cudaMemsetAsync(ncnt->p, 0, sizeof(unsigned long long) * n, st));
      CK(nxt->ensure(sizeof(uint16_t) * std::max<long long>(1, NO) * T));
      a.nxt = nxt->as<uint16_t>();
      a.nxt_cnt = ncnt->as<unsigned long long>();
      a.nxt_off = B[B_NXTOFF].as<long long>();
      a.nxt_cap = B[B_NXTCAP].as<long long>();
      c.stats.kernel_launches += launch_stage2_level(a, total, st);
    }
    CK(cudaGetLastError());
  }
  if (diag) c.stats.kernel_launches += launch_stage2_blocked(a, st);
  if (last || total == 0) return JSV_OK;
  // next frontier: slots [nxt_off, nxt_off + nxt_cap) per probe, live counts on the device
  return bb_level(S, L + 1, nxt, ncnt, nxt_off, nxt_cap, nkey);
}

static int run_stage2(jsv_problem& p, BatchState& bs, bool diag, bool want_config,
                      const std::vector<int>& active, std::vector<long long>* nodes_out) {
  jsv_context& c = *p.ctx;
  cudaStream_t st = c.st;
  auto& B = c.buf;
  const int n = bs.n, T = p.T;
  BBState S;
  S.p = &p;
  S.bs = &bs;
  S.diag = diag;
  S.nodes_out = nodes_out;
  // Deep graphs' full plans: small chunks make the search depth-first enough that
  // leaves -- and with them the incumbent whose objective bound prunes every level --
  // come early (layered 1->4->4->3: 3 s; one 2^25-slot level at a time does not finish).
  // Shallow graphs and feasibility probes keep wide levels (fewer round trips).
  S.max_slots = (!bs.feasible_only && T >= 6) ? (1LL << 16) : (1LL << 25);
  if (const char* e = getenv("JSV_BB_MAX_SLOTS")) S.max_slots = std::max(1LL, atoll(e));
  if (timing_on())
    fprintf(stderr, "[jsv t] bb run n %d T %d fonly %d diag %d max_slots %lld\n", n, T, bs.feasible_only, (int)diag,
            S.max_slots);
  S2Args& a = S.a;
  s2_base(p, bs, a);
  a.diag = diag ? 1 : 0;
  a.want_config = want_config ? 1 : 0;
  const bool fonly = bs.feasible_only != 0;
  a.mode = fonly ? (want_config ? LEAF_FIRST : LEAF_ANY) : LEAF_FULL;
  a.ipt = 16;
  a.dbg = getenv("JSV_DEBUG") ? 1 : 0;
  CK(B[B_INC].ensure(sizeof(unsigned long long) * n));
  CK(cudaMemsetAsync(B[B_INC].p, 0, sizeof(unsigned long long) * n, st));
  CK(B[B_ACTIVE].ensure(sizeof(int) * n));
  CK(cudaMemsetAsync(B[B_ACTIVE].p, 0, sizeof(int) * n, st));
  a.inc = B[B_INC].as<unsigned long long>();
  a.active = B[B_ACTIVE].as<int>();
  // level-0 frontier: one empty prefix per active probe
  std::vector<long long> foff(n), fcap(n, 1);
  std::vector<unsigned long long> cnt0(n);
  for (int i = 0; i < n; ++i) {
    foff[i] = i;
    cnt0[i] = (active[i] && !bs.dead[i]) ? 1 : 0;
  }
  CK(B[B_FR0].ensure(sizeof(uint16_t) * n * T));
  CK(cudaMemsetAsync(B[B_FR0].p, 0xFF, sizeof(uint16_t) * n * T, st));
  CK(B[B_CNT2].ensure(sizeof(unsigned long long) * n));
  CK(cudaMemcpyAsync(B[B_CNT2].p, cnt0.data(), sizeof(unsigned long long) * n,
                     cudaMemcpyHostToDevice, st));
  int rc = bb_level(S, 0, &B[B_FR0], &B[B_CNT2], foff, fcap);
  if (rc) return rc;
  int err = 0;
  CK(cudaMemcpyAsync(&err, B[B_ERR].p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (err) return fail(JSV_ERR_CAPACITY, "stage-2 frontier capacity exceeded");
  if (nodes_out) c.stats.nodes += S.nodes;  // (not the diagnostic re-run)
  return JSV_OK;
}

static int stage2_prep(jsv_problem& p, BatchState& bs) {
  jsv_context& c = *p.ctx;
  auto& B = c.buf;
  const long long jobs = (long long)bs.n * p.T;
  CK(B[B_S2LAT2].ensure(sizeof(double) * jobs));
  CK(B[B_S2SL].ensure(sizeof(int) * jobs));
  CK(B[B_S2ACC].ensure(sizeof(double) * jobs));
  CK(B[B_FUT].ensure(sizeof(int) * bs.n * (p.T + 1)));
  CK(B[B_BEST].ensure(sizeof(BestRec) * bs.n));
  // (every byte defined: the host copies whole records back)
  CK(cudaMemsetAsync(B[B_BEST].p, 0, sizeof(BestRec) * bs.n, c.st));
  S2Args a;
  s2_base(p, bs, a);
  a.min_lat2 = bs.s1.pool_min_lat2;
  a.min_sl = bs.s1.pool_min_sl;
  a.acc_ub = bs.s1.pool_acc_ub;
  c.stats.kernel_launches += launch_stage2_prep(a, B[B_S2LAT2].as<double>(), B[B_S2SL].as<int>(),
                                                B[B_S2ACC].as<double>(), B[B_FUT].as<int>(), c.st);
  CK(cudaGetLastError());
  return JSV_OK;
}

static int finalize(jsv_problem& p, BatchState& bs, bool uninformed, jsv_plan_out* out,
                    const std::vector<long long>* nodes) {
  jsv_context& c = *p.ctx;
  cudaStream_t st = c.st;
  auto& B = c.buf;
  const int n = bs.n;
  CK(B[B_DEAD].ensure(sizeof(int) * n));
  {
    // (through pinned staging slot 0: its Stage-1 uploads completed before the
    // synchronisations behind us; a pageable source is a staged driver copy)
    int* h = static_cast<int*>(c.pinned(sizeof(int) * n, 0));
    if (!h) return fail(JSV_ERR_CUDA, "cudaHostAlloc failed");
    memcpy(h, bs.dead.data(), sizeof(int) * n);
    CK(cudaMemcpyAsync(B[B_DEAD].p, h, sizeof(int) * n, cudaMemcpyHostToDevice, st));
  }
  CK(B[B_OUT].ensure(sizeof(jsv_plan_out) * n));
  // (every byte of the records defined: k_finalize writes only the graph's tasks/paths)
  CK(cudaMemsetAsync(B[B_OUT].p, 0, sizeof(jsv_plan_out) * n, st));
  FinArgs f{};
  f.g = p.dgraph.as<DGraph>();
  f.tb = p.dt;
  f.rq = B[B_REQ].as<DReq>();
  f.probes = B[B_PROBES].as<DProbe>();
  f.n_probes = n; f.T = p.T; f.W = bs.s1.W; f.maxi = bs.s1.maxi; f.maxout = p.maxout;
  f.C_probe = bs.s1.C_probe;
  for (int t = 0; t <= p.T; ++t) f.task_base[t] = bs.s1.task_base[t];
  f.pool_n = bs.s1.pool_n;
  f.pool_trunc = bs.s1.pool_trunc;
  f.pool_cand = bs.s1.pool_cand;
  f.items = bs.s1.items;
  f.nitems = bs.s1.nitems;
  f.p_sl = bs.s1.p_sl;
  f.p_cap = bs.s1.p_cap;
  f.p_acc = bs.s1.p_acc;
  f.p_lat = bs.s1.p_lat;
  f.p_fan = bs.s1.p_fan;
  f.best = B[B_BEST].as<BestRec>();
  f.dead = B[B_DEAD].as<int>();
  f.uninformed = uninformed ? 1 : 0;
  f.pick = B[B_PICK].as<int>();
  f.uni_kills = B[B_UKILL].as<int>();
  f.out = B[B_OUT].as<jsv_plan_out>();
  if (uninformed) {
    const long long jobs = (long long)n * p.T;
    CK(B[B_PICK].ensure(sizeof(int) * jobs));
    CK(B[B_UKILL].ensure(sizeof(int) * jobs * 5));
    CK(B[B_BEST].ensure(sizeof(BestRec) * n));
    CK(cudaMemsetAsync(B[B_BEST].p, 0, sizeof(BestRec) * n, st));
    f.pick = B[B_PICK].as<int>();
    f.uni_kills = B[B_UKILL].as<int>();
    f.best = B[B_BEST].as<BestRec>();
    S2Args a;
    s2_base(p, bs, a);
    c.stats.kernel_launches +=
        launch_uninformed(a, f, B[B_PICK].as<int>(), B[B_UKILL].as<int>(), st);
  }
  c.stats.kernel_launches += launch_finalize(f, st);
  CK(cudaGetLastError());
  // results through the pinned staging buffer (a pageable copy of the ~5 KB
  // records is staged by the driver at a fraction of the link rate)
  // (a caller's page-locked buffer -- jsv_host_alloc -- takes the copy directly)
  cudaPointerAttributes pa{};
  const bool out_pinned = cudaPointerGetAttributes(&pa, out) == cudaSuccess &&
                          pa.type == cudaMemoryTypeHost;
  cudaGetLastError();  // (an unregistered pointer must not leave a sticky error)
  jsv_plan_out* h =
      out_pinned ? nullptr : static_cast<jsv_plan_out*>(c.pinned(sizeof(jsv_plan_out) * n));
  if (h) {
    CK(cudaMemcpyAsync(h, f.out, sizeof(jsv_plan_out) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    memcpy(out, h, sizeof(jsv_plan_out) * n);
  } else {
    CK(cudaMemcpyAsync(out, f.out, sizeof(jsv_plan_out) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  if (nodes)
    for (int i = 0; i < n; ++i) out[i].nodes += (*nodes)[i];
  return JSV_OK;
}

// Exhaustive Stage 2 (jsv_exhaustive.cuh) for the probes whose Stage-1
// cross-product is at most the context limit; clears active[i] for them.
static int run_exhaustive(jsv_problem& p, BatchState& bs, bool want_config,
                          std::vector<int>& active) {
  jsv_context& c = *p.ctx;
  if (c.strategy == JSV_STRATEGY_SEARCH) return JSV_OK;
  // Feasibility probes (max_demand) under auto: the level-synchronous
  // branch-and-bound prunes infeasible probes early but cannot stop at the first
  // feasible leaf (it materialises whole levels: millions of prefixes at low
  // demand), while the sweep stops as soon as any block finds one.  So the sweep
  // first scans a budget of each probe's index space from the front (DFS order:
  // a leaf found there is the first feasible leaf overall); probes decided there
  // -- found, or swept completely -- are done, the rest go to the search.
  long long fo_budget = 0;
  if (c.strategy == JSV_STRATEGY_AUTO && bs.feasible_only) {
    if (c.shard_world > 1 || getenv("JSV_NO_FEAS_SWEEP")) return JSV_OK;
    // (configs[2] sweep, points/s by budget: 2^18 4,120; 1.5 x 2^18 5,380; 2^19 5,340;
    // 1.5 x 2^19 5,300; 2^20 5,150; 2^22 3,600 -- 2^19 keeps a margin to the cliff)
    fo_budget = 1LL << 19;
    if (const char* e = getenv("JSV_FEAS_BUDGET")) fo_budget = std::max(1LL, atoll(e));
  }
  std::vector<int> truncated(bs.n, 0);
  cudaStream_t st = c.st;
  auto& B = c.buf;
  const int n = bs.n, T = p.T;
  const int W = bs.s1.W;
  const size_t smem_cap = 200 * 1024;
  std::vector<XProbe> xp(n);
  long long cand = 0;
  int max_pn_last = 1, nx = 0;
  for (int i = 0; i < n; ++i) {
    if (!active[i] || bs.dead[i]) continue;
    XProbe& x = xp[i];
    memset(&x, 0, sizeof(x));
    unsigned __int128 N = 1;
    bool over = false;
    for (int k = 0; k < T; ++k) {
      const int t = p.topo[k];
      x.pn[k] = bs.pool_n[(size_t)i * T + t];
      x.radix[k] = x.pn[k] + (int)((bs.probes[i].could_zero >> t) & 1u);
      if (!over) N *= (unsigned)x.radix[k];
      if (N > (unsigned __int128)c.exh_limit) over = true;  // keep filling pn/radix
    }
    if (over || N == 0) continue;
    if (x_smem_bytes(x.pn[T - 1], p.P, p.lat_fast) > smem_cap) continue;
    x.R = x.radix[T - 1];
    const long long Q = (long long)(N / (unsigned)x.R);
    x.q0 = (long long)((__int128)Q * c.shard_rank / c.shard_world);
    const long long q1 = (long long)((__int128)Q * (c.shard_rank + 1) / c.shard_world);
    x.nq = q1 - x.q0;
    if (fo_budget > 0) {
      const long long cap = std::max<long long>(1, fo_budget / x.R);
      if (x.nq > cap) {
        x.nq = cap;
        truncated[i] = 1;
      }
    }
    int glog = 0;
    while ((1 << glog) < x.R && glog < 5) ++glog;
    x.glog = glog;
    x.rounds = 1;  // exhaustive probe
    cand += x.nq * x.R;
    max_pn_last = std::max(max_pn_last, x.pn[T - 1]);
    active[i] = 0;
    ++nx;
  }
  if (nx == 0) return JSV_OK;
  JSV_T("exh: probes planned");
  // every probe's prefix range, concatenated (k_x_live); live lists at the same offsets
  // prefixes per round: short rounds for small batches (their live prefixes spread over
  // more warps; JSV_XROUND overrides)
  int n_slots = x_slots(p.P);
  if (nx <= 8) n_slots = std::min(n_slots, 8);
  if (const char* e = getenv("JSV_XROUND")) n_slots = std::max(1, std::min(x_slots(p.P), atoi(e)));
  // k_x_live's work units: upper prefixes (all prefix digits but the fastest)
  std::vector<long long> uoff(n + 1, 0);
  long long n_pref = 0, n_upper = 0, max_rounds = 0;
  for (int i = 0; i < n; ++i) {
    uoff[i] = n_upper;
    xp[i].loff = n_pref;
    if (xp[i].rounds && xp[i].nq > 0) {
      n_pref += xp[i].nq;
      max_rounds += (xp[i].nq + n_slots - 1) / n_slots;
      const long long Rl = T >= 2 ? xp[i].radix[T - 2] : 1;
      n_upper += (xp[i].q0 + xp[i].nq - 1) / Rl - xp[i].q0 / Rl + 1;
    }
  }
  uoff[n] = n_upper;
  c.stats.exh_candidates += cand;
  c.stats.exh_probes += nx;
  // register records: <= 512 bundles per sink pool (ceil(pool / 32) records per lane)
  int reg = 0;
  if (p.P <= 4 && max_pn_last <= 512 && bs.s1.S < 0x7FFF) reg = 1;
  if (getenv("JSV_NO_RPL")) reg = 0;
  for (int i = 0; i < n; ++i)
    if (xp[i].rounds > 0) xp[i].rpl = reg ? (xp[i].pn[T - 1] + 31) / 32 : 0;
  JSV_T("exh: before xprobe copy");
  // one staged upload for the sweep's per-batch inputs (a copy per array costs
  // microseconds of host time each, on the path to the first Stage-2 kernel):
  // [uoff n+1][roff n+1][work 1][live_cnt n][active n][xr_done n] pad [XProbe n]
  // -- uoff and the probes from the host, everything else zero
  const size_t x_ints = (size_t)(2 * (n + 1) + 1) * sizeof(long long) + 3 * sizeof(int) * (size_t)n;
  const size_t x_head = (x_ints + 15) & ~(size_t)15;
  const size_t x_bytes = x_head + sizeof(XProbe) * (size_t)n;
  CK(B[B_XBOFF].ensure(x_bytes));
  char* xb = B[B_XBOFF].as<char>();
  {
    char* h = static_cast<char*>(c.pinned(x_bytes, 1));
    if (!h) return fail(JSV_ERR_CUDA, "cudaHostAlloc failed");
    memset(h, 0, x_head);
    memcpy(h, uoff.data(), sizeof(long long) * (n + 1));
    memcpy(h + x_head, xp.data(), sizeof(XProbe) * n);
    CK(cudaMemcpyAsync(xb, h, x_bytes, cudaMemcpyHostToDevice, st));
  }
  long long* xL = reinterpret_cast<long long*>(xb);
  int* xI = reinterpret_cast<int*>(xL + 2 * (n + 1) + 1);
  XArgs a;
  memset(&a, 0, sizeof(a));
  s2_base(p, bs, a.s);
  a.s.active = xI + n;
  const bool fonly = bs.feasible_only != 0;
  a.mode = fonly ? (want_config ? LEAF_FIRST : LEAF_ANY) : LEAF_FULL;
  a.xp = reinterpret_cast<XProbe*>(xb + x_head);
  a.tma = (W % 4 == 0) ? 1 : 0;
  a.fast = p.lat_fast ? 1 : 0;
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(bs.probes[i].slo_eff) || !std::isfinite(bs.probes[i].demand)) a.fast = 0;
  {
    const int tl = p.topo[T - 1];
    double mx = 0.0;
    for (int k = p.key_off[tl]; k < p.key_off[tl + 1]; ++k) mx = std::max(mx, p.key_lat[k]);
    a.lat2_max = 2.0 * mx;
  }
  a.max_pn_last = max_pn_last;
  a.rpl = reg;
  a.round = n_slots;
  if (a.fast) {
    CK(B[B_XSACC].ensure(sizeof(double) * (size_t)n * W));
    CK(B[B_XSCAP].ensure(sizeof(double) * (size_t)n * W));
    CK(B[B_XSLAT].ensure(sizeof(double) * (size_t)n * W));
    CK(B[B_XRANK].ensure(sizeof(uint4) * (size_t)n * W));
    CK(B[B_XPACK].ensure(sizeof(uint2) * (size_t)n * W));
    a.xpack = B[B_XPACK].as<uint2>();
    a.sacc = B[B_XSACC].as<double>();
    a.scap = B[B_XSCAP].as<double>();
    a.slat2 = B[B_XSLAT].as<double>();
    a.xrank = B[B_XRANK].as<uint4>();
  }
  a.prune = getenv("JSV_NO_PRUNE") ? 0 : 1;
  if (a.mode == LEAF_FULL) {
    // m tie-breaks: packed keys when T <= 5 and every pool's lists fit k_m_rank's
    // shared memory (ranks of 2 n + 2 <= 2048 sequences fit 11 bits), else ranks
    int max_pool = 0;
    for (int i = 0; i < n; ++i)
      if (xp[i].rounds)
        for (int k = 0; k < T; ++k) max_pool = std::max(max_pool, xp[i].pn[k]);
    a.mkey = (T <= 5 && max_pool <= 1023 && (long long)max_pool * bs.s1.maxi <= 4096 &&
              !getenv("JSV_NO_MKEY")) ? 1 : 0;
    if (a.mkey) {
      CK(B[B_MRANK].ensure(sizeof(uint32_t) * ((size_t)n * T * W + (size_t)n * T)));
      a.s.mkey = B[B_MRANK].as<uint32_t>();
      a.s.mnone = B[B_MRANK].as<uint32_t>() + (size_t)n * T * W;
    } else {
      CK(B[B_MRANK].ensure(sizeof(uint32_t) * (size_t)n * T * W));
      a.s.mrank = B[B_MRANK].as<uint32_t>();
    }
  }
  if (getenv("JSV_NO_FAST")) a.fast = 0;
  if (getenv("JSV_NO_TMA")) a.tma = 0;
  // live lists + their round offsets are built on the device; persistent blocks take
  // fixed chunks of X_CHUNK rounds; the segment of probe i inside chunk o reduces
  // into part slot o + i
  const size_t smem = x_smem_bytes(max_pn_last, p.P, a.fast != 0);
  const long long G = std::max<long long>(1, x_resident_blocks(a, p.P, smem));
  CK(B[B_XLIVE].ensure(sizeof(unsigned) * (size_t)std::max<long long>(1, n_pref)));
  CK(B[B_XPART].ensure(sizeof(XPart) * (size_t)std::max<long long>(1, max_rounds)));
  a.uoff = xL;
  a.roff = xL + (n + 1);
  a.roff_w = xL + (n + 1);
  a.work = reinterpret_cast<unsigned long long*>(xL + 2 * (n + 1));
  a.live_cnt = xI;
  a.live = B[B_XLIVE].as<unsigned>();
  a.xr_done = xI + 2 * n;
  a.xr_zeroed = 1;  // (uploaded as zeros above)
  const long long grid = std::min(G, std::max<long long>(1, (max_rounds + 7) / 8));
  a.part = B[B_XPART].as<XPart>();
  JSV_T("exh: before launch");
  c.stats.kernel_launches +=
      launch_stage2_exhaustive(a, grid, p.P, smem, st, getenv("JSV_NO_SIDE") ? st : c.st2, c.fork,
                               c.join, n_upper, getenv("JSV_NO_SIDE") ? nullptr : c.st3, c.join2);
  CK(cudaGetLastError());
  bool any_trunc = false;
  for (int i = 0; i < n; ++i) any_trunc = any_trunc || truncated[i];
  if (any_trunc) {
    // budgeted feasibility sweep: undecided probes (nothing found in the scanned
    // front of a larger space) continue with the branch-and-bound
    std::vector<BestRec> best(n);
    CK(cudaMemcpyAsync(best.data(), B[B_BEST].p, sizeof(BestRec) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int i = 0; i < n; ++i)
      if (truncated[i] && !best[i].has) active[i] = 1;
  }
  return JSV_OK;
}

// Exhaustive Stage 2 planned on the device (k_x_plan): issued right behind Stage 1
// with no host round trip; the caller synchronises once and reads which probes the
// sweep took (`handled`) and which feasibility scans were truncated.  Returns with
// `issued` false when the batch needs the host-planned path (run_exhaustive).
struct DevExh {
  bool issued = false;
  int* handled_h = nullptr;  // pinned readbacks (valid after the caller's sync)
  int* trunc_h = nullptr;
  long long* totals_h = nullptr;
};

static int run_exhaustive_dev(jsv_problem& p, BatchState& bs, bool want_config, DevExh& dx) {
  jsv_context& c = *p.ctx;
  dx.issued = false;
  // (opt-in, JSV_DEVICE_PLAN=1: measured 2% slower than the host-planned path on the
  // 64-solve batch -- k_x_plan's single block and the grid-stride k_x_live cost more
  // than the host round trip they remove -- and no faster for one solve)
  if (c.strategy == JSV_STRATEGY_SEARCH || !getenv("JSV_DEVICE_PLAN")) return JSV_OK;
  long long fo_budget = 0;
  if (c.strategy == JSV_STRATEGY_AUTO && bs.feasible_only) {
    if (c.shard_world > 1 || getenv("JSV_NO_FEAS_SWEEP")) return JSV_OK;
    fo_budget = 1LL << 19;
    if (const char* e = getenv("JSV_FEAS_BUDGET")) fo_budget = std::max(1LL, atoll(e));
  }
  const int n = bs.n, T = p.T;
  const int W = bs.s1.W;
  if (W > 512 || p.P > 4 || bs.s1.S >= 0x7FFF) return JSV_OK;  // (host path: looped sweeps)
  // live-list capacity bound: per probe min(exh_limit, (W + 1)^(T - 1)) prefixes
  long long per = 1;
  for (int k = 0; k < T - 1 && per <= c.exh_limit; ++k) per *= (long long)(W + 1);
  per = std::min(per, c.exh_limit);
  if (fo_budget > 0) per = std::min(per, fo_budget);
  const long long live_cap = per * n;
  if (live_cap > (64LL << 20)) return JSV_OK;  // > 256 MB of live lists: host-planned path
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(bs.probes[i].slo_eff) || !std::isfinite(bs.probes[i].demand)) return JSV_OK;
  if (!p.lat_fast) return JSV_OK;
  cudaStream_t st = c.st;
  auto& B = c.buf;
  const int n_slots = x_slots(p.P);
  const long long max_rounds = (live_cap + n_slots - 1) / n_slots + n;
  CK(B[B_XPROBE].ensure(sizeof(XProbe) * n));
  CK(B[B_ACTIVE].ensure(sizeof(int) * n));
  CK(cudaMemsetAsync(B[B_ACTIVE].p, 0, sizeof(int) * n, st));
  CK(B[B_XLIVE].ensure(sizeof(unsigned) * (size_t)live_cap));
  CK(B[B_XPART].ensure(sizeof(XPart) * (size_t)max_rounds));
  // [uoff n+1][roff n+1][work 1][totals 4][live_cnt n][handled n][trunc n][xr_done n]
  const size_t ll = (size_t)(2 * (n + 1) + 1 + 4);
  CK(B[B_XBOFF].ensure(sizeof(long long) * ll + sizeof(int) * 4 * (size_t)n));
  long long* L = B[B_XBOFF].as<long long>();
  int* I = reinterpret_cast<int*>(L + ll);
  CK(cudaMemsetAsync(L + (n + 1), 0, sizeof(long long) * (n + 2 + 4) + sizeof(int) * 4 * n, st));
  XArgs a;
  memset(&a, 0, sizeof(a));
  s2_base(p, bs, a.s);
  a.s.active = B[B_ACTIVE].as<int>();
  const bool fonly = bs.feasible_only != 0;
  a.mode = fonly ? (want_config ? LEAF_FIRST : LEAF_ANY) : LEAF_FULL;
  a.xp = B[B_XPROBE].as<XProbe>();
  a.fast = 1;
  {
    const int tl = p.topo[T - 1];
    double mx = 0.0;
    for (int k = p.key_off[tl]; k < p.key_off[tl + 1]; ++k) mx = std::max(mx, p.key_lat[k]);
    a.lat2_max = 2.0 * mx;
  }
  a.max_pn_last = W;
  a.rpl = 1;
  a.round = n_slots;  // (device-planned batches keep full rounds)
  a.prune = getenv("JSV_NO_PRUNE") ? 0 : 1;
  if (a.mode == LEAF_FULL) {
    a.mkey = (T <= 5 && (long long)W * bs.s1.maxi <= 4096 && !getenv("JSV_NO_MKEY")) ? 1 : 0;
    if (a.mkey) {
      CK(B[B_MRANK].ensure(sizeof(uint32_t) * ((size_t)n * T * W + (size_t)n * T)));
      a.s.mkey = B[B_MRANK].as<uint32_t>();
      a.s.mnone = B[B_MRANK].as<uint32_t>() + (size_t)n * T * W;
    } else {
      CK(B[B_MRANK].ensure(sizeof(uint32_t) * (size_t)n * T * W));
      a.s.mrank = B[B_MRANK].as<uint32_t>();
    }
  }
  CK(B[B_XSACC].ensure(sizeof(double) * (size_t)n * W));
  CK(B[B_XSCAP].ensure(sizeof(double) * (size_t)n * W));
  CK(B[B_XSLAT].ensure(sizeof(double) * (size_t)n * W));
  CK(B[B_XRANK].ensure(sizeof(uint4) * (size_t)n * W));
  CK(B[B_XPACK].ensure(sizeof(uint2) * (size_t)n * W));
  a.xpack = B[B_XPACK].as<uint2>();
  a.sacc = B[B_XSACC].as<double>();
  a.scap = B[B_XSCAP].as<double>();
  a.slat2 = B[B_XSLAT].as<double>();
  a.xrank = B[B_XRANK].as<uint4>();
  a.uoff = L;
  a.roff = L + (n + 1);
  a.roff_w = L + (n + 1);
  a.work = reinterpret_cast<unsigned long long*>(L + 2 * (n + 1));
  long long* totals = L + 2 * (n + 1) + 1;
  a.dev_totals = totals;
  a.live_cnt = I;
  a.live = B[B_XLIVE].as<unsigned>();
  a.xr_done = I + 3 * n;
  a.part = B[B_XPART].as<XPart>();
  XPlanArgs pa{};
  pa.exh_limit = c.exh_limit;
  pa.fo_budget = fo_budget;
  pa.live_cap = live_cap;
  pa.shard_rank = c.shard_rank;
  pa.shard_world = c.shard_world;
  pa.reg = 1;
  pa.xp = B[B_XPROBE].as<XProbe>();
  pa.handled = I + n;
  pa.trunc = I + 2 * n;
  pa.uoff = L;
  pa.totals = totals;
  pa.err = B[B_ERR].as<int>();
  c.stats.kernel_launches += launch_x_plan(a, pa, st);
  const size_t smem = x_smem_bytes(W, p.P, true);
  const long long G = std::max<long long>(1, x_resident_blocks(a, p.P, smem));
  c.stats.kernel_launches +=
      launch_stage2_exhaustive(a, G, p.P, smem, st, getenv("JSV_NO_SIDE") ? st : c.st2, c.fork,
                               c.join, -1, getenv("JSV_NO_SIDE") ? nullptr : c.st3, c.join2);
  CK(cudaGetLastError());
  // readbacks for the caller's sync: handled / truncated flags and the totals
  char* h = static_cast<char*>(c.pinned(sizeof(long long) * 4 + sizeof(int) * 2 * (size_t)n, 1));
  if (!h) return fail(JSV_ERR_CUDA, "cudaHostAlloc failed");
  dx.totals_h = reinterpret_cast<long long*>(h);
  dx.handled_h = reinterpret_cast<int*>(h + sizeof(long long) * 4);
  dx.trunc_h = dx.handled_h + n;
  CK(cudaMemcpyAsync(dx.totals_h, totals, sizeof(long long) * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(dx.handled_h, I + n, sizeof(int) * 2 * (size_t)n, cudaMemcpyDeviceToHost, st));
  dx.issued = true;
  return JSV_OK;
}

// Fan-out graphs (one entry, every other task a leaf fed only by it) whose
// cross-product is too large to sweep: knapsack-DP bounded enumeration of the
// near-optimal class vectors + exact evaluation (jsv_fanout.cuh).  Full plans
// only; clears active[i] for the probes it solved.
static int run_fanout(jsv_problem& p, BatchState& bs, std::vector<int>& active, bool want_config) {
  jsv_context& c = *p.ctx;
  // feasible_only with a configuration wanted returns the first feasible leaf in DFS
  // order, not an argmax: the branch-and-bound's job.  Verdict-only probes
  // (max_demand's feasibility probes) need only whether the argmax exists.
  const bool verdict = bs.feasible_only && !want_config;
  if (c.strategy == JSV_STRATEGY_SEARCH || (bs.feasible_only && want_config) || !p.lat_fast)
    return JSV_OK;
  if (getenv("JSV_NO_FANOUT")) return JSV_OK;
  const int n = bs.n, T = p.T;
  if (T < 3 || p.P != T - 1) return JSV_OK;
  FoArgs a;
  memset(&a, 0, sizeof(a));
  a.entry = p.topo[0];
  a.k = T - 1;
  if (p.succ_off[a.entry + 1] - p.succ_off[a.entry] != T - 1) return JSV_OK;
  for (int j = 0; j < a.k; ++j) {
    if (p.path_off[j + 1] - p.path_off[j] != 2 || p.path_task[p.path_off[j]] != a.entry)
      return JSV_OK;
    const int l = p.path_task[p.path_off[j] + 1];
    if (p.succ_off[l + 1] != p.succ_off[l] || p.pred_off[l + 1] - p.pred_off[l] != 1) return JSV_OK;
    a.leaf[j] = l;
    a.edge[j] = p.pred_edge[p.pred_off[l]];
  }
  const int W = bs.s1.W;
  if (W > 1024) return JSV_OK;
  std::vector<int> act(n, 0);
  int P0max = 0, nact = 0;
  for (int i = 0; i < n; ++i) {
    const DProbe& pr = bs.probes[i];
    if (!active[i] || bs.dead[i] || !(pr.alpha > 0) || !(pr.beta >= 0) ||
        !std::isfinite(pr.alpha) || !std::isfinite(pr.beta))
      continue;
    act[i] = 1;
    ++nact;
    P0max = std::max(P0max, bs.pool_n[(size_t)i * T + a.entry]);
  }
  if (nact == 0 || P0max == 0) return JSV_OK;
  cudaStream_t st = c.st;
  auto& B = c.buf;
  a.P0max = P0max;
  a.SB = bs.s1.S;
  const size_t nb0 = (size_t)n * P0max;
  CK(B[B_FOACT].ensure(sizeof(int) * n));
  CK(B[B_FOCLS].ensure(sizeof(FoCls) * nb0 * a.k * W));
  CK(B[B_FONCLS].ensure(sizeof(int) * nb0 * a.k));
  CK(B[B_FOF].ensure(sizeof(double) * nb0 * (a.k + 1) * (size_t)(a.SB + 1)));
  CK(B[B_FOB0].ensure(sizeof(double) * nb0));
  CK(B[B_FOTAU].ensure(sizeof(double) * n));
  const long long cap = 1LL << 22;
  CK(B[B_FOCAND].ensure(sizeof(FoCand) * (size_t)cap));
  CK(B[B_FONCAND].ensure(sizeof(unsigned long long)));
  CK(B[B_FOOVF].ensure(sizeof(int)));
  CK(cudaMemsetAsync(B[B_FOOVF].p, 0, sizeof(int), st));
  CK(cudaMemcpyAsync(B[B_FOACT].p, act.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
  s2_base(p, bs, a.s);
  a.act = B[B_FOACT].as<int>();
  a.cls = B[B_FOCLS].as<FoCls>();
  a.ncls = B[B_FONCLS].as<int>();
  a.F = B[B_FOF].as<double>();
  a.b0best = B[B_FOB0].as<double>();
  a.tau = B[B_FOTAU].as<double>();
  a.cand = B[B_FOCAND].as<FoCand>();
  a.ncand = B[B_FONCAND].as<unsigned long long>();
  a.cand_cap = cap;
  a.overflow = B[B_FOOVF].as<int>();
  a.shard_rank = c.shard_rank;
  a.shard_world = c.shard_world;
  c.stats.kernel_launches += launch_fanout_prep(a, st);
  c.stats.kernel_launches += launch_fanout_tau(a, 1e-9, st);
  CK(cudaGetLastError());
  std::vector<double> tau(n);
  std::vector<BestRec> best(n);
  std::vector<double> step(n, 1e-6);
  for (int round = 0; round < 12; ++round) {
    long long nc = 0;
    c.stats.kernel_launches += launch_fanout_round(a, &nc, st);
    CK(cudaGetLastError());
    if (nc < 0) return fail(JSV_ERR_CAPACITY, "fan-out solver: candidate capacity exceeded");
    c.stats.leaves += nc;
    CK(cudaMemcpyAsync(best.data(), B[B_BEST].p, sizeof(BestRec) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(tau.data(), a.tau, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    bool more = false;
    if (getenv("JSV_DEBUG"))
      for (int i = 0; i < n; ++i)
        if (act[i])
          fprintf(stderr, "[jsv fanout] round %d probe %d cand %lld tau %.17g has %d obj %.17g\n",
                  round, i, nc, tau[i], best[i].has, best[i].obj);
    for (int i = 0; i < n; ++i) {
      if (!act[i]) continue;
      if (!std::isfinite(tau[i])) {  // no entry bundle reaches the accuracy SLO: infeasible
        act[i] = 0;
        // (a full plan's re-run supplies the binding constraint; a shard of a split
        // solve reports "nothing in my block" -- shard.combine_sharded re-runs the
        // whole solve when no shard is feasible)
        if (verdict || c.shard_world > 1) active[i] = 0;
        continue;
      }
      if (best[i].has && verdict) {  // a feasible allocation exists: the probe's verdict
        act[i] = 0;
        active[i] = 0;
        continue;
      }
      if (best[i].has) {
        const double eps = 1e-11 * (1.0 + std::fabs(best[i].obj));
        if (tau[i] <= best[i].obj - eps) {
          act[i] = 0;  // every candidate that could beat or tie the optimum was evaluated
          active[i] = 0;
          continue;
        }
        tau[i] = best[i].obj - 2.0 * eps;
      } else {
        tau[i] -= step[i];
        step[i] *= 100.0;
      }
      more = true;
    }
    if (!more) break;
    CK(cudaMemcpyAsync(a.tau, tau.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(B[B_FOACT].p, act.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
  }
  // probes left active (no feasible plan found) go to the branch-and-bound, whose
  // diagnostic re-run also supplies the binding constraint
  return JSV_OK;
}

// plan() for a batch of probes sharing one request
static int plan_batch_internal(jsv_problem& p, const jsv_request& rq, int n, const jsv_probe* in,
                               jsv_plan_out* out, bool want_config, bool feas_only = false) {
  jsv_context& c = *p.ctx;
  cudaStream_t st = c.st;
  if (rq.pareto_width < 1 || rq.pareto_width > 32766) return fail(JSV_ERR_ARG, "pareto_width");
  if (rq.n_mix < 0 || rq.n_mix > JSV_MAX_MIX) return fail(JSV_ERR_ARG, "too many mix fractions");
  BatchState bs;
  bs.feasible_only = rq.feasible_only;
  // Stage 1 (planner.py:586-635) reads a probe only through its demand upper
  // bounds r_upper: probes with identical bounds (a sweep's shared doubling
  // points, coinciding bisection brackets) get one Stage-1 computation.  The
  // batch is permuted so the distinct probes come first; outputs are permuted
  // back at the end.
  JSV_T("batch entry");
  std::vector<DProbe> fp(n);
  ProbeFactors pf;
  probe_factors(p, rq, pf);
  for (int i = 0; i < n; ++i) fill_probe(p, rq, in[i], fp[i], &pf, true);  // (fp value-initialised)
  JSV_T("probes filled");
  std::vector<int> perm;  // batch slot -> caller index
  std::vector<int> rep;   // batch slot -> slot whose Stage-1 pools it shares
  int n_s1 = n;
  {
    // probes whose Stage-1 inputs (both r_upper rows) are bit-identical share one
    // Stage 1: a 64-bit hash of the rows per probe, the hash set verified by memcmp
    const bool no_dedup = getenv("JSV_NO_S1DEDUP") != nullptr;
    const size_t row = sizeof(double) * p.T;
    auto same = [&](int x, int y) {
      return memcmp(fp[x].r_upper[0], fp[y].r_upper[0], row) == 0 &&
             memcmp(fp[x].r_upper[1], fp[y].r_upper[1], row) == 0;
    };
    std::unordered_map<unsigned long long, int> seen;  // hash -> first slot (chained below)
    seen.reserve(2 * (size_t)n);
    std::vector<int> chain(n, -1);  // next probe index with the same hash
    std::vector<int> slot_of(n, -1);
    std::vector<int> first, dups, dup_rep;
    for (int i = 0; i < n; ++i) {
      unsigned long long h = 1469598103934665603ull;
      for (int a = 0; a < 2; ++a) {
        const unsigned char* b = reinterpret_cast<const unsigned char*>(fp[i].r_upper[a]);
        for (size_t k = 0; k < row; ++k) h = (h ^ b[k]) * 1099511628211ull;
      }
      int match = -1;
      auto it = seen.find(h);
      if (it != seen.end() && !no_dedup)
        for (int j = it->second; j >= 0; j = chain[j])
          if (same(i, j)) {
            match = j;
            break;
          }
      if (match < 0) {
        slot_of[i] = (int)first.size();
        first.push_back(i);
        if (it == seen.end()) seen.emplace(h, i);
        else {
          chain[i] = it->second;
          it->second = i;
        }
      } else {
        dups.push_back(i);
        dup_rep.push_back(slot_of[match]);
      }
    }
    n_s1 = (int)first.size();
    perm = first;
    perm.insert(perm.end(), dups.begin(), dups.end());
    rep.resize(n);
    for (int k = 0; k < n_s1; ++k) rep[k] = k;
    for (size_t k = 0; k < dups.size(); ++k) rep[n_s1 + k] = dup_rep[k];
  }
  if (n_s1 == n) {
    bs.probes.swap(fp);  // (perm is the identity)
  } else {
    bs.probes.resize(n);
    for (int k = 0; k < n; ++k) bs.probes[k] = fp[perm[k]];
  }
  std::unique_ptr<jsv_plan_out[]> pout;  // (uninitialised: every used record is written)
  jsv_plan_out* out_caller = out;
  if (n_s1 < n) {
    pout.reset(new jsv_plan_out[n]);
    out = pout.get();
  }
  JSV_T("batch begin");
  if (timing_on()) fprintf(stderr, "[jsv t] probes %d (stage-1 distinct %d)\n", n, n_s1);
  CK(cudaEventRecord(c.ev[0], st));
  int rc = run_stage1(p, rq, n, bs.probes.data(), bs, n_s1, rep);
  if (rc) return rc;
  JSV_T("stage1 done");
  CK(cudaEventRecord(c.ev[1], st));
  const bool informed = (rq.space & JSV_SPACE_T) != 0;
  std::vector<long long> nodes(n, 0);
  if (informed) {
    rc = stage2_prep(p, bs);
    if (rc) return rc;
    JSV_T("s2 prep issued");
    std::vector<int> active(n, 1);
    DevExh dx;
    rc = run_exhaustive_dev(p, bs, want_config, dx);
    if (rc) return rc;
    CK(cudaStreamSynchronize(st));
    rc = stage1_collect(p, bs);
    if (rc) return rc;
    if (dx.issued) {
      JSV_T("device-planned exhaustive synced");
      int err = 0;
      CK(cudaMemcpy(&err, c.buf[B_ERR].p, sizeof(int), cudaMemcpyDeviceToHost));
      if (err) return fail(JSV_ERR_CAPACITY, "exhaustive live-list capacity exceeded");
      c.stats.exh_candidates += dx.totals_h[2];
      c.stats.exh_probes += (int)dx.totals_h[3];
      std::vector<BestRec> best0;
      bool any_trunc = false;
      for (int i = 0; i < n; ++i) any_trunc = any_trunc || dx.trunc_h[i];
      if (any_trunc) {
        best0.resize(n);
        CK(cudaMemcpy(best0.data(), c.buf[B_BEST].p, sizeof(BestRec) * n, cudaMemcpyDeviceToHost));
      }
      for (int i = 0; i < n; ++i)
        active[i] = !dx.handled_h[i] || (dx.trunc_h[i] && !best0[i].has);
    } else {
      rc = run_exhaustive(p, bs, want_config, active);
      if (rc) return rc;
    }
    JSV_T("exhaustive issued");
    rc = run_fanout(p, bs, active, want_config);
    if (rc) return rc;
    bool any_search = false;
    for (int i = 0; i < n; ++i) any_search = any_search || (active[i] && !bs.dead[i]);
    if (any_search) {
      rc = run_stage2(p, bs, false, want_config, active, &nodes);
      if (rc) return rc;
    }
    JSV_T("search issued");
    // infeasible full plans: diagnostic re-run for the binding constraint
    std::vector<BestRec> best(n);
    CK(cudaMemcpyAsync(best.data(), c.buf[B_BEST].p, sizeof(BestRec) * n, cudaMemcpyDeviceToHost,
                       st));
    CK(cudaStreamSynchronize(st));
    JSV_T("stage2 synced");
    std::vector<int> redo(n, 0);
    bool any = false;
    if (getenv("JSV_DEBUG"))
      for (int i = 0; i < n; ++i)
        fprintf(stderr, "[jsv] probe %d has %d leaves %llu obj %.17g\n", i, best[i].has,
                best[i].leaves, best[i].obj);
    for (int i = 0; i < n; ++i) {
      // (a shard of a split solve skips the diagnosis: shard.combine_sharded re-runs the
      // whole solve when no shard is feasible)
      if (!best[i].has && !bs.dead[i] && want_config && c.shard_world == 1) {
        redo[i] = 1;
        any = true;
      }
      c.stats.leaves += (long long)best[i].leaves;
      c.stats.swept += (long long)best[i].nodes;
      c.stats.live_prefixes += (long long)best[i].live;
    }
    if (any) {
      rc = run_stage2(p, bs, true, want_config, redo, nullptr);
      if (rc) return rc;
    }
    if (feas_only && !want_config) {
      // max_demand probes need only the verdict: a feasible leaf was found
      // (every found leaf passed derive/validate), no derivation of outputs
      CK(cudaEventRecord(c.ev[2], st));
      CK(cudaEventRecord(c.ev[3], st));
      CK(cudaEventSynchronize(c.ev[3]));
      // (only the verdict fields: this path serves max_demand's internal probes,
      // which read nothing else -- zeroing ~5 KB per record cost more than the round)
      for (int k = 0; k < n; ++k) {
        jsv_plan_out& o = out_caller[perm[k]];
        o.feasible = (!bs.dead[k] && best[k].has) ? 1 : 0;
        o.dead = bs.dead[k];
      }
      collect_prof(c);
      float ms1 = 0, ms2 = 0, mst = 0;
      cudaEventElapsedTime(&ms1, c.ev[0], c.ev[1]);
      cudaEventElapsedTime(&ms2, c.ev[1], c.ev[2]);
      cudaEventElapsedTime(&mst, c.ev[0], c.ev[3]);
      c.stats.ms_stage1 += ms1;
      c.stats.ms_stage2 += ms2;
      c.stats.ms_total += mst;
      return JSV_OK;
    }
  }
  JSV_T("stage2 done");
  if (bs.s1_pending) {  // (uninformed plans: no Stage-2 synchronisation happened)
    CK(cudaStreamSynchronize(st));
    rc = stage1_collect(p, bs);
    if (rc) return rc;
  }
  CK(cudaEventRecord(c.ev[2], st));
  rc = finalize(p, bs, !informed, out, &nodes);
  if (rc) return rc;
  if (out != out_caller)
    for (int k = 0; k < n; ++k) out_caller[perm[k]] = out[k];
  CK(cudaEventRecord(c.ev[3], st));
  CK(cudaEventSynchronize(c.ev[3]));
  JSV_T("finalize done");
  collect_prof(c);
  float ms1 = 0, ms2 = 0, mst = 0;
  cudaEventElapsedTime(&ms1, c.ev[0], c.ev[1]);
  cudaEventElapsedTime(&ms2, c.ev[1], c.ev[2]);
  cudaEventElapsedTime(&mst, c.ev[0], c.ev[3]);
  c.stats.ms_stage1 += ms1;
  c.stats.ms_stage2 += ms2;
  c.stats.ms_total += mst;
  return JSV_OK;
}

extern "C" int jsv_plan_batch(jsv_context* ctx, const jsv_problem* prob, const jsv_request* req,
                              int32_t n, const jsv_probe* probes, jsv_plan_out* out) {
  if (!ctx || !prob || !req || !probes || !out || n < 0) return fail(JSV_ERR_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
  if (n == 0) return JSV_OK;
  CK(cudaSetDevice(ctx->device));
  memset(&ctx->stats, 0, sizeof(ctx->stats));
  ProfScope ps(ctx);
  return plan_batch_internal(*const_cast<jsv_problem*>(prob), *req, n, probes, out, true);
}

extern "C" int jsv_plan_batch_shard(jsv_context* ctx, const jsv_problem* prob,
                                    const jsv_request* req, int32_t n, const jsv_probe* probes,
                                    int32_t rank, int32_t world, jsv_plan_out* out) {
  if (!ctx || !prob || !req || !probes || !out || n < 0) return fail(JSV_ERR_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
  if (world < 1 || rank < 0 || rank >= world) return fail(JSV_ERR_ARG, "bad shard rank/world");
  const int r0 = ctx->shard_rank, w0 = ctx->shard_world;
  ctx->shard_rank = rank;
  ctx->shard_world = world;
  const int rc = jsv_plan_batch(ctx, prob, req, n, probes, out);
  ctx->shard_rank = r0;
  ctx->shard_world = w0;
  return rc;
}

extern "C" int jsv_set_strategy(jsv_context* ctx, int strategy, int64_t max_candidates) {
  if (!ctx) return fail(JSV_ERR_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
  if (strategy < JSV_STRATEGY_SEARCH || strategy > JSV_STRATEGY_AUTO)
    return fail(JSV_ERR_ARG, "unknown strategy");
  if (max_candidates < 1) return fail(JSV_ERR_ARG, "max_candidates must be positive");
  ctx->strategy = strategy;
  ctx->exh_limit = max_candidates;
  return JSV_OK;
}

extern "C" int jsv_set_shard(jsv_context* ctx, int rank, int world) {
  if (!ctx) return fail(JSV_ERR_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
  if (world < 1 || rank < 0 || rank >= world) return fail(JSV_ERR_ARG, "bad shard rank/world");
  ctx->shard_rank = rank;
  ctx->shard_world = world;
  return JSV_OK;
}

extern "C" void* jsv_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    fail(JSV_ERR_CUDA, "cudaHostAlloc failed");
    return nullptr;
  }
  return p;
}

extern "C" void jsv_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

extern "C" int jsv_last_stats(jsv_context* ctx, jsv_stats* out) {
  if (!ctx || !out) return fail(JSV_ERR_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
  *out = ctx->stats;
  return JSV_OK;
}

// ------------------------------------------------------------- max_demand

struct PointState {
  double lo = 0, hi = 0;
  int phase = 0;  // 0 start, 1 doubling, 2 bisection, 3 done
  int probes = 0;
  int status = 0;
};

extern "C" int jsv_max_demand_batch(jsv_context* ctx, const jsv_problem* prob,
                                    const jsv_request* req, int32_t n, const jsv_probe* points,
                                    double rel_tol, jsv_demand_out* out, jsv_plan_out* plans) {
  if (!ctx || !prob || !req || !points || !out || n < 0) return fail(JSV_ERR_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
  if (req->budget <= 0) return fail(JSV_ERR_CONFIG, "slice budget must be positive");
  if (n == 0) return JSV_OK;
  CK(cudaSetDevice(ctx->device));
  memset(&ctx->stats, 0, sizeof(ctx->stats));
  ProfScope pscope(ctx);
  jsv_problem& p = *const_cast<jsv_problem*>(prob);
  jsv_request preq = *req;
  preq.feasible_only = 1;
  std::vector<PointState> ps(n);
  std::vector<long long> gpu_probes(n, 0);
  const double tiny = 1e-6;
  // speculative evaluation helper: run the listed (point, demand) probes
  auto run = [&](const std::vector<std::pair<int, double>>& work, std::vector<int>& feas) -> int {
    std::vector<jsv_probe> pr(work.size());
    for (size_t k = 0; k < work.size(); ++k) {
      pr[k] = points[work[k].first];
      pr[k].demand = work[k].second;
      gpu_probes[work[k].first]++;
    }
    if (getenv("JSV_DEBUG_DUP")) {
      std::vector<double> dd;
      for (auto& w : work) dd.push_back(w.second);
      std::sort(dd.begin(), dd.end());
      const size_t distinct = std::unique(dd.begin(), dd.end()) - dd.begin();
      fprintf(stderr, "[jsv dup] probes %zu distinct demands %zu\n", work.size(), distinct);
    }
    // (verdict-only probes: plan_batch_internal writes just feasible/dead of each
    // record, so the ~5 KB records are neither zeroed nor filled)
    std::unique_ptr<jsv_plan_out[]> res(new jsv_plan_out[work.size()]);
    int rc = plan_batch_internal(p, preq, (int)work.size(), pr.data(), res.get(), false, true);
    if (rc) return rc;
    feas.resize(work.size());
    for (size_t k = 0; k < work.size(); ++k) feas[k] = res[k].feasible;
    return JSV_OK;
  };
  // step 1: tiny and 1.0 (planner.py:1152-1157)
  {
    std::vector<std::pair<int, double>> w;
    for (int i = 0; i < n; ++i) {
      w.push_back({i, tiny});
      w.push_back({i, 1.0});
    }
    std::vector<int> f;
    int rc = run(w, f);
    if (rc) return rc;
    for (int i = 0; i < n; ++i) {
      PointState& s = ps[i];
      s.probes = 1;
      if (!f[2 * i]) {
        s.status = 1;
        s.phase = 3;
        s.lo = 0.0;
        continue;
      }
      s.probes = 2;
      if (f[2 * i + 1]) {
        s.lo = 1.0; s.hi = 2.0; s.phase = 1;
      } else {
        s.lo = tiny; s.hi = 1.0; s.phase = 2;
      }
    }
  }
  // speculation depth: a round costs ~F of latency (launches, host round trips)
  // plus ~c per probe; a depth-d bisection subtree resolves d levels with
  // 2^d - 1 probes, so pick d minimising (F + active (2^d - 1) c) / d
  double round_ms = 1.0, probe_ms = 0.01;
  if (const char* e = getenv("JSV_SPEC_ROUND_MS")) round_ms = atof(e);
  if (const char* e = getenv("JSV_SPEC_PROBE_MS")) probe_ms = atof(e);
  const int force_depth = getenv("JSV_SPEC_DEPTH") ? atoi(getenv("JSV_SPEC_DEPTH")) : 0;
  while (true) {
    int active = 0;
    for (auto& s : ps) active += (s.phase == 1 || s.phase == 2);
    if (!active) break;
    int depth = 1;
    double best_rate = 1e300;
    for (int d = 1; d <= 8; ++d) {
      const double r = (round_ms + (double)active * ((1 << d) - 1) * probe_ms) / d;
      if (r < best_rate) {
        best_rate = r;
        depth = d;
      }
    }
    if (force_depth > 0) depth = force_depth;
    std::vector<std::pair<int, double>> w;
    std::vector<std::vector<double>> tree(n);
    for (int i = 0; i < n; ++i) {
      PointState& s = ps[i];
      if (s.phase == 1) {
        // speculative doubling: hi, 2hi, 4hi, ...
        const int k = std::max(2, depth + 2);
        double h = s.hi;
        for (int j = 0; j < k && h <= std::ldexp(1.0, 61); ++j) {
          w.push_back({i, h});
          tree[i].push_back(h);
          h *= 2.0;
        }
      } else if (s.phase == 2) {
        // complete bisection subtree of the given depth (heap order)
        std::vector<std::pair<double, double>> nodes{{s.lo, s.hi}};
        std::vector<double>& mids = tree[i];
        mids.clear();
        for (int lvl = 0; lvl < depth; ++lvl) {
          std::vector<std::pair<double, double>> nxtn;
          for (auto& nd : nodes) {
            double lo = nd.first, hi = nd.second;
            double mid = NAN;
            if (!std::isnan(lo) && hi - lo > rel_tol * lo) {
              mid = (lo + hi) / 2.0;
              if (mid <= lo || mid >= hi) mid = NAN;
            }
            mids.push_back(mid);
            if (!std::isnan(mid)) w.push_back({i, mid});
            // children: feasible -> (mid, hi), infeasible -> (lo, mid)
            if (std::isnan(mid)) {
              nxtn.push_back({NAN, NAN});
              nxtn.push_back({NAN, NAN});
            } else {
              nxtn.push_back({mid, hi});
              nxtn.push_back({lo, mid});
            }
          }
          nodes.swap(nxtn);
        }
      }
    }
    std::vector<int> f;
    int rc = run(w, f);
    if (rc) return rc;
    // replay decisions exactly (planner.py:1157-1173)
    size_t cursor = 0;
    for (int i = 0; i < n; ++i) {
      PointState& s = ps[i];
      if (s.phase == 1) {
        const size_t cnt = tree[i].size();
        for (size_t k = 0; k < cnt; ++k) {
          s.probes++;
          if (f[cursor + k]) {
            s.lo = s.hi;
            s.hi *= 2.0;
            if (s.hi > std::ldexp(1.0, 60)) {
              s.status = 2;
              s.phase = 3;
              break;
            }
          } else {
            s.phase = 2;
            break;
          }
        }
        cursor += cnt;
      } else if (s.phase == 2) {
        // walk the heap-ordered subtree
        std::vector<double>& mids = tree[i];
        std::vector<int> fv(mids.size(), 0);
        size_t q = cursor;
        for (size_t k = 0; k < mids.size(); ++k)
          if (!std::isnan(mids[k])) fv[k] = f[q++];
        cursor = q;
        size_t node = 0;
        while (node < mids.size()) {
          if (!(s.hi - s.lo > rel_tol * s.lo)) { s.phase = 3; break; }
          const double mid = (s.lo + s.hi) / 2.0;
          if (mid <= s.lo || mid >= s.hi) { s.phase = 3; break; }
          s.probes++;
          if (fv[node]) {
            s.lo = mid;
            node = 2 * node + 1;
          } else {
            s.hi = mid;
            node = 2 * node + 2;
          }
        }
        if (s.phase == 2 && !(s.hi - s.lo > rel_tol * s.lo)) s.phase = 3;
        if (s.phase == 2) {
          const double mid = (s.lo + s.hi) / 2.0;
          if (mid <= s.lo || mid >= s.hi) s.phase = 3;
        }
      }
    }
  }
  for (int i = 0; i < n; ++i) {
    if (ps[i].status == 2)
      return fail(JSV_ERR_CONFIG, "demand search diverged; profile throughput looks unbounded");
  }
  // final plans with the caller's options (planner.py:1155, 1174)
  if (plans) {
    std::vector<jsv_probe> fin(n);
    for (int i = 0; i < n; ++i) {
      fin[i] = points[i];
      fin[i].demand = ps[i].status == 1 ? tiny : ps[i].lo;
    }
    int rc = plan_batch_internal(p, *req, n, fin.data(), plans, true);
    if (rc) return rc;
  }
  for (int i = 0; i < n; ++i) {
    out[i].demand = ps[i].status == 1 ? 0.0 : ps[i].lo;
    out[i].probes = ps[i].probes;
    out[i].status = ps[i].status;
    out[i].gpu_probes = gpu_probes[i];
  }
  return JSV_OK;
}

// --------------------------------------------------------- derive / validate

extern "C" int jsv_derive(jsv_context* ctx, const jsv_problem* prob, const jsv_request* req,
                          const jsv_probe* probe, const int32_t* n_items, const uint32_t* items,
                          jsv_plan_out* out) {
  if (!ctx || !prob || !req || !probe || !n_items || !items || !out)
    return fail(JSV_ERR_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
  CK(cudaSetDevice(ctx->device));
  jsv_problem& p = *const_cast<jsv_problem*>(prob);
  auto& B = ctx->buf;
  cudaStream_t st = ctx->st;
  DReq hreq;
  fill_req(p, *req, hreq);
  DProbe hp;
  fill_probe(p, *req, *probe, hp);
  CK(B[B_REQ].ensure(sizeof(DReq)));
  CK(B[B_PROBES].ensure(sizeof(DProbe)));
  CK(B[B_DN].ensure(sizeof(int) * MAXT));
  CK(B[B_DITEMS].ensure(sizeof(uint32_t) * MAXT * MAXI));
  CK(B[B_OUT].ensure(sizeof(jsv_plan_out)));
  CK(cudaMemcpyAsync(B[B_REQ].p, &hreq, sizeof(DReq), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(B[B_PROBES].p, &hp, sizeof(DProbe), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(B[B_DN].p, n_items, sizeof(int) * p.T, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(B[B_DITEMS].p, items, sizeof(uint32_t) * p.T * MAXI, cudaMemcpyHostToDevice, st));
  DeriveArgs a{};
  a.g = p.dgraph.as<DGraph>();
  a.tb = p.dt;
  a.rq = B[B_REQ].as<DReq>();
  a.probe = B[B_PROBES].as<DProbe>();
  a.n_items = B[B_DN].as<int>();
  a.items = B[B_DITEMS].as<uint32_t>();
  a.out = B[B_OUT].as<jsv_plan_out>();
  launch_derive(a, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, a.out, sizeof(jsv_plan_out), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return JSV_OK;
}

// --------------------------------------------------------- brute_force_plan

extern "C" int jsv_brute_force(jsv_context* ctx, const jsv_problem* prob, const jsv_request* req,
                               const jsv_probe* probe, int32_t max_count, int64_t max_assignments,
                               int64_t* assignments, int32_t* found, jsv_plan_out* out) {
  if (!ctx || !prob || !req || !probe || !assignments || !found || !out)
    return fail(JSV_ERR_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
  CK(cudaSetDevice(ctx->device));
  jsv_problem& p = *const_cast<jsv_problem*>(prob);
  // the request space's keys in the reference's sorted (task, variant, segment, batch)
  // order: tasks by id rank, keys of a task in local key order (planner.py:1210-1227)
  const int sub = ((req->space & JSV_SPACE_A) ? 2 : 0) + ((req->space & JSV_SPACE_S) ? 1 : 0);
  std::vector<int> kt, kl, kc;
  for (int t = 0; t < p.T; ++t) {
    const int lo = p.sub_off[t * 4 + sub], hi = p.sub_off[t * 4 + sub + 1];
    if (hi - lo > MAXI)
      return fail(JSV_ERR_CONFIG, "oracle refuses: more than 16 profile keys for one task "
                                  "(sm_100a brute_force_plan limit)");
    for (int k = lo; k < hi; ++k) {
      const int loc = p.sub_key[k];
      kt.push_back(t);
      kl.push_back(loc);
      kc.push_back(p.key_cost[p.key_off[t] + loc]);
      if (kc.back() < 1) return fail(JSV_ERR_ARG, "slice cost < 1");
    }
  }
  const int K = (int)kt.size(), S = req->budget;
  if (K > BF_MAXK)
    return fail(JSV_ERR_CONFIG, "oracle refuses: more than 64 profile keys "
                                "(sm_100a brute_force_plan limit)");
  if (S < 0) return fail(JSV_ERR_ARG, "negative slice budget");
  if (max_count < 0 || max_count > 0xFFFF) return fail(JSV_ERR_ARG, "max_count outside [0, 65535]");
  // ways[i][left]: suffix counts, saturated above the assignment cap
  const long long SAT = (long long)max_assignments + 1;
  std::vector<long long> ways((size_t)(K + 1) * (S + 1), 1);
  for (int i = K - 1; i >= 0; --i)
    for (int left = 0; left <= S; ++left) {
      long long n = 0;
      const int cap = std::min<int>(max_count, left / kc[i]);
      for (int c = 0; c <= cap && n < SAT; ++c) n += ways[(size_t)(i + 1) * (S + 1) + left - c * kc[i]];
      ways[(size_t)i * (S + 1) + left] = std::min(n, SAT);
    }
  const long long total = ways[S];
  *assignments = total;
  if (total > max_assignments) return fail(JSV_ERR_CONFIG, "oracle refuses: assignment cap exceeded");
  auto& B = ctx->buf;
  cudaStream_t st = ctx->st;
  DReq hreq;
  fill_req(p, *req, hreq);
  DProbe hp;
  fill_probe(p, *req, *probe, hp);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  const int blocks = (int)std::max(1LL, std::min<long long>((total + 255) / 256, (long long)sms * 8));
  CK(B[B_REQ].ensure(sizeof(DReq)));
  CK(B[B_PROBES].ensure(sizeof(DProbe)));
  CK(B[B_BFKEY].ensure(sizeof(int) * 3 * (K + 1)));
  CK(B[B_BFWAYS].ensure(sizeof(long long) * ways.size()));
  CK(B[B_BFPART].ensure(sizeof(BruteBest) * blocks));
  CK(B[B_BFOUT].ensure(64));
  CK(B[B_DN].ensure(sizeof(int) * MAXT));
  CK(B[B_DITEMS].ensure(sizeof(uint32_t) * MAXT * MAXI));
  CK(B[B_OUT].ensure(sizeof(jsv_plan_out)));
  std::vector<int> keys(3 * (K + 1), 0);
  std::copy(kt.begin(), kt.end(), keys.begin());
  std::copy(kl.begin(), kl.end(), keys.begin() + (K + 1));
  std::copy(kc.begin(), kc.end(), keys.begin() + 2 * (K + 1));
  CK(cudaMemcpyAsync(B[B_REQ].p, &hreq, sizeof(DReq), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(B[B_PROBES].p, &hp, sizeof(DProbe), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(B[B_BFKEY].p, keys.data(), sizeof(int) * keys.size(), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(B[B_BFWAYS].p, ways.data(), sizeof(long long) * ways.size(),
                     cudaMemcpyHostToDevice, st));
  BruteArgs a{};
  a.g = p.dgraph.as<DGraph>();
  a.tb = p.dt;
  a.rq = B[B_REQ].as<DReq>();
  a.probe = B[B_PROBES].as<DProbe>();
  a.K = K;
  a.S = S;
  a.maxc = max_count;
  a.key_task = B[B_BFKEY].as<int>();
  a.key_local = B[B_BFKEY].as<int>() + (K + 1);
  a.key_cost = B[B_BFKEY].as<int>() + 2 * (K + 1);
  a.ways = B[B_BFWAYS].as<long long>();
  a.total = total;
  a.part = B[B_BFPART].as<BruteBest>();
  a.found = B[B_BFOUT].as<int>();
  a.win = reinterpret_cast<long long*>(B[B_BFOUT].as<char>() + 8);
  a.n_items = B[B_DN].as<int>();
  a.items = B[B_DITEMS].as<uint32_t>();
  int launches = launch_brute(a, blocks, st);
  DeriveArgs d{};
  d.g = a.g;
  d.tb = p.dt;
  d.rq = a.rq;
  d.probe = a.probe;
  d.n_items = a.n_items;
  d.items = a.items;
  d.out = B[B_OUT].as<jsv_plan_out>();
  launches += launch_derive(d, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, d.out, sizeof(jsv_plan_out), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(found, a.found, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  ctx->stats = jsv_stats{};
  ctx->stats.leaves = total;
  ctx->stats.kernel_launches = launches;
  return JSV_OK;
}

extern "C" int jsv_validate(jsv_context* ctx, const jsv_problem* prob, const jsv_request* req,
                            const jsv_probe* probe, const double* latency, const double* capacity,
                            const double* demand, int32_t total_slices, double a_obj,
                            uint32_t uncovered_mask, jsv_plan_out* out) {
  if (!ctx || !prob || !req || !probe || !latency || !capacity || !demand || !out)
    return fail(JSV_ERR_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
  CK(cudaSetDevice(ctx->device));
  jsv_problem& p = *const_cast<jsv_problem*>(prob);
  auto& B = ctx->buf;
  cudaStream_t st = ctx->st;
  DReq hreq;
  fill_req(p, *req, hreq);
  DProbe hp;
  fill_probe(p, *req, *probe, hp);
  CK(B[B_REQ].ensure(sizeof(DReq)));
  CK(B[B_PROBES].ensure(sizeof(DProbe)));
  CK(B[B_VAL].ensure(sizeof(double) * 3 * MAXT));
  CK(B[B_OUT].ensure(sizeof(jsv_plan_out)));
  double vals[3 * MAXT];
  for (int t = 0; t < p.T; ++t) {
    vals[t] = latency[t];
    vals[MAXT + t] = capacity[t];
    vals[2 * MAXT + t] = demand[t];
  }
  CK(cudaMemcpyAsync(B[B_REQ].p, &hreq, sizeof(DReq), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(B[B_PROBES].p, &hp, sizeof(DProbe), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(B[B_VAL].p, vals, sizeof(vals), cudaMemcpyHostToDevice, st));
  ValidateArgs a{};
  a.g = p.dgraph.as<DGraph>();
  a.rq = B[B_REQ].as<DReq>();
  a.probe = B[B_PROBES].as<DProbe>();
  a.lat = B[B_VAL].as<double>();
  a.cap = B[B_VAL].as<double>() + MAXT;
  a.dem = B[B_VAL].as<double>() + 2 * MAXT;
  a.total_sl = total_slices;
  a.a_obj = a_obj;
  a.uncovered = uncovered_mask;
  a.out = B[B_OUT].as<jsv_plan_out>();
  launch_validate(a, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, a.out, sizeof(jsv_plan_out), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return JSV_OK;
}

extern "C" int jsv_pool_dump(jsv_context* ctx, const jsv_problem* prob, const jsv_request* req,
                             const jsv_probe* probe, int32_t task, int32_t cap, int32_t* n_out,
                             int32_t* n_items, uint32_t* items, double* stats, int32_t* truncated) {
  if (!ctx || !prob || !req || !probe || !n_out) return fail(JSV_ERR_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
  CK(cudaSetDevice(ctx->device));
  jsv_problem& p = *const_cast<jsv_problem*>(prob);
  if (task < 0 || task >= p.T) return fail(JSV_ERR_ARG, "task index");
  BatchState bs;
  bs.probes.resize(1);
  fill_probe(p, *req, *probe, bs.probes[0]);
  int rc = run_stage1(p, *req, 1, bs.probes.data(), bs, 1, std::vector<int>{0});
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->st));
  rc = stage1_collect(p, bs);
  if (rc) return rc;
  const S1Args& a = bs.s1;
  const int P = bs.pool_n[task];
  *n_out = P;
  if (truncated) CK(cudaMemcpy(truncated, a.pool_trunc + task, sizeof(int), cudaMemcpyDeviceToHost));
  if (P > cap) return fail(JSV_ERR_CAPACITY, "output capacity too small");
  const int W = a.W;
  const int outd = p.succ_off[task + 1] - p.succ_off[task];
  std::vector<int> pc(P), sl(P);
  std::vector<double> capv(P), acc(P), lat(P), fan((size_t)P * p.maxout);
  const long long q0 = (long long)task * W;
  if (P > 0) {
    CK(cudaMemcpy(pc.data(), a.pool_cand + q0, sizeof(int) * P, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sl.data(), a.p_sl + q0, sizeof(int) * P, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(capv.data(), a.p_cap + q0, sizeof(double) * P, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(acc.data(), a.p_acc + q0, sizeof(double) * P, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(lat.data(), a.p_lat + q0, sizeof(double) * P, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(fan.data(), a.p_fan + q0 * p.maxout, sizeof(double) * P * p.maxout,
                  cudaMemcpyDeviceToHost));
  }
  const long long base = a.task_base[task];
  for (int k = 0; k < P; ++k) {
    const long long cnd = base + pc[k];
    int ni = 0;
    CK(cudaMemcpy(&ni, a.nitems + cnd, sizeof(int), cudaMemcpyDeviceToHost));
    if (n_items) n_items[k] = ni;
    if (items) {
      uint32_t tmp[MAXI] = {0};
      CK(cudaMemcpy(tmp, a.items + cnd * a.maxi, sizeof(uint32_t) * ni, cudaMemcpyDeviceToHost));
      for (int i = 0; i < MAXI; ++i) items[(size_t)k * MAXI + i] = tmp[i];
    }
    if (stats) {
      double* s = stats + (size_t)k * (4 + outd);
      s[0] = (double)sl[k];
      s[1] = capv[k];
      s[2] = acc[k];
      s[3] = lat[k];
      for (int j = 0; j < outd; ++j) s[4 + j] = fan[(size_t)k * p.maxout + j];
    }
  }
  return JSV_OK;
}
