#include <map>
#include <cub/block/block_scan.cuh>
// jsv_exhaustive.cuh -- exhaustive Stage 2: every allocation of the Stage-1
// cross-product is derived, validated and folded into the argmax (included by
// jsv_stage2.cu).
//
// Candidate space of one probe (one plan() call): a mixed-radix number whose
// digit k (k = topological position, most significant first) picks a bundle of
// task topo[k]'s pool, or -- for a task whose derived demand may be 0
// (_Search.could_zero, planner.py:772-774) -- the extra digit value pool_n = "no
// instances".  A candidate is a leaf of the reference's search tree
// (_Search._visit, planner.py:860-912) iff every chosen digit agrees with the
// derived demand ("no instances" <=> demand 0, planner.py:868-875); all other
// digit vectors are rejected after demand propagation.  Because every filter
// of the reference's branch-and-bound is admissible, plan() equals the
// lexicographic argmax of (objective desc, total slices asc, m asc) over the
// feasible leaves, and feasible_only's "first feasible
// leaf" is the smallest feasible index (digit order = DFS order).
//
// Work decomposition: the last topological task is always a sink, so the
// index splits into (prefix q, last digit b).  A group of G lanes (G = the
// last radix rounded up to a power of two, <= 32) owns one prefix: the lanes
// decode q once, propagate demand and build the prefix's partial verdicts in
// registers (topological order), then sweep b = lane, lane + G, ... over the
// last task's pool, which the block staged into shared memory with one TMA
// bulk copy per column (cp.async.bulk + mbarrier).  Every candidate pays only
// the sink's part of derive/validate.  Two evaluators:
//
//  * rank space (problems whose latencies, capacities, accuracies and path
//    fractions are finite and >= +0 -- every realistic profile): each of the
//    sink's verdicts is monotone in one bundle field, so per prefix the lanes
//    turn the verdict into a threshold on that field's rank among the pool's
//    sorted values (bisection with the reference's own float expressions), and
//    a candidate is decided by four integer compares on one 16-byte record
//    {rank(capacity), rank(accuracy), rank(2 L), slices}.  Latency uses a
//    margin: t = fl(f + 2L) more than 4x the compensated-sum error bound below
//    the SLO passes, above it fails, and the few in between redo CPython 3.12's
//    sum() step exactly.  Feasible leaves recompute W, a_obj and the objective
//    in the reference's order;
//  * float (any other profile): the sink's part of derive/validate in float,
//    one Neumaier step per path through the sink, the accuracy products and
//    path sum, the capacity, resource and accuracy verdicts (model.py:267-299,
//    planner.py:243-361).
// Reduction: per lane, warp shuffles, one shared-memory pass per block, then a
// per-probe fold of the block partials (k_s2_xreduce), all with the same
// lexicographic comparison (ties on m resolved by the canonical item lists).

__device__ __forceinline__ void x_digits(const XProbe& xp, int T, long long idx, uint16_t* ch) {
  unsigned long long v = (unsigned long long)idx;
  for (int k = T - 1; k >= 0; --k) {
    const unsigned r = (unsigned)xp.radix[k];
    unsigned d;
    if (v < 0x100000000ull) {  // 32-bit division once the remaining index fits
      const unsigned v32 = (unsigned)v;
      d = v32 % r;
      v = v32 / r;
    } else {
      d = (unsigned)(v % r);
      v /= r;
    }
    ch[k] = (d == (unsigned)xp.pn[k]) ? (uint16_t)NONE16 : (uint16_t)d;
  }
}

// The canonical m (planner.py:262) lists every item ((task, variant, segment,
// batch), count) in task-id order, so two candidates' m tuples first differ
// inside the item lists of the first task (by id) whose bundles differ.  There the
// m-order ranks decide (k_m_rank) -- unless one list is a proper prefix of the
// other: then the shorter m continues with the next non-empty task's first entry
// (a larger task id: it is the larger tuple) or ends (the smaller one).
// "no instances" is the empty list.
__device__ __forceinline__ bool x_mr_later(const S2Args& a, const uint16_t* ch, int probe, int u) {
  const DGraph& g = *a.g;
  for (int v = u + 1; v < a.T; ++v) {
    const int c = ch[g.pos_of[v]];
    if (c != NONE16 && !(a.mrank[(long long)(probe * a.T + v) * a.W + c] >> 31)) return true;
  }
  return false;
}

// list(task u, bundle c1) vs list(task u, bundle c2), c1 != c2: -1 / +1 when the
// lists differ before either ends, -2 when list 1 is a proper prefix of list 2,
// +2 when list 2 is a proper prefix of list 1
__device__ __forceinline__ int x_mr_cmp(const S2Args& a, int probe, int u, int c1, int c2) {
  const long long q = (long long)(probe * a.T + u) * a.W;
  const unsigned m1 = c1 == NONE16 ? 0x80000000u : a.mrank[q + c1];
  const unsigned m2 = c2 == NONE16 ? 0x80000000u : a.mrank[q + c2];
  const bool e1 = m1 >> 31, e2 = m2 >> 31;
  if (e1 || e2) return e1 && e2 ? 0 : (e1 ? -2 : 2);  // the empty list prefixes every other
  const unsigned r1 = m1 & 0xFFFFu, x1 = (m1 >> 16) & 0x7FFFu;
  const unsigned r2 = m2 & 0xFFFFu, x2 = (m2 >> 16) & 0x7FFFu;
  if (r1 < r2 && r2 <= x1) return -2;
  if (r2 < r1 && r1 <= x2) return 2;
  return r1 < r2 ? -1 : 1;
}

// m(candidate i1) vs m(candidate i2) as Python tuple comparison (planner.py:852)
__device__ __noinline__ int x_cmp_m(const S2Args& a, const XProbe& xp, int probe, long long i1,
                                    long long i2) {
  uint16_t x[MAXT], y[MAXT];
  x_digits(xp, a.T, i1, x);
  x_digits(xp, a.T, i2, y);
  const DGraph& g = *a.g;
  for (int u = 0; u < a.T; ++u) {
    const int p = g.pos_of[u];
    if (x[p] == y[p]) continue;
    const int c = x_mr_cmp(a, probe, u, x[p], y[p]);
    if (c == 0) continue;  // two empty lists
    if (c == -2) return x_mr_later(a, x, probe, u) ? 1 : -1;
    if (c == 2) return x_mr_later(a, y, probe, u) ? -1 : 1;
    return c;
  }
  return 0;
}

// Two leaves of the same prefix differ only in the sink's bundle: its lists decide
// (a proper prefix is the larger m when a later task is non-empty).
__device__ __forceinline__ int x_sink_cmp(const S2Args& a, int probe, int tl, int b1, int b2,
                                          bool later_nonempty) {
  if (b1 == b2) return 0;
  const int c = x_mr_cmp(a, probe, tl, b1, b2);
  if (c == -2) return later_nonempty ? 1 : -1;
  if (c == 2) return later_nonempty ? -1 : 1;
  return c;
}

struct XBest {
  int has, sl;
  double obj;
  long long idx;
  unsigned long long mk;  // packed m key (XArgs::mkey)
};
__device__ __forceinline__ XBest x_none() {
  XBest b;
  b.has = 0; b.sl = 0; b.obj = 0.0; b.idx = 0; b.mk = 0;
  return b;
}

// Packed m keys (XArgs::mkey, T <= 5): the canonical m (planner.py:262) is the
// concatenation of the tasks' item lists in task-id order, so comparing two m
// tuples compares, task by task, each task's list -- followed by "a larger
// entry" when a later task is non-empty, or by the end of the tuple.  k_m_rank
// ranks every list in both forms (11 bits); the key packs them by task id.
__device__ __forceinline__ unsigned long long x_mk_task(const S2Args& s, int probe, int u, int c,
                                                        bool later) {
  const int job = probe * s.T + u;
  const unsigned k = (c == NONE16) ? s.mnone[job] : s.mkey[(long long)job * s.W + c];
  return (unsigned long long)(later ? (k >> 16) : (k & 0xFFFFu)) << (11 * (s.T - 1 - u));
}

// is A a better feasible candidate than B?
__device__ __forceinline__ bool x_better(const XArgs& a, const XProbe& xp, int probe,
                                         const XBest& A, const XBest& B) {
  if (!A.has) return false;
  if (!B.has) return true;
  if (a.mode != LEAF_FULL) return A.idx < B.idx;
  if (A.obj != B.obj) return A.obj > B.obj;
  if (A.sl != B.sl) return A.sl < B.sl;
  if (A.idx == B.idx) return false;
  if (a.mkey) return A.mk < B.mk;
  return x_cmp_m(a.s, xp, probe, A.idx, B.idx) < 0;
}

__device__ __forceinline__ XBest x_shfl_down(const XBest& v, int d) {
  XBest o;
  o.has = __shfl_down_sync(0xffffffffu, v.has, d);
  o.sl = __shfl_down_sync(0xffffffffu, v.sl, d);
  o.obj = __shfl_down_sync(0xffffffffu, v.obj, d);
  o.idx = __shfl_down_sync(0xffffffffu, v.idx, d);
  o.mk = __shfl_down_sync(0xffffffffu, v.mk, d);
  return o;
}

// ------------------------------------------------------------ prefix state

// Per-warp prefix state in shared memory, NS slots (one per computing lane).
template <int PM, int NS>
struct XWarpState {
  double need[NS];        // r_sink * (1.0 + slack)
  long long q[NS];        // prefix index
  int sl[NS];             // slices of the prefix
  int flags[NS];          // bit0 leaf prefix, bit1 prefix verdicts hold, bit2 later task
                          // non-empty, bit3 sink demand 0
  // rank space, per prefix {a_cap, a_acc, l_lat, rem}: a candidate passes every
  // verdict iff rank(cap) >= a_cap, rank(acc) >= a_acc, rank(2L) < l_lat (then
  // the exact latency test if t > lo) and slices <= rem
  uint4 th[NS];
  uint2 sw[NS];           // the same thresholds as the SWAR subtrahends of the packed records
  double s0[PM][NS];      // path through the sink: Neumaier f; other path: frac * product
  double s1[PM][NS];      // path through the sink: Neumaier c
  double s2[PM][NS];      // path through the sink: accuracy product before the sink
  double lo[PM][NS];      // rank space: t = f + 2L <= lo passes without the exact sum
  unsigned long long mk[NS], mkz[NS];  // packed m key of the prefix tasks (sink non-empty / none)
};

// Shared-memory view of the sink pool for the rank-space evaluator.
struct XRankView {
  const uint4* rank;      // {rank(cap), rank(acc), rank(2L), slices} per bundle (+ padding)
  const uint2* pack;      // SWAR form: {H | rank(cap) << 16 | rank(acc),
                          //             H | (0x7FFF - rank(2L)) << 16 | (0x7FFF - slices)}
  const double* scap;     // sorted capacities
  const double* sacc;     // sorted accuracies
  const double* slat2;    // sorted 2 L
  int n;
};

// accuracy verdict of a leaf from its path-weighted sum W (model.py:293,
// planner.py:350-351; W >= acc_thr is the same test, see DProbe.acc_thr)
__device__ __forceinline__ bool x_acc_ok(double W, const DProbe& pr, double a_max) {
  return pr.acc_thr_ok ? (W >= pr.acc_thr) : (W / a_max - pr.acc_slo >= 0);
}

// first k in [0, n] with pred(k) (pred monotone false -> true; n = "none")
template <class F>
__device__ __forceinline__ int x_first(int n, F pred) {
  int lo = -1, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pred(mid)) hi = mid;
    else lo = mid;
  }
  return hi;
}

// derive_configuration of one prefix (all tasks but the sink): demand
// propagation in topological order (model.py:239-264), the verdicts that do not
// involve the sink, and the per-path partial latency sums / accuracy products;
// in rank space also the sink-verdict thresholds.
// Digits of prefix qp, demand propagation in topological order (model.py:239-264),
// the prefix tasks' throughput verdicts (planner.py:345-347) and slices.  Returns
// X_LEAF (every digit agrees with its derived demand), X_THRU (the prefix tasks'
// throughput verdicts hold) and X_ZERO (the sink's demand is 0).
#define X_LEAF 1
#define X_OKPRE 2
#define X_LATER 4
#define X_ZERO 8
#define X_SWEEP 16
#define X_THRU 32
__device__ __forceinline__ int x_demand(const S2Args& s, const DGraph& g, const XProbe& xp,
                                        const DProbe& pr, int probe, long long qp, uint16_t* ch,
                                        double* dem, int& sl_pre) {
  const DReq& rq = *s.rq;
  const int T = s.T, tl = g.topo[T - 1], jb = probe * T;
  {
    unsigned long long idx = (unsigned long long)qp;
    for (int k = T - 2; k >= 0; --k) {
      const unsigned r = (unsigned)xp.radix[k];
      unsigned d;
      if (idx < 0x100000000ull) {
        const unsigned i32 = (unsigned)idx;
        d = i32 % r;
        idx = i32 / r;
      } else {
        d = (unsigned)(idx % r);
        idx /= r;
      }
      ch[k] = (d == (unsigned)xp.pn[k]) ? (uint16_t)NONE16 : (uint16_t)d;
    }
  }
  bool valid = true, ok = true;
  int sl = 0;
  const double sf = 1.0 + rq.slack;
  for (int i = 0; i < T; ++i) {
    const int t = g.topo[i];
    double d;
    if (t == g.entry) {
      d = pr.demand;
    } else {
      d = 0.0;
      for (int k = g.pred_off[t]; k < g.pred_off[t + 1]; ++k) {
        const int e = g.pred_edge[k];
        const int src = g.edge_src[e];
        const int cs = ch[g.pos_of[src]];
        double fan;
        if (rq.has_ov[e]) fan = rq.ov[e];
        else if (cs == NONE16) fan = 0.0;
        else fan = s.p_fan[((long long)(jb + src) * s.W + cs) * s.maxout + (e - g.succ_off[src])];
        d += dem[src] * fan;
      }
    }
    dem[t] = d;
    if (i < T - 1) {
      const int c = ch[i];
      // a leaf of the search tree has "no instances" exactly where demand is 0
      if ((c == NONE16) != (d == 0.0)) valid = false;
      const double cap = (c == NONE16) ? 0.0 : s.p_cap[(long long)(jb + t) * s.W + c];
      if (!(cap - d * sf >= 0)) ok = false;  // planner.py:345-347
      if (c != NONE16) sl += s.p_sl[(long long)(jb + t) * s.W + c];
    }
  }
  sl_pre = sl;
  return (valid ? X_LEAF : 0) | (ok ? X_THRU : 0) | (dem[tl] == 0.0 ? X_ZERO : 0);
}

template <int PM, int NS, bool RANK>
__device__ __forceinline__ void x_prefix(const S2Args& s, const DGraph& g, const XProbe& xp,
                                         const DProbe& pr, int probe, long long qp,
                                         const double* frac, unsigned thru, int slot,
                                         double lat2_max, const XRankView& rv,
                                         XWarpState<PM, NS>& ws, int mkey) {
  const DReq& rq = *s.rq;
  const int T = s.T, P = g.P, tl = g.topo[T - 1], jb = probe * T;
  uint16_t ch[MAXT];
  double dem[MAXT];
  int sl_pre = 0;
  const int dfl = x_demand(s, g, xp, pr, probe, qp, ch, dem, sl_pre);
  const bool valid = (dfl & X_LEAF) != 0;
  bool ok_pre = (dfl & X_THRU) != 0;
  const double sf = 1.0 + rq.slack;
  bool later = false;
  for (int u = tl + 1; u < T; ++u) later = later || ch[g.pos_of[u]] != NONE16;
  double f[PM], c[PM], pp[PM], px[PM];
#pragma unroll
  for (int p = 0; p < PM; ++p) {
    f[p] = 0.0; c[p] = 0.0; pp[p] = 1.0; px[p] = 0.0;
    if (p < P) {
      PySum ps;
      double prod = 1.0;
      const bool through = (thru >> p) & 1u;
      for (int k = g.path_off[p]; k < g.path_off[p + 1]; ++k) {
        const int u = g.path_task[k];
        if (u == tl) break;  // the sink ends every path through it
        const int cc = ch[g.pos_of[u]];
        double lat = 0.0, acc = 1.0;
        if (cc != NONE16) {
          const long long qq = (long long)(jb + u) * s.W + cc;
          lat = s.p_lat[qq];
          acc = s.p_acc[qq];
        }
        ps.add(2.0 * lat);
        prod *= acc;
      }
      if (through) {
        // f = c = 0 reproduces the first-term branch of PySum exactly
        f[p] = ps.any ? ps.f : 0.0;
        c[p] = ps.any ? ps.c : 0.0;
        pp[p] = prod;
      } else {
        if (!(pr.slo_eff - ps.result() >= 0)) ok_pre = false;  // planner.py:339-343
        px[p] = frac[p] * prod;
        f[p] = px[p];
      }
      ws.s0[p][slot] = f[p];
      ws.s1[p][slot] = c[p];
      ws.s2[p][slot] = pp[p];
    }
  }
  const double need = dem[tl] * sf;
  bool sweep = false;
  if (RANK) {
    // Every sink verdict is monotone in one sorted column; the thresholds are
    // found by lockstep binary lifting (first k in [0, n] whose predicate holds,
    // the same count as a bisection), the searches interleaved for latency.
    //  capacity: cap - need >= 0 <=> cap >= need (finite) <=> rank(cap) >= #{caps < need}
    //  accuracy: W is non-decreasing in the sink accuracy (fractions, products >= 0)
    //  latency: the exact compensated sum differs from t = fl(f + 2L) by at most
    //    1.01 (|c| + 2^-52 (f + 2L)); with M = 4x that (+ the rounding of slo -/+ M)
    //    t <= slo - M passes, t > slo + M fails, in between the exact sum decides
    const double slo = pr.slo_eff;
    const bool thr_ok = pr.acc_thr_ok != 0;
    const double acc_thr = pr.acc_thr, acc_slo = pr.acc_slo, a_max = g.a_max;
    double hi[PM];
    int pl[PM];
#pragma unroll
    for (int p = 0; p < PM; ++p) {
      pl[p] = 0;
      hi[p] = 0.0;
      if ((thru >> p) & 1u) {
        const double M = 4.0 * (fabs(c[p]) + 2.220446049250313e-16 * (f[p] + lat2_max + fabs(slo))) +
                         1e-300;
        hi[p] = slo + M;
        ws.lo[p][slot] = slo - M;
      }
    }
    // binary lifting with the probe index clamped to n - 1 (a clamped probe repeats
    // the last predicate, which keeps every sequence monotone), result clamped to n
    const int n = rv.n, nm1 = n - 1;
    const int top = n > 0 ? (1 << (31 - __clz(n))) : 0;
    int pc = 0, pa = 0;
    const double* __restrict__ scap = rv.scap;
    const double* __restrict__ sacc = rv.sacc;
    const double* __restrict__ slat = rv.slat2;
    if (thr_ok) {
      for (int step = top; step > 0; step >>= 1) {
        pc += (scap[min(pc + step - 1, nm1)] >= need) ? 0 : step;
        const double acc = sacc[min(pa + step - 1, nm1)];
        double W = 0.0;
#pragma unroll
        for (int p = 0; p < PM; ++p)
          if (p < P) W += ((thru >> p) & 1u) ? frac[p] * (pp[p] * acc) : px[p];
        pa += (W >= acc_thr) ? 0 : step;
#pragma unroll
        for (int p = 0; p < PM; ++p)
          if ((thru >> p) & 1u) pl[p] += (f[p] + slat[min(pl[p] + step - 1, nm1)] <= hi[p]) ? step : 0;
      }
    } else {
      for (int step = top; step > 0; step >>= 1) {
        pc += (scap[min(pc + step - 1, nm1)] >= need) ? 0 : step;
        const double acc = sacc[min(pa + step - 1, nm1)];
        double W = 0.0;
#pragma unroll
        for (int p = 0; p < PM; ++p)
          if (p < P) W += ((thru >> p) & 1u) ? frac[p] * (pp[p] * acc) : px[p];
        pa += (W / a_max - acc_slo >= 0) ? 0 : step;
#pragma unroll
        for (int p = 0; p < PM; ++p)
          if ((thru >> p) & 1u) pl[p] += (f[p] + slat[min(pl[p] + step - 1, nm1)] <= hi[p]) ? step : 0;
      }
    }
    pc = min(pc, n);
    pa = min(pa, n);
#pragma unroll
    for (int p = 0; p < PM; ++p) pl[p] = min(pl[p], n);
    int l_lat = ok_pre ? n : 0;
#pragma unroll
    for (int p = 0; p < PM; ++p)
      if ((thru >> p) & 1u) l_lat = pl[p] < l_lat ? pl[p] : l_lat;
    // resources: float(S - total) >= 0 <=> slices <= S - prefix; negative fails all
    const int rem = rq.S - sl_pre;
    const uint4 th = make_uint4((unsigned)pc, (unsigned)pa, rem >= 0 ? (unsigned)l_lat : 0u,
                                rem >= 0 ? (unsigned)rem : 0u);
    ws.th[slot] = th;
    // SWAR: two 15-bit fields per word, all "x >= threshold" with a guard bit;
    // (w | H) - B keeps bit 15 of a field iff that field passes
    const unsigned rm = th.w < 0x7FFFu ? th.w : 0x7FFFu;
    // (a slot that is not swept -- not a leaf prefix, or sink demand 0 -- gets
    // l_lat = 0, which no record passes: rank(2L) field 0x7FFF - r never reaches 0x8000)
    const bool swept = valid && dem[tl] != 0.0;
    ws.sw[slot] = make_uint2((th.x << 16) | th.y,
                             ((0x8000u - (swept ? th.z : 0u)) << 16) | (0x7FFFu - rm));
    // some record can pass every threshold: the register sweep visits only these slots
    // (a slot outside it holds subtrahends no record passes, so skipping it is exact)
    sweep = swept && ok_pre && rem >= 0 && l_lat > 0 && pc < n && pa < n;
  }
  if (mkey) {
    // the prefix tasks' part of the packed m key; the later-non-empty flag of a task
    // below the sink's id depends on the sink: non-empty (mk) or "no instances" (mkz)
    unsigned long long pk = 0, pkz = 0;
    bool ne = false, nez = false;
    for (int u = T - 1; u >= 0; --u) {
      if (u == tl) {
        ne = true;
        continue;
      }
      const int cu = ch[g.pos_of[u]];
      pk |= x_mk_task(s, probe, u, cu, ne);
      pkz |= x_mk_task(s, probe, u, cu, nez);
      if (cu != NONE16) ne = nez = true;
    }
    ws.mk[slot] = pk;
    ws.mkz[slot] = pkz;
  }
  ws.need[slot] = need;
  ws.sl[slot] = sl_pre;
  ws.flags[slot] = (valid ? X_LEAF : 0) | (ok_pre ? X_OKPRE : 0) | (later ? X_LATER : 0) |
                   (dem[tl] == 0.0 ? X_ZERO : 0) | (sweep ? X_SWEEP : 0);
  ws.q[slot] = qp;
}

// The sink-dependent part of derive + validate for one candidate, in float.
// Returns the conjunction of all verdicts (W, the path-weighted accuracy sum of
// model.py:275-282, is formed up to the sign of zero; feasible leaves redo it).
template <int PM, bool FIN>
__device__ __forceinline__ bool x_sink_eval(const double lat2, const double cap, const double acc,
                                            const int sl, const double need, const int sl_pre,
                                            const bool ok_pre, const double* f, const double* c,
                                            const double* pp, const double* frac, unsigned thru,
                                            int P, double slo, int S, const DProbe& pr,
                                            double a_max) {
  // throughput verdict of the sink (planner.py:345-347); fl(a - b) >= 0 <=> a >= b
  // for finite operands (FIN problems)
  bool ok = ok_pre & (FIN ? (cap >= need) : (cap - need >= 0));
  double W = 0.0;
#pragma unroll
  for (int p = 0; p < PM; ++p) {
    if (p < P) {
      double x;
      if ((thru >> p) & 1u) {
        // one step of CPython 3.12's compensated sum() + its final rounding
        const double t = f[p] + lat2;
        const bool fb = fabs(f[p]) >= fabs(lat2);
        const double big = fb ? f[p] : lat2, small = fb ? lat2 : f[p];
        const double cc = c[p] + ((big - t) + small);
        const double tot_lat = (cc != 0.0 && fabs(cc) < INFINITY) ? t + cc : t;
        ok &= (slo - tot_lat >= 0);  // latency verdict (planner.py:339-343)
        x = frac[p] * (pp[p] * acc);
      } else {
        x = f[p];  // frac * product of a path that avoids the sink
      }
      W = (p == 0) ? x : W + x;
    }
  }
  ok &= (S - (sl_pre + sl) >= 0);  // resources verdict, float(S - total) >= 0
  ok &= x_acc_ok(W, pr, a_max);
  return ok;
}

// Fold one feasible leaf of the current prefix into the lane's prefix best.
template <int PM>
__device__ __forceinline__ bool x_take(const XArgs& a, int probe, int tl, long long qp, long long R,
                                       int b, double acc, int sl_pre, int sl, const double* f,
                                       const double* pp, const double* frac, unsigned thru, int P,
                                       double alpha, double beta, double a_max, bool later,
                                       unsigned long long pk, int bc, XBest& rb) {
  // exact W, a_obj and objective in the reference order (model.py:275-293, planner.py:313)
  double Wx = 0.0;
#pragma unroll
  for (int p = 0; p < PM; ++p)
    if (p < P) Wx += ((thru >> p) & 1u) ? frac[p] * (pp[p] * acc) : f[p];
  XBest cb;
  cb.has = 1;
  cb.sl = sl_pre + sl;
  cb.obj = alpha * (Wx / a_max) - beta * (double)cb.sl;
  cb.idx = qp * R + b;
  // (the packed m key -- a dependent global load -- only when it decides a tie or
  // the candidate is taken: most feasible leaves lose on the objective)
  cb.mk = 0ull;
  bool take, have_mk = false;
  if (!rb.has || a.mode != LEAF_FULL) take = !rb.has;
  else if (cb.obj != rb.obj) take = cb.obj > rb.obj;
  else if (cb.sl != rb.sl) take = cb.sl < rb.sl;
  else if (a.mkey) {
    cb.mk = pk | x_mk_task(a.s, probe, tl, bc, later);
    have_mk = true;
    take = cb.mk < rb.mk;
  } else take = x_sink_cmp(a.s, probe, tl, b, (int)(rb.idx - qp * R), later) < 0;
  if (take) {
    if (a.mkey && !have_mk) cb.mk = pk | x_mk_task(a.s, probe, tl, bc, later);
    rb = cb;
  }
  return a.mode != LEAF_FULL;  // feasible-only: first feasible of this lane (b ascending)
}

// ------------------------------------------------------------------ kernel

constexpr int XU = 4;  // candidates per lane and iteration in rank space (independent chains)

// Block-invariant context of the rare feasible path of the register sweep.
template <int PM>
struct XCtx {
  const XArgs* a;
  const XProbe* xp;
  int probe, tl, P;
  long long q, R;
  double slo, a_max, alpha, beta;
  unsigned thru;
  double frac[PM];
};

// Register sweep, feasible records of prefix slot j: `mask` bit k = record
// lane + 32 k passed the four rank compares.  Exact latency step where t is
// within the margin, then the exact objective and the (obj, slices, m) fold
// (kept out of line: ~2% of the (lane, prefix) pairs reach it).
template <int PM, int NS>
__device__ __noinline__ void x_slow_reg(const XCtx<PM>& cx, const XWarpState<PM, NS>& ws, int j,
                                        unsigned mask, XBest& best) {
  const XArgs& a = *cx.a;
  const S2Args& s = a.s;
  const int lane = threadIdx.x & 31;
  const long long qp = ws.q[j];
  const int sl_pre = ws.sl[j];
  const bool later = (ws.flags[j] & 4) != 0;
  double f[PM], c[PM], pp[PM], lo[PM];
#pragma unroll
  for (int p = 0; p < PM; ++p) {
    f[p] = ws.s0[p][j];
    c[p] = ws.s1[p][j];
    pp[p] = ws.s2[p][j];
    lo[p] = ws.lo[p][j];
  }
  XBest rb;
  rb = x_none();
  while (mask) {
    const int k = __ffs(mask) - 1;
    mask &= mask - 1;
    const int b = lane + 32 * k;
    const double lat2 = 2.0 * s.p_lat[cx.q + b];
    // t within the margin of the SLO: CPython 3.12 sum() step exactly
    bool lat_ok = true;
#pragma unroll
    for (int p = 0; p < PM; ++p) {
      if ((cx.thru >> p) & 1u) {
        const double t = f[p] + lat2;
        if (t <= lo[p]) continue;
        const bool fb = fabs(f[p]) >= fabs(lat2);
        const double big = fb ? f[p] : lat2, small = fb ? lat2 : f[p];
        const double cc = c[p] + ((big - t) + small);
        lat_ok &= (t + cc <= cx.slo);  // c finite and +0 when zero (RANK problems)
      }
    }
    if (!lat_ok) continue;
    if (x_take<PM>(a, cx.probe, cx.tl, qp, cx.R, b, s.p_acc[cx.q + b], sl_pre, (int)s.p_sl[cx.q + b],
                   f, pp, cx.frac, cx.thru, cx.P, cx.alpha, cx.beta, cx.a_max, later, ws.mk[j], b, rb))
      break;
  }
  if (rb.has && x_better(a, *cx.xp, cx.probe, rb, best)) best = rb;
}

// Register sweep, prefixes whose sink demand is 0 (bit j of zmask): the only
// child is "no instances" (planner.py:868-875); lane 0 derives each leaf.
template <int PM, int NS>
__device__ __noinline__ unsigned x_zero_reg(const XCtx<PM>& cx, const DProbe& pr, int S,
                                            const XWarpState<PM, NS>& ws, unsigned zmask,
                                            XBest& best) {
  const XArgs& a = *cx.a;
  unsigned n = 0;
  while (zmask) {
    const int j = __ffs(zmask) - 1;
    zmask &= zmask - 1;
    ++n;
    double f[PM], c[PM], pp[PM];
#pragma unroll
    for (int p = 0; p < PM; ++p) {
      f[p] = ws.s0[p][j];
      c[p] = ws.s1[p][j];
      pp[p] = ws.s2[p][j];
    }
    const int fl = ws.flags[j];
    XBest rb;
    rb = x_none();
    if (x_sink_eval<PM, true>(0.0, 0.0, 1.0, 0, ws.need[j], ws.sl[j], (fl & 2) != 0, f, c, pp,
                              cx.frac, cx.thru, cx.P, cx.slo, S, pr, cx.a_max))
      x_take<PM>(a, cx.probe, cx.tl, ws.q[j], cx.R, cx.xp->pn[a.s.T - 1], 1.0, ws.sl[j], 0, f, pp,
                 cx.frac, cx.thru, cx.P, cx.alpha, cx.beta, cx.a_max, (fl & 4) != 0, ws.mkz[j], NONE16,
                 rb);
    if (rb.has && x_better(a, *cx.xp, cx.probe, rb, best)) best = rb;
  }
  return n;
}

#define X_H 0x80008000u
// guard bits of record r against SWAR subtrahends B: X_H iff all four verdicts pass
#define X_V(r, B) (((r).x - (B).x) & ((r).y - (B).y) & X_H)

// Register sweep of one round: every lane keeps records lane + 32 k (k < K =
// ceil(pool / 32), the probe's count) of the sink pool in registers and tests
// them against each leaf prefix of the warp (bit j of vmask), two prefixes per
// iteration (independent max chains).  Per candidate: two IADD (often issued as
// IMAD.IADD on the FMA pipe), one LOP3 and half a three-input VIMNMX.
template <int PM, int NS, int K>
__device__ __forceinline__ void x_sweep_k(const XCtx<PM>& cx, const uint2* __restrict__ pack,
                                          int pn, const XWarpState<PM, NS>& ws, unsigned vmask,
                                          XBest& best) {
  const int lane = threadIdx.x & 31;
  uint2 rec[K];
  // records past the pool fail every threshold (rank(2L) field 0x7FFF never passes)
#pragma unroll
  for (int k = 0; k < K; ++k)
    rec[k] = (lane + 32 * k < pn) ? pack[lane + 32 * k] : make_uint2(0x80008000u, 0x80008000u);
  // the set bits of vmask two at a time (two independent max chains); an odd
  // last slot is paired with subtrahends no record passes
  unsigned vm = vmask;
#pragma unroll 1
  while (vm) {  // warp-uniform
    const int j0 = __ffs(vm) - 1;
    vm &= vm - 1;
    const int j1 = vm ? __ffs(vm) - 1 : -1;
    if (vm) vm &= vm - 1;
    const uint2 b0 = ws.sw[j0];
    const uint2 b1 = j1 >= 0 ? ws.sw[j1] : make_uint2(0u, 0x80000000u);
    unsigned m0 = 0u, m1 = 0u;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      m0 = max(m0, X_V(rec[k], b0));
      m1 = max(m1, X_V(rec[k], b1));
    }
    if (m0 == X_H) {
      unsigned mask = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) mask |= (X_V(rec[k], b0) == X_H ? 1u : 0u) << k;
      x_slow_reg<PM, NS>(cx, ws, j0, mask, best);
    }
    if (m1 == X_H) {
      unsigned mask = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) mask |= (X_V(rec[k], b1) == X_H ? 1u : 0u) << k;
      x_slow_reg<PM, NS>(cx, ws, j1, mask, best);
    }
  }
}

template <int PM, int NS>
__device__ __forceinline__ void x_sweep_reg(const XCtx<PM>& cx, const uint2* __restrict__ pack,
                                            int pn, const XWarpState<PM, NS>& ws, unsigned vmask,
                                            int rpl, XBest& best) {
  switch (rpl) {
#define JSV_XSW(K) \
  case K: x_sweep_k<PM, NS, K>(cx, pack, pn, ws, vmask, best); break;
    JSV_XSW(1) JSV_XSW(2) JSV_XSW(3) JSV_XSW(4) JSV_XSW(5) JSV_XSW(6) JSV_XSW(7) JSV_XSW(8)
    JSV_XSW(9) JSV_XSW(10) JSV_XSW(11) JSV_XSW(12) JSV_XSW(13) JSV_XSW(14) JSV_XSW(15) JSV_XSW(16)
#undef JSV_XSW
    default: break;
  }
}

// Persistent warps: every warp takes rounds -- x_slots(P) consecutive entries of
// one probe's live list (k_x_live), the concatenation ordered by probe (round
// offsets from k_x_sched) -- one at a time from a counter, derives the round's
// prefixes (one per lane) and sweeps the probe's sink pool for them, and writes
// its best of the round into part slot `round` (k_s2_xreduce folds them per
// probe).  No block barriers: the sink pool's rank records and sorted columns
// are read through L1 (a few KB per probe, shared by every warp on the SM).
template <int PM, bool RANK, bool REG>
__global__ void __launch_bounds__(XBLOCK, (RANK && REG) ? JSV_XMINB : 1)
    k_s2_exh(const __grid_constant__ XArgs a) {
  constexpr int NS = x_slots(PM);
  using WS = XWarpState<PM, NS>;
  extern __shared__ __align__(16) unsigned char x_smem[];
  __shared__ __align__(16) DGraph s_g;  // the graph, read by every prefix derivation
  const S2Args& s = a.s;
  {
    const int2* src = reinterpret_cast<const int2*>(s.g);
    int2* dst = reinterpret_cast<int2*>(&s_g);
    for (int i = threadIdx.x; i < (int)(sizeof(DGraph) / 8); i += blockDim.x) dst[i] = src[i];
    static_assert(sizeof(DGraph) % 8 == 0, "DGraph copy granularity");
  }
  __syncthreads();
  const DGraph& g = s_g;
  const int T = s.T, P = g.P;
  const int tl = g.topo[T - 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WS& ws = reinterpret_cast<WS*>(x_smem)[wid];
  double frac[PM];
  unsigned thru = 0;
#pragma unroll
  for (int p = 0; p < PM; ++p) {
    frac[p] = (p < P) ? g.path_frac[p] : 0.0;
    if (p < P && ((g.path_mask[p] >> tl) & 1u)) thru |= 1u << p;
  }
  const int S = s.rq->S;
  volatile int* found = s.active;
  const int n_probes = s.n_probes;
  const long long n_rounds = a.roff[n_probes];

  while (true) {
    long long rd = 0;
    if (lane == 0) rd = (long long)atomicAdd(a.work, 1ull);
    rd = __shfl_sync(0xffffffffu, rd, 0);
    if (rd >= n_rounds) break;
    const int probe = find_probe(a.roff, n_probes, rd);
    const XProbe& xp = a.xp[probe];
    const DProbe& pr = s.probes[probe];
    const int pn = xp.pn[T - 1];
    const long long q = (long long)(probe * T + tl) * s.W;
    const long long o = (long long)probe * s.W;
    XRankView rv;
    rv.n = pn;
    if (RANK) {
      rv.rank = a.xrank + o; rv.pack = a.xpack + o;
      rv.scap = a.scap + o; rv.sacc = a.sacc + o; rv.slat2 = a.slat2 + o;
    }
    XBest best;
    best = x_none();
    unsigned nswept = 0;     // register sweep: prefixes whose sink pool the warp swept
    unsigned long long swept = 0;
    if (!(a.mode == LEAF_ANY && __shfl_sync(0xffffffffu, lane == 0 ? found[probe] : 0, 0))) {
      const int glog = xp.glog, G = 1 << glog;
      const int gw = 32 >> glog;  // prefix groups per warp
      const int gi = lane >> glog, lane_g = lane & (G - 1);
      const double slo = pr.slo_eff, a_max = g.a_max;
      const double alpha = pr.alpha, beta = pr.beta;
      const long long R = xp.R;
      XCtx<PM> cx;
      if (REG) {
        cx.a = &a; cx.xp = &xp; cx.probe = probe; cx.tl = tl; cx.P = P; cx.q = q; cx.R = R;
        cx.slo = slo; cx.a_max = a_max; cx.alpha = alpha; cx.beta = beta; cx.thru = thru;
#pragma unroll
        for (int p = 0; p < PM; ++p) cx.frac[p] = frac[p];
      }
      // ---- one live prefix per lane -> the warp state in shared memory
      // (a round is a.round prefixes <= NS: small batches use short rounds so their few
      // live prefixes spread over more warps)
      if (lane < NS) {
        const long long qi = (rd - a.roff[probe]) * a.round + lane;
        if (lane < a.round && qi < a.live_cnt[probe])
          x_prefix<PM, NS, RANK>(s, g, xp, pr, probe, xp.q0 + a.live[xp.loff + qi], frac, thru,
                                 lane, a.lat2_max, rv, ws, a.mkey);
        else {
          ws.flags[lane] = 0;
          if (RANK) ws.sw[lane] = make_uint2(0u, 0x80000000u);  // fails every record
        }
      }
      __syncwarp();
      if constexpr (RANK && REG && NS == 32) {
        // NS == 32 here: lane j derived prefix j
        const int myfl = ws.flags[lane];
        const unsigned vmask = __ballot_sync(0xffffffffu, (myfl & X_SWEEP) != 0);
        const unsigned zmask =
            __ballot_sync(0xffffffffu, (myfl & (X_LEAF | X_ZERO)) == (X_LEAF | X_ZERO));
        nswept = (unsigned)__popc(vmask);
        x_sweep_reg<PM, NS>(cx, rv.pack, pn, ws, vmask, xp.rpl, best);
        // sink demand 0: the only child is "no instances" (planner.py:868-875)
        if (zmask && lane == 0) x_zero_reg<PM, NS>(cx, pr, S, ws, zmask, best);
      } else {
        // ---- groups of G lanes sweep the sink pool for each prefix
        for (int j = gi; j < NS; j += gw) {
          const int fl = ws.flags[j];
          if (!(fl & X_LEAF)) continue;  // not a leaf prefix (group-uniform)
          const long long qp = ws.q[j];
          const double need = ws.need[j];
          const int sl_pre = ws.sl[j];
          const bool ok_pre = (fl & X_OKPRE) != 0, later = (fl & X_LATER) != 0;
          double f[PM], c[PM], pp[PM];
#pragma unroll
          for (int p = 0; p < PM; ++p) {
            f[p] = ws.s0[p][j];
            c[p] = ws.s1[p][j];
            pp[p] = ws.s2[p][j];
          }
          XBest rb;
          rb = x_none();
          if (fl & X_ZERO) {
            // sink demand 0: its only child is "no instances" (planner.py:868-875)
            if (lane_g == 0) {
              if (x_sink_eval<PM, RANK>(0.0, 0.0, 1.0, 0, need, sl_pre, ok_pre, f, c, pp, frac, thru,
                                        P, slo, S, pr, a_max))
                x_take<PM>(a, probe, tl, qp, R, pn, 1.0, sl_pre, 0, f, pp, frac, thru, P, alpha, beta,
                           a_max, later, ws.mkz[j], NONE16, rb);
            }
          } else if (RANK && !(fl & X_SWEEP)) {
            // no record passes every threshold: all children fail (decided)
          } else if (RANK) {
            if (lane_g < pn) swept += (unsigned)((pn - lane_g + G - 1) >> glog);
            const uint4 th = ws.th[j];
            const unsigned a_cap = th.x, a_acc = th.y, l_lat = th.z, rem = th.w;
            double lo[PM];
#pragma unroll
            for (int p = 0; p < PM; ++p) lo[p] = ws.lo[p][j];
            // every verdict of every candidate: four integer compares on its record
            for (int b0 = lane_g; b0 < pn; b0 += XU * G) {
              bool ok[XU], any = false;
              unsigned slv[XU];
#pragma unroll
              for (int u = 0; u < XU; ++u) {
                const int b = b0 + u * G;
                const uint4 r = b < pn ? rv.rank[b] : make_uint4(0u, 0u, 0xFFFFFFFFu, 0xFFFFFFFFu);
                ok[u] = (r.x >= a_cap) & (r.y >= a_acc) & (r.z < l_lat) & (r.w <= rem);
                slv[u] = r.w;
                any |= ok[u];
              }
              if (!any) continue;
              bool stop = false;
#pragma unroll
              for (int u = 0; u < XU; ++u) {
                if (stop || !ok[u]) continue;
                const int b = b0 + u * G;
                const double lat2 = 2.0 * s.p_lat[q + b];
                // t within the margin of the SLO: CPython 3.12 sum() step exactly
                bool lat_ok = true;
#pragma unroll
                for (int p = 0; p < PM; ++p) {
                  if ((thru >> p) & 1u) {
                    const double t = f[p] + lat2;
                    if (t <= lo[p]) continue;
                    const bool fb = fabs(f[p]) >= fabs(lat2);
                    const double big = fb ? f[p] : lat2, small = fb ? lat2 : f[p];
                    const double cc = c[p] + ((big - t) + small);
                    lat_ok &= (t + cc <= slo);  // c finite and +0 when zero (RANK problems)
                  }
                }
                if (!lat_ok) continue;
                stop = x_take<PM>(a, probe, tl, qp, R, b, s.p_acc[q + b], sl_pre, (int)slv[u], f, pp,
                                  frac, thru, P, alpha, beta, a_max, later, ws.mk[j], b, rb);
              }
              if (stop) break;
            }
          } else if (!ok_pre) {
            // a prefix verdict failed: every child fails (decided)
          } else {
            if (lane_g < pn) swept += (unsigned)((pn - lane_g + G - 1) >> glog);
            for (int b = lane_g; b < pn; b += G) {
              const double lat2 = 2.0 * s.p_lat[q + b], cap = s.p_cap[q + b], acc = s.p_acc[q + b];
              const int sl = s.p_sl[q + b];
              if (!x_sink_eval<PM, false>(lat2, cap, acc, sl, need, sl_pre, ok_pre, f, c, pp, frac,
                                          thru, P, slo, S, pr, a_max))
                continue;
              if (x_take<PM>(a, probe, tl, qp, R, b, acc, sl_pre, sl, f, pp, frac, thru, P, alpha,
                             beta, a_max, later, ws.mk[j], b, rb))
                break;
            }
          }
          if (rb.has && x_better(a, xp, probe, rb, best)) best = rb;
        }
      }
      __syncwarp();
      if (RANK && REG && lane < pn) swept += (unsigned long long)nswept * ((pn - lane + 31) >> 5);
    }
    // the warp's best of the round -> part slot rd
    if (a.mode == LEAF_ANY && best.has) found[probe] = 1;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const XBest ob = x_shfl_down(best, d);
      if (x_better(a, xp, probe, ob, best)) best = ob;
      swept += __shfl_down_sync(0xffffffffu, swept, d);
    }
    if (lane == 0) {
      XPart& op = a.part[rd];
      op.has = best.has; op.sl = best.sl; op.obj = best.obj; op.idx = best.idx; op.mk = best.mk;
      op.leaves = 0;
      op.swept = swept;
    }
  }
}

// Live prefixes of every exhaustive probe.  Work unit: one *upper prefix* (every
// prefix digit but the fastest, position T - 2) of one probe, one warp each.  The
// upper part of the derivation -- digits, demand propagation up to task
// t = topo[T - 2], whose demand depends only on earlier positions, and the
// throughput verdicts of the upper tasks (planner.py:345-347, model.py:239-264)
// -- is computed once per warp; the lanes then run over t's digit d: its
// validity ("no instances" exactly where demand is 0), its throughput verdict
// and the sink's demand (the leaf count: 1 child when it is 0, the whole sink
// pool otherwise).  A prefix failing a throughput verdict fails for every sink
// child -- the reference's _visit kills it at that task (planner.py:876-881) --
// so it is decided here; the others (every leaf prefix when pruning is off) are
// appended to the probe's live list for the full derivation + sweep (k_s2_exh).
// BestRec.leaves ends equal to the probe's whole cross-product of leaves.
__global__ void __launch_bounds__(256, 3) k_x_live(const __grid_constant__ XArgs a, long long total_arg) {
  __shared__ __align__(16) DGraph s_g;
  const S2Args& s = a.s;
  {
    const int2* src = reinterpret_cast<const int2*>(s.g);
    int2* dst = reinterpret_cast<int2*>(&s_g);
    for (int i = threadIdx.x; i < (int)(sizeof(DGraph) / 8); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const DGraph& g = s_g;
  const DReq& rq = *s.rq;
  const int T = s.T, tl = g.topo[T - 1];
  const int lane = threadIdx.x & 31;
  const long long n_warps = (long long)gridDim.x * (blockDim.x >> 5);
  const double sf = 1.0 + rq.slack;
  // (device-planned batches: the number of upper prefixes comes from k_x_plan)
  const long long total = a.dev_totals ? a.dev_totals[0] : total_arg;
  for (long long wu = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); wu < total;
       wu += n_warps) {
    const int probe = find_probe(a.uoff, s.n_probes, wu);
    const XProbe& xp = a.xp[probe];
    const DProbe& pr = s.probes[probe];
    const int jb = probe * T;
    const long long Rl = T >= 2 ? xp.radix[T - 2] : 1;
    const long long u = xp.q0 / Rl + (wu - a.uoff[probe]);
    const long long dlo = max(0LL, xp.q0 - u * Rl), dhi = min(Rl, xp.q0 + xp.nq - u * Rl);
    // ---- upper digits (positions 0 .. T-3) and demand up to topo[T - 2]
    uint16_t ch[MAXT];
    double dem[MAXT];
    {
      unsigned long long v = (unsigned long long)u;
      for (int k = T - 3; k >= 0; --k) {
        const unsigned r = (unsigned)xp.radix[k];
        const unsigned dd = (unsigned)(v % r);
        v /= r;
        ch[k] = (dd == (unsigned)xp.pn[k]) ? (uint16_t)NONE16 : (uint16_t)dd;
      }
    }
    bool valid_up = true, ok_up = true;
    for (int i = 0; i < T - 1; ++i) {
      const int t = g.topo[i];
      double d;
      if (t == g.entry) {
        d = pr.demand;
      } else {
        d = 0.0;
        for (int k = g.pred_off[t]; k < g.pred_off[t + 1]; ++k) {
          const int e = g.pred_edge[k];
          const int src = g.edge_src[e];
          const int cs = ch[g.pos_of[src]];
          double fan;
          if (rq.has_ov[e]) fan = rq.ov[e];
          else if (cs == NONE16) fan = 0.0;
          else fan = s.p_fan[((long long)(jb + src) * s.W + cs) * s.maxout + (e - g.succ_off[src])];
          d += dem[src] * fan;
        }
      }
      dem[t] = d;
      if (i < T - 2) {
        const int c = ch[i];
        if ((c == NONE16) != (d == 0.0)) valid_up = false;
        const double cap = (c == NONE16) ? 0.0 : s.p_cap[(long long)(jb + t) * s.W + c];
        if (!(cap - d * sf >= 0)) ok_up = false;  // planner.py:345-347
      }
    }
    if (!valid_up) continue;  // no leaf below (warp-uniform)
    const int tp = T >= 2 ? g.topo[T - 2] : -1;
    const double dem_t = T >= 2 ? dem[tp] : 0.0;
    const int pn_t = T >= 2 ? xp.pn[T - 2] : 0;
    const unsigned long long pn_s = (unsigned long long)xp.pn[T - 1];
    // the sink's demand (model.py:239-264, predecessors in order) as a function of
    // t's digit: the terms before t's edge summed here (A), t's term per digit, the
    // terms after it (at most XL_AFT, else the generic loop) added in order
    constexpr int XL_AFT = 4;
    double A = 0.0, aft[XL_AFT];
    int n_aft = 0, e_t = -1;
    bool generic = false;
    if (tl == g.entry) {
      A = pr.demand;
    } else {
      for (int k = g.pred_off[tl]; k < g.pred_off[tl + 1]; ++k) {
        const int e = g.pred_edge[k];
        const int src = g.edge_src[e];
        if (src == tp) {
          e_t = e;
          continue;
        }
        const int cs = ch[g.pos_of[src]];
        double fan;
        if (rq.has_ov[e]) fan = rq.ov[e];
        else if (cs == NONE16) fan = 0.0;
        else fan = s.p_fan[((long long)(jb + src) * s.W + cs) * s.maxout + (e - g.succ_off[src])];
        const double term = dem[src] * fan;
        if (e_t < 0) A += term;
        else if (n_aft < XL_AFT) aft[n_aft++] = term;
        else generic = true;
      }
    }
    const bool t_ov = e_t >= 0 && rq.has_ov[e_t];
    const double ov_t = t_ov ? rq.ov[e_t] : 0.0;
    const double* fan_t = e_t >= 0 ? s.p_fan + (long long)(jb + tp) * s.W * s.maxout + (e_t - g.succ_off[tp])
                                   : nullptr;
    const double* cap_t = T >= 2 ? s.p_cap + (long long)(jb + tp) * s.W : nullptr;
    unsigned n_valid = 0, n_zero = 0;  // leaf prefixes; those whose sink demand is 0
    const int idlo = (int)dlo, idhi = (int)dhi;  // (digits < 2^15)
    const unsigned ubase = (unsigned)(u * Rl - xp.q0);
    const bool need_fan = e_t >= 0 && !t_ov;
    const bool simple = T >= 2 && !generic && n_aft == 0 && e_t >= 0 && !t_ov;
    const double need_t = dem_t * sf;
    // digits in groups of XL_IT x 32: every load of the group issued first, one
    // live-list reservation per group
    constexpr int XL_IT = 8;
    for (int d0 = idlo; d0 < idhi; d0 += 32 * XL_IT) {
      double capv[XL_IT], fanv[XL_IT];
#pragma unroll
      for (int it = 0; it < XL_IT; ++it) {
        const int d = d0 + it * 32 + lane;
        const bool real = T >= 2 && d < idhi && d != pn_t;  // a pool bundle of t
        capv[it] = real ? cap_t[d] : 0.0;
        fanv[it] = (real && need_fan) ? fan_t[(long long)d * s.maxout] : 0.0;
      }
      unsigned lm[XL_IT];
      if (simple) {
        // t feeds the sink through one fan-out edge, no overrides, nothing after it
#pragma unroll
        for (int it = 0; it < XL_IT; ++it) {
          const int d = d0 + it * 32 + lane;
          const bool none = d == pn_t;
          const bool valid = d < idhi && (none == (dem_t == 0.0));
          const bool thr = (capv[it] - need_t >= 0);  // planner.py:345-347 (cap 0 for none)
          const double ds = A + dem_t * fanv[it];
          n_valid += valid;
          n_zero += valid && ds == 0.0;
          lm[it] = __ballot_sync(0xffffffffu, valid && (!a.prune || (ok_up && thr)));
        }
      } else {
#pragma unroll
      for (int it = 0; it < XL_IT; ++it) {
        const int d = d0 + it * 32 + lane;
        bool valid = d < idhi, thr = true;
        const bool none = T >= 2 && d == pn_t;
        if (T >= 2 && valid) {
          if (none != (dem_t == 0.0)) valid = false;
          thr = (capv[it] - dem_t * sf >= 0);  // planner.py:345-347
        }
        bool live = false;
        if (valid) {
          double ds;
          if (generic) {
            const int c = none ? NONE16 : d;
            ds = 0.0;
            for (int k = g.pred_off[tl]; k < g.pred_off[tl + 1]; ++k) {
              const int e = g.pred_edge[k];
              const int src = g.edge_src[e];
              const int cs = (src == tp) ? c : ch[g.pos_of[src]];
              double fan;
              if (rq.has_ov[e]) fan = rq.ov[e];
              else if (cs == NONE16) fan = 0.0;
              else fan = s.p_fan[((long long)(jb + src) * s.W + cs) * s.maxout + (e - g.succ_off[src])];
              ds += dem[src] * fan;
            }
          } else {
            ds = A;
            if (e_t >= 0) {
              ds += dem_t * (t_ov ? ov_t : fanv[it]);  // ("no instances": fan 0)
              for (int k = 0; k < n_aft; ++k) ds += aft[k];
            }
          }
          ++n_valid;
          n_zero += ds == 0.0;
          live = !a.prune || (ok_up && thr);
        }
        lm[it] = __ballot_sync(0xffffffffu, live);
      }
      }
      int tot = 0;
#pragma unroll
      for (int it = 0; it < XL_IT; ++it) tot += __popc(lm[it]);
      int base = 0;
      if (lane == 0 && tot) base = atomicAdd(&a.live_cnt[probe], tot);
      base = __shfl_sync(0xffffffffu, base, 0);
      unsigned* dst = a.live + xp.loff + base;
#pragma unroll
      for (int it = 0; it < XL_IT; ++it) {
        if ((lm[it] >> lane) & 1u)
          dst[__popc(lm[it] & ((1u << lane) - 1u))] = ubase + (unsigned)(d0 + it * 32 + lane);
        dst += __popc(lm[it]);
      }
    }
    unsigned long long lv = (unsigned long long)n_zero + (unsigned long long)(n_valid - n_zero) * pn_s;
    for (int dd = 16; dd > 0; dd >>= 1) lv += __shfl_down_sync(0xffffffffu, lv, dd);
    if (lane == 0 && lv) atomicAdd(&s.best[probe].leaves, lv);
  }
}

// XProbe of every probe from its Stage-1 pool sizes (one block): the radices
// (pool + "no instances" where demand may be 0), the cross-product (swept when <=
// exh_limit and no task is dead), this shard's prefix block, the feasibility
// truncation, the upper-prefix and live-list offsets (block scans).
__global__ void __launch_bounds__(1024) k_x_plan(const __grid_constant__ XArgs a,
                                                 const __grid_constant__ XPlanArgs pa) {
  typedef cub::BlockScan<long long, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ long long c_up, c_nq, c_cand, c_nx;
  const S2Args& s = a.s;
  const DGraph& g = *s.g;
  const int n = s.n_probes, T = s.T;
  if (threadIdx.x == 0) c_up = c_nq = c_cand = c_nx = 0;
  __syncthreads();
  for (int i0 = 0; i0 < n; i0 += 1024) {
    const int i = i0 + threadIdx.x;
    long long nup = 0, nq = 0, cand = 0;
    XProbe x;
    memset(&x, 0, sizeof(x));
    int handled = 0, trunc = 0;
    if (i < n) {
      const DProbe& pr = s.probes[i];
      unsigned __int128 N = 1;
      bool over = false, dead = false;
      for (int k = 0; k < T; ++k) {
        const int t = g.topo[k];
        x.pn[k] = s.pool_n[i * T + t];
        const int cz = (int)((pr.could_zero >> t) & 1u);
        if (x.pn[k] == 0 && !cz) dead = true;
        x.radix[k] = x.pn[k] + cz;
        if (!over) N *= (unsigned)x.radix[k];
        if (N > (unsigned __int128)pa.exh_limit) over = true;
      }
      if (!dead && !over && N != 0) {
        x.R = x.radix[T - 1];
        const long long Q = (long long)(N / (unsigned)x.R);
        x.q0 = (long long)((__int128)Q * pa.shard_rank / pa.shard_world);
        const long long q1 = (long long)((__int128)Q * (pa.shard_rank + 1) / pa.shard_world);
        x.nq = q1 - x.q0;
        if (pa.fo_budget > 0) {
          const long long cap = max(1LL, pa.fo_budget / x.R);
          if (x.nq > cap) {
            x.nq = cap;
            trunc = 1;
          }
        }
        int glog = 0;
        while ((1 << glog) < x.R && glog < 5) ++glog;
        x.glog = glog;
        x.rounds = 1;
        x.rpl = pa.reg ? (x.pn[T - 1] + 31) / 32 : 0;
        handled = 1;
        nq = x.nq;
        cand = x.nq * x.R;
        if (nq > 0) {
          const long long Rl = T >= 2 ? x.radix[T - 2] : 1;
          nup = (x.q0 + x.nq - 1) / Rl - x.q0 / Rl + 1;
        }
      }
    }
    long long up_off, up_tot, nq_off, nq_tot;
    Scan(tmp).ExclusiveSum(nup, up_off, up_tot);
    __syncthreads();
    Scan(tmp).ExclusiveSum(nq, nq_off, nq_tot);
    if (i < n) {
      x.loff = c_nq + nq_off;
      pa.xp[i] = x;
      pa.handled[i] = handled;
      pa.trunc[i] = trunc;
      pa.uoff[i] = c_up + up_off;
    }
    long long cs = cand;
    for (int d = 16; d > 0; d >>= 1) cs += __shfl_down_sync(0xffffffffu, cs, d);
    const unsigned hb = __ballot_sync(0xffffffffu, handled != 0);
    if ((threadIdx.x & 31) == 0) {
      atomicAdd((unsigned long long*)&c_cand, (unsigned long long)cs);
      atomicAdd((unsigned long long*)&c_nx, (unsigned long long)__popc(hb));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      c_up += up_tot;
      c_nq += nq_tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pa.uoff[n] = c_up;
    pa.totals[0] = c_up;
    pa.totals[1] = c_nq;
    pa.totals[2] = c_cand;
    pa.totals[3] = c_nx;
    if (c_nq > pa.live_cap) atomicExch(pa.err, 4);
  }
}

int launch_x_plan(const XArgs& a, const XPlanArgs& pa, cudaStream_t st) {
  k_x_plan<<<1, 1024, 0, st>>>(a, pa);
  return 1;
}

// Round offsets of the live lists (rounds of x_slots(P) prefixes): roff[i] =
// rounds of probes < i, roff[n] = all rounds.  One block.
__global__ void __launch_bounds__(1024) k_x_sched(const __grid_constant__ XArgs a, int ns) {
  typedef cub::BlockScan<long long, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ long long carry;
  const int n = a.s.n_probes;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int i0 = 0; i0 < n; i0 += 1024) {
    const int i = i0 + threadIdx.x;
    const long long r = (i < n && a.xp[i].rounds) ? ((long long)a.live_cnt[i] + ns - 1) / ns : 0;
    long long off, tot;
    Scan(tmp).ExclusiveSum(r, off, tot);
    if (i < n) a.roff_w[i] = carry + off;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) a.roff_w[n] = carry;
}

// m-order ranks of the pool bundles, one block per job; bundles' item lists are
// u32 entries key << 16 | count in canonical order (word order = tuple order),
// read from shared memory when the pool's lists fit.
//  * XArgs::mkey: S2Args::mkey / mnone -- the rank (number of smaller sequences)
//    of every list L and of every "L + later entry" (L followed by a symbol above
//    every entry), "no instances" being the empty list: a bitonic sort of the
//    2 n + 2 sequences, ranks by binary search for the first equal one;
//  * otherwise S2Args::mrank (x_cmp_m): rank and prefix interval of every list.
#define MR_SMEM_WORDS 4096
__global__ void __launch_bounds__(512) k_m_rank(const __grid_constant__ XArgs a) {
  __shared__ uint32_t s_it[MR_SMEM_WORDS];
  __shared__ int s_n[1024];
  __shared__ int s_ix[2048];
  const S2Args& s = a.s;
  const int job = blockIdx.x;
  const int probe = job / s.T, t = job % s.T;
  if (!a.xp[probe].rounds) return;  // not an exhaustive probe
  const int n = s.pool_n[job];
  const int mi = s.maxi;
  const long long base = (long long)probe * s.C_probe + s.task_base[t];
  const int* pc = s.pool_cand + (long long)job * s.W;
  const bool sm = (long long)n * mi <= MR_SMEM_WORDS && n <= 1023;
  if (sm) {
    for (int b = threadIdx.x; b < n; b += blockDim.x) s_n[b] = s.nitems[base + pc[b]];
    __syncthreads();
    for (int i = threadIdx.x; i < n * mi; i += blockDim.x) {
      const int b = i / mi, k = i % mi;
      // (only the list's own entries: the slot's tail is never written by Stage 1)
      s_it[i] = k < s_n[b] ? s.items[(base + pc[b]) * mi + k] : 0u;
    }
    __syncthreads();
  }
  auto item = [&](int b, int k) -> uint32_t {
    return sm ? s_it[b * mi + k] : s.items[(base + pc[b]) * mi + k];
  };
  auto len = [&](int b) -> int { return b >= n ? 0 : (sm ? s_n[b] : s.nitems[base + pc[b]]); };
  if (a.mkey) {
    // (1) bitonic sort of the lists (distinct: a bundle's position r is its rank);
    // lists of <= 4 entries are packed into two 64-bit words (a missing entry is 0,
    // below every entry key << 16 | count, count >= 1: a proper prefix sorts first)
    __shared__ int s_maxn;
    __shared__ unsigned long long s_k[2048];
    if (threadIdx.x == 0) s_maxn = 0;
    __syncthreads();
    for (int b = threadIdx.x; b < n; b += blockDim.x) atomicMax(&s_maxn, len(b));
    __syncthreads();
    const bool packed = s_maxn <= 4;
    if (packed) {
      for (int b = threadIdx.x; b < n; b += blockDim.x) {
        const int nb = len(b);
        unsigned long long w[4] = {0, 0, 0, 0};
        for (int k = 0; k < nb; ++k) w[k] = item(b, k);
        s_k[2 * b] = (w[0] << 32) | w[1];
        s_k[2 * b + 1] = (w[2] << 32) | w[3];
      }
      __syncthreads();
    }
    auto cmp = [&](int x, int y) -> int {
      if (packed) {
        const unsigned long long x0 = s_k[2 * x], y0 = s_k[2 * y];
        if (x0 != y0) return x0 < y0 ? -1 : 1;
        const unsigned long long x1 = s_k[2 * x + 1], y1 = s_k[2 * y + 1];
        return x1 == y1 ? 0 : (x1 < y1 ? -1 : 1);
      }
      const int nx = len(x), ny = len(y), mm = min(nx, ny);
      for (int k = 0; k < mm; ++k) {
        const uint32_t u = item(x, k), v = item(y, k);
        if (u != v) return u < v ? -1 : 1;
      }
      return nx - ny;
    };
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) s_ix[i] = i < n ? i : -1;
    __syncthreads();
    for (int kk = 2; kk <= n2; kk <<= 1) {
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int h = threadIdx.x; h < (n2 >> 1); h += blockDim.x) {
          const int i = ((h & ~(j - 1)) << 1) | (h & (j - 1)), l = i | j;
          const int x = s_ix[i], y = s_ix[l];
          const bool gt = (x < 0) ? (y >= 0) : (y >= 0 && cmp(x, y) > 0);  // padding last
          if (gt == ((i & kk) == 0)) {
            s_ix[i] = y;
            s_ix[l] = x;
          }
        }
        __syncthreads();
      }
    }
    // (2) ext(position r) = last position whose list extends list(r): the lists with
    // list(r) as a prefix follow it contiguously
    int* s_ext = s_ix + 1024;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      const int b = s_ix[r], nb = len(b);
      int lo = r, hi = n - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1, o = s_ix[mid];
        bool pre = len(o) >= nb;
        for (int k = 0; k < nb && pre; ++k) pre = item(o, k) == item(b, k);
        if (pre) lo = mid;
        else hi = mid - 1;
      }
      s_ext[r] = lo;
    }
    __syncthreads();
    // (3) merged order of every L and "L + later": a depth-first walk of the prefix
    // tree -- L opens at its position, closes (L + later) after its last extension,
    // deeper lists closing first; "no instances" is 0 and 2 n + 1
    // closed(x) = #{c : ext(c) < x}: histogram of ext values, exclusive scan
    int* s_cl = reinterpret_cast<int*>(s_k);  // (the packed keys are no longer needed)
    for (int i = threadIdx.x; i <= n; i += blockDim.x) s_cl[i] = 0;
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x) atomicAdd(&s_cl[s_ext[r] + 1], 1);
    __syncthreads();
    if (threadIdx.x < 32) {
      // warp scan over n + 1 <= 1024 entries
      int carry = 0;
      for (int i0 = 0; i0 <= n; i0 += 32) {
        const int i = i0 + threadIdx.x;
        int v = i <= n ? s_cl[i] : 0;
        for (int d = 1; d < 32; d <<= 1) {
          const int o = __shfl_up_sync(0xffffffffu, v, d);
          if ((int)threadIdx.x >= d) v += o;
        }
        if (i <= n) s_cl[i] = carry + v;
        carry += __shfl_sync(0xffffffffu, v, 31);
      }
    }
    __syncthreads();
    uint32_t* out = const_cast<uint32_t*>(s.mkey) + (long long)job * s.W;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      const int e = s_ext[r];
      // lists closing with r (same ext) that are deeper: extensions of r in (r, e]
      int deeper = 0;
      for (int c = r + 1; c <= e; ++c) deeper += s_ext[c] == e;
      const unsigned k0 = 1u + (unsigned)(r + s_cl[r]);
      const unsigned k1 = 2u + (unsigned)(e + s_cl[e] + deeper);
      out[s_ix[r]] = k0 | (k1 << 16);
    }
    if (threadIdx.x == 0) const_cast<uint32_t*>(s.mnone)[job] = (uint32_t)(2 * n + 1) << 16;
    return;
  }
  uint32_t* out = const_cast<uint32_t*>(s.mrank) + (long long)job * s.W;
  for (int b = threadIdx.x; b < n; b += blockDim.x) {
    const int nb = len(b);
    unsigned rank = 0, pre = 0;
    for (int o = 0; o < n; ++o) {
      if (o == b) continue;
      const int no = len(o), m = min(no, nb);
      int k = 0;
      while (k < m && item(o, k) == item(b, k)) ++k;
      if (k < m) {
        rank += item(o, k) < item(b, k);
      } else if (no < nb) {
        ++rank;  // o's list is a proper prefix of b's: smaller
      } else if (no > nb) {
        ++pre;   // b's list is a proper prefix of o's
      }
    }
    out[b] = rank | ((rank + pre) << 16) | (nb == 0 ? 0x80000000u : 0u);
  }
}

// per-probe fold of the block partials into BestRec (choices by topo position)
__global__ void __launch_bounds__(XBLOCK) k_s2_xreduce(const __grid_constant__ XArgs a) {
  __shared__ XBest s_warp[XBLOCK / 32];
  __shared__ unsigned long long s_leaves;
  const int probe = blockIdx.x;
  // one part slot per round of the probe
  const long long b0 = a.roff[probe], b1 = a.roff[probe + 1];
  if (threadIdx.x == 0) a.s.best[probe].live = (unsigned long long)a.live_cnt[probe];
  if (b0 == b1) return;
  const XProbe& xp = a.xp[probe];
  if (threadIdx.x == 0) s_leaves = 0;
  __syncthreads();
  XBest best;
  best = x_none();
  unsigned long long leaves = 0;
  // LEAF_FULL: first the best (objective, slices) key over the parts -- no m
  // comparisons -- then only the parts holding exactly that key are folded by
  // x_better (m ties).  Usually one part holds it and no m comparison runs.
  // (A NaN objective keeps the plain fold: x_better's order is not total then.)
  unsigned long long swept = 0;
  for (long long i = b0 + threadIdx.x; i < b1; i += blockDim.x) swept += a.part[i].swept;
  for (int d = 16; d > 0; d >>= 1) swept += __shfl_down_sync(0xffffffffu, swept, d);
  if ((threadIdx.x & 31) == 0 && swept) atomicAdd(&a.s.best[probe].nodes, swept);
  bool key_pass = a.mode == LEAF_FULL;
  int kh = 0, ks = 0;
  double ko = 0.0;
  if (key_pass) {
    int nan = 0;
    for (long long i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
      const XPart& p = a.part[i];
      leaves += p.leaves;
      if (!p.has) continue;
      nan |= p.obj != p.obj;
      if (!kh || p.obj > ko || (p.obj == ko && p.sl < ks)) { kh = 1; ko = p.obj; ks = p.sl; }
    }
    for (int d = 16; d > 0; d >>= 1) {
      const int oh = __shfl_down_sync(0xffffffffu, kh, d);
      const double oo = __shfl_down_sync(0xffffffffu, ko, d);
      const int os = __shfl_down_sync(0xffffffffu, ks, d);
      if (oh && (!kh || oo > ko || (oo == ko && os < ks))) { kh = 1; ko = oo; ks = os; }
    }
    nan = __any_sync(0xffffffffu, nan);
    if ((threadIdx.x & 31) == 0) {
      s_warp[threadIdx.x >> 5].has = kh;
      s_warp[threadIdx.x >> 5].obj = ko;
      s_warp[threadIdx.x >> 5].sl = ks;
      s_warp[threadIdx.x >> 5].idx = nan;
    }
    __syncthreads();
    kh = 0;
    int any_nan = 0;
    for (int w = 0; w < XBLOCK / 32; ++w) {
      const XBest& o = s_warp[w];
      any_nan |= (int)o.idx;
      if (o.has && (!kh || o.obj > ko || (o.obj == ko && o.sl < ks))) { kh = 1; ko = o.obj; ks = o.sl; }
    }
    __syncthreads();
    key_pass = !any_nan;
  } else {
    for (long long i = b0 + threadIdx.x; i < b1; i += blockDim.x) leaves += a.part[i].leaves;
  }
  if (!key_pass || kh) {
    for (long long i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
      const XPart& p = a.part[i];
      if (!p.has || (key_pass && (p.obj != ko || p.sl != ks))) continue;
      XBest c;
      c.has = p.has; c.sl = p.sl; c.obj = p.obj; c.idx = p.idx; c.mk = p.mk;
      if (x_better(a, xp, probe, c, best)) best = c;
    }
  }
  for (int d = 16; d > 0; d >>= 1) {
    const XBest o = x_shfl_down(best, d);
    if (x_better(a, xp, probe, o, best)) best = o;
    leaves += __shfl_down_sync(0xffffffffu, leaves, d);
  }
  if ((threadIdx.x & 31) == 0) {
    s_warp[threadIdx.x >> 5] = best;
    atomicAdd(&s_leaves, leaves);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    XBest b = s_warp[0];
    for (int w = 1; w < XBLOCK / 32; ++w)
      if (x_better(a, xp, probe, s_warp[w], b)) b = s_warp[w];
    BestRec* B = a.s.best + probe;
    B->leaves += s_leaves;
    if (b.has) {
      uint16_t ch[MAXT];
      x_digits(xp, a.s.T, b.idx, ch);
      for (int k = 0; k < a.s.T; ++k) B->choice[k] = ch[k];
      B->has = 1;
      B->found = 1;
      B->obj = b.obj;
      B->sl = b.sl;
    }
  }
}

// Rank-space tables of each probe's sink pool: the capacities, accuracies and
// 2 L sorted ascending, and per bundle {rank(cap), rank(acc), rank(2 L), slices}
// where rank(x) = #{pool values < x} (bitonic sort in shared memory, one block
// per probe).  For a verdict "x >= v" that holds on an up-set of the sorted
// values, x passes iff rank(x) >= #{failing values}; for a down-set ("t(x) <=
// hi"), iff rank(x) < #{passing values}.
// keys sorted side by side when their tables fit (one barrier per bitonic
// stage for all three instead of three sorts in a row)
// Rank-space tables of each probe's sink pool: the capacities, accuracies and
// 2 L sorted ascending, and per bundle {rank(cap), rank(acc), rank(2 L), slices}
// where rank(x) = #{pool values < x}.  For a verdict "x >= v" that holds on an
// up-set of the sorted values, x passes iff rank(x) >= #{failing values}; for a
// down-set ("t(x) <= hi"), iff rank(x) < #{passing values}.  One block per
// (probe, column): a bitonic sort of the column in shared memory (one
// compare-exchange per thread and stage); the probe's last block to finish also
// writes the SWAR records.
__global__ void __launch_bounds__(512) k_x_rank(const __grid_constant__ XArgs a, int n2) {
  extern __shared__ __align__(16) unsigned char k_smem[];
  __shared__ int s_last;
  double* v = reinterpret_cast<double*>(k_smem);  // [n2]
  int* ix = reinterpret_cast<int*>(v + n2);       // [n2]
  const int probe = blockIdx.x, key = blockIdx.y;
  const XProbe& xp = a.xp[probe];
  if (xp.rounds == 0) return;  // not an exhaustive probe
  const S2Args& s = a.s;
  const int T = s.T;
  const int tl = s.g->topo[T - 1];
  const int n = xp.pn[T - 1];
  const long long q = (long long)(probe * T + tl) * s.W;
  const long long o = (long long)probe * s.W;
  unsigned* rk = reinterpret_cast<unsigned*>(a.xrank + o);
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    double x = INFINITY;
    if (i < n) x = key == 0 ? s.p_cap[q + i] : key == 1 ? s.p_acc[q + i] : 2.0 * s.p_lat[q + i];
    v[i] = x;
    ix[i] = i;
  }
  __syncthreads();
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int h = threadIdx.x; h < (n2 >> 1); h += blockDim.x) {
        const int i = ((h & ~(j - 1)) << 1) | (h & (j - 1)), l = i | j;
        const bool up = (i & k) == 0;
        const double x = v[i], y = v[l];
        if ((x > y) == up) {
          v[i] = y; v[l] = x;
          const int tt = ix[i]; ix[i] = ix[l]; ix[l] = tt;
        }
      }
      __syncthreads();
    }
  }
  double* out = key == 0 ? a.scap : key == 1 ? a.sacc : a.slat2;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = v[i];
    out[o + i] = x;
    const int r = x_first(i, [&](int k) { return v[k] >= x; });  // #{values < x} (sorted)
    rk[4 * ix[i] + key] = (unsigned)r;
  }
  if (key == 0)
    for (int i = threadIdx.x; i < n; i += blockDim.x) rk[4 * i + 3] = (unsigned)s.p_sl[q + i];
  // the probe's last column block writes the SWAR records
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&a.xr_done[probe], 1) == 2;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // (used when every field fits 15 bits: pool <= 32767, slices <= 32767)
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint4 r = __ldcg(a.xrank + o + i);  // (written by the other column blocks)
    const unsigned sl = r.w < 0x7FFFu ? r.w : 0x7FFFu;
    a.xpack[o + i] = make_uint2(0x80008000u | (r.x << 16) | r.y,
                                0x80008000u | ((0x7FFFu - r.z) << 16) | (0x7FFFu - sl));
  }
}

size_t x_smem_bytes(int max_pn_last, int P, bool rank) {
  (void)max_pn_last;
  (void)rank;
  size_t ws;
  if (P <= 1) ws = sizeof(XWarpState<1, x_slots(1)>);
  else if (P <= 2) ws = sizeof(XWarpState<2, x_slots(2)>);
  else if (P <= 4) ws = sizeof(XWarpState<4, x_slots(4)>);
  else if (P <= 8) ws = sizeof(XWarpState<8, x_slots(8)>);
  else if (P <= 16) ws = sizeof(XWarpState<16, x_slots(16)>);
  else ws = sizeof(XWarpState<MAXP, x_slots(MAXP)>);
  return (XBLOCK / 32) * ws;
}

// resident blocks of the kernel instance a launch with these arguments uses
#define JSV_XDISPATCH(MAC)                              \
  do {                                                  \
    if (P <= 1) { JSV_XD(1, MAC); }                     \
    else if (P <= 2) { JSV_XD(2, MAC); }                \
    else if (P <= 4) { JSV_XD(4, MAC); }                \
    else if (P <= 8) { JSV_XDN(8, MAC); }               \
    else if (P <= 16) { JSV_XDN(16, MAC); }             \
    else { JSV_XDN(MAXP, MAC); }                        \
  } while (0)
#define JSV_XD(PMV, MAC)                                \
  if (!a.fast) MAC(PMV, false, false);                  \
  else if (a.rpl) MAC(PMV, true, true);                 \
  else MAC(PMV, true, false)
#define JSV_XDN(PMV, MAC)                               \
  if (a.fast) MAC(PMV, true, false);                    \
  else MAC(PMV, false, false)
#define JSV_XOCC(PMV, F, RP)                                                                  \
  do {                                                                                        \
    if (smem > 40 * 1024)                                                                     \
      jsv_smem_attr((const void*)k_s2_exh<PMV, F, RP>, smem);                                                        \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_s2_exh<PMV, F, RP>, XBLOCK, smem); \
  } while (0)
#define JSV_XLAUNCH(PMV, F, RP)                                                                \
  do {                                                                                        \
    if (smem > 40 * 1024)                                                                     \
      jsv_smem_attr((const void*)k_s2_exh<PMV, F, RP>, smem);                                                        \
    k_s2_exh<PMV, F, RP><<<(unsigned)grid, XBLOCK, smem, st>>>(a);                            \
  } while (0)

long long x_resident_blocks(const XArgs& a, int P, size_t smem) {
  int dev = 0, n_sm = 148, per_sm = 1;
  cudaGetDevice(&dev);
  // the occupancy query costs tens of microseconds of host time on every solve:
  // memoise it per (device, kernel instance, shared memory)
  const int inst = (P <= 1 ? 0 : P <= 2 ? 1 : P <= 4 ? 2 : P <= 8 ? 3 : P <= 16 ? 4 : 5) * 8 +
                   (a.fast ? 4 : 0) + (a.rpl ? 2 : 0);
  const long long key = ((long long)dev << 48) ^ ((long long)inst << 32) ^ (long long)smem;
  static thread_local std::map<long long, long long> memo;
  auto it = memo.find(key);
  if (it != memo.end()) return it->second;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  JSV_XDISPATCH(JSV_XOCC);
  const long long r = (long long)(per_sm > 0 ? per_sm : 1) * n_sm;
  memo[key] = r;
  return r;
}

// rank tables of the sink pools (rank-space probes); issued before the host
// plans the chunk schedule so the two overlap
int launch_x_rank(const XArgs& a, cudaStream_t st) {
  if (!a.fast) return 0;
  int n2 = 1;
  while (n2 < a.max_pn_last) n2 <<= 1;
  const size_t sm2 = (sizeof(double) + sizeof(int)) * n2;
  if (sm2 > 48 * 1024) jsv_smem_attr((const void*)k_x_rank, sm2);
  if (!a.xr_zeroed) cudaMemsetAsync(a.xr_done, 0, sizeof(int) * a.s.n_probes, st);
  PROF_BEGIN_ON(K_S2_XSORT, st);
  k_x_rank<<<dim3(a.s.n_probes, 3), 512, sm2, st>>>(a, n2);
  PROF_END_ON(st);
  return 1;
}

// Stage 2 of the exhaustive probes.  On the side stream: the sink-pool rank tables
// (k_x_rank) and the m-order keys (k_m_rank, full plans); concurrently on the main
// stream: the live lists (k_x_live) and their round offsets (k_x_sched).  Then
// the sweep and the per-probe fold.
int launch_stage2_exhaustive(const XArgs& a, long long grid, int P, size_t smem, cudaStream_t st,
                             cudaStream_t st2, cudaEvent_t fork, cudaEvent_t join,
                             long long n_upper, cudaStream_t st3, cudaEvent_t join2) {
  if (grid <= 0) return 0;
  int launches = 0;
  // (the main stream's chain is issued first: the side stream's launches do not
  // delay the live pass, which is the critical path)
  cudaEventRecord(fork, st);
  PROF_BEGIN(K_X_LIVE);
  if (n_upper != 0) {
    // one warp per upper prefix (n_upper < 0: counted on the device, grid-stride)
    const long long blocks =
        n_upper > 0 ? std::min<long long>((n_upper + 7) / 8, 148LL * 8) : 148LL * 8;
    k_x_live<<<(unsigned)blocks, 256, 0, st>>>(a, n_upper);
    ++launches;
  }
  k_x_sched<<<1, 1024, 0, st>>>(a, a.round);
  PROF_END();
  cudaStreamWaitEvent(st2, fork, 0);
  launches += launch_x_rank(a, st2);
  // (the m keys on a third stream when there is one: the rank tables and the m keys
  // are independent, and the two side kernels in series outlast the live pass)
  const bool third = st3 && join2 && a.mode == LEAF_FULL;
  if (third) cudaStreamWaitEvent(st3, fork, 0);
  if (a.mode == LEAF_FULL) {
    cudaStream_t sm = third ? st3 : st2;
    PROF_BEGIN_ON(K_MRANK, sm);
    k_m_rank<<<a.s.n_probes * a.s.T, 512, 0, sm>>>(a);
    PROF_END_ON(sm);
    ++launches;
  }
  cudaEventRecord(join, st2);
  cudaStreamWaitEvent(st, join, 0);
  if (third) {
    cudaEventRecord(join2, st3);
    cudaStreamWaitEvent(st, join2, 0);
  }
  PROF_BEGIN(K_S2_EXH);
  JSV_XDISPATCH(JSV_XLAUNCH);
  PROF_END();
  PROF_BEGIN(K_S2_XREDUCE);
  k_s2_xreduce<<<a.s.n_probes, XBLOCK, 0, st>>>(a);
  PROF_END();
  return launches + 3;
}
#undef JSV_XDISPATCH
#undef JSV_XD
#undef JSV_XDN
#undef JSV_XOCC
#undef JSV_XLAUNCH
