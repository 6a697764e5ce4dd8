#include <map>
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

// m(candidate i1) vs m(candidate i2) as Python tuple comparison (planner.py:852)
__device__ __noinline__ int x_cmp_m(const S2Args& a, const XProbe& xp, int probe, long long i1,
                              long long i2) {
  uint16_t x[MAXT], y[MAXT];
  x_digits(xp, a.T, i1, x);
  x_digits(xp, a.T, i2, y);
  MCursor cx{&a, probe, x, 0, 0, 0, 0}, cy{&a, probe, y, 0, 0, 0, 0};
  cx.open_task();
  cy.open_task();
  while (true) {
    unsigned long long ex = 0, ey = 0;
    const bool hx = cx.next(ex), hy = cy.next(ey);
    if (!hx || !hy) return hx == hy ? 0 : (hx ? 1 : -1);
    if (ex != ey) return ex < ey ? -1 : 1;
  }
}

// Two leaves of the same prefix differ only in the sink's bundle, so their m
// tuples (planner.py:852) first differ inside the sink's item list; when one
// list is a proper prefix of the other the shorter m continues with the next
// non-empty task (task id > sink: larger) or ends (smaller).
__device__ __forceinline__ int x_sink_cmp(const S2Args& a, int probe, int tl, int b1, int b2,
                                          bool later_nonempty) {
  const long long jq = (long long)(probe * a.T + tl) * a.W;
  const long long base = (long long)probe * a.C_probe + a.task_base[tl];
  const long long c1 = base + a.pool_cand[jq + b1], c2 = base + a.pool_cand[jq + b2];
  const int n1 = a.nitems[c1], n2 = a.nitems[c2];
  const int n = n1 < n2 ? n1 : n2;
  for (int k = 0; k < n; ++k) {
    const uint32_t e1 = a.items[c1 * a.maxi + k], e2 = a.items[c2 * a.maxi + k];
    if (e1 != e2) return e1 < e2 ? -1 : 1;
  }
  if (n1 == n2) return 0;
  const int shorter = (n1 < n2) ? -1 : 1;  // -1: candidate 1 is the prefix
  return later_nonempty ? -shorter : shorter;
}

struct XBest {
  int has, sl;
  double obj;
  long long idx;
};

// is A a better feasible candidate than B?
__device__ __forceinline__ bool x_better(const XArgs& a, const XProbe& xp, int probe,
                                         const XBest& A, const XBest& B) {
  if (!A.has) return false;
  if (!B.has) return true;
  if (a.mode != LEAF_FULL) return A.idx < B.idx;
  if (A.obj != B.obj) return A.obj > B.obj;
  if (A.sl != B.sl) return A.sl < B.sl;
  if (A.idx == B.idx) return false;
  return x_cmp_m(a.s, xp, probe, A.idx, B.idx) < 0;
}

__device__ __forceinline__ XBest x_shfl_down(const XBest& v, int d) {
  XBest o;
  o.has = __shfl_down_sync(0xffffffffu, v.has, d);
  o.sl = __shfl_down_sync(0xffffffffu, v.sl, d);
  o.obj = __shfl_down_sync(0xffffffffu, v.obj, d);
  o.idx = __shfl_down_sync(0xffffffffu, v.idx, d);
  return o;
}

// ------------------------------------------------------------- TMA staging

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  unsigned done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
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
template <int PM, int NS, bool RANK>
__device__ __forceinline__ void x_prefix(const S2Args& s, const DGraph& g, const XProbe& xp,
                                         const DProbe& pr, int probe, long long qp,
                                         const double* frac, unsigned thru, int slot,
                                         double lat2_max, const XRankView& rv,
                                         XWarpState<PM, NS>& ws) {
  const DReq& rq = *s.rq;
  const int T = s.T, P = g.P, tl = g.topo[T - 1], jb = probe * T;
  uint16_t ch[MAXT];
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
  double dem[MAXT];
  bool valid = true, ok_pre = true;
  int sl_pre = 0;
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
      if (!(cap - d * sf >= 0)) ok_pre = false;  // planner.py:345-347
      if (c != NONE16) sl_pre += s.p_sl[(long long)(jb + t) * s.W + c];
    }
  }
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
  }
  ws.need[slot] = need;
  ws.sl[slot] = sl_pre;
  ws.flags[slot] = (valid ? 1 : 0) | (ok_pre ? 2 : 0) | (later ? 4 : 0) | (dem[tl] == 0.0 ? 8 : 0);
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
                                       XBest& rb) {
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
  bool take;
  if (!rb.has || a.mode != LEAF_FULL) take = !rb.has;
  else if (cb.obj != rb.obj) take = cb.obj > rb.obj;
  else if (cb.sl != rb.sl) take = cb.sl < rb.sl;
  else take = x_sink_cmp(a.s, probe, tl, b, (int)(rb.idx - qp * R), later) < 0;
  if (take) rb = cb;
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
  rb.has = 0; rb.sl = 0; rb.obj = 0.0; rb.idx = 0;
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
                   f, pp, cx.frac, cx.thru, cx.P, cx.alpha, cx.beta, cx.a_max, later, rb))
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
    rb.has = 0; rb.sl = 0; rb.obj = 0.0; rb.idx = 0;
    if (x_sink_eval<PM, true>(0.0, 0.0, 1.0, 0, ws.need[j], ws.sl[j], (fl & 2) != 0, f, c, pp,
                              cx.frac, cx.thru, cx.P, cx.slo, S, pr, cx.a_max))
      x_take<PM>(a, cx.probe, cx.tl, ws.q[j], cx.R, cx.xp->pn[a.s.T - 1], 1.0, ws.sl[j], 0, f, pp,
                 cx.frac, cx.thru, cx.P, cx.alpha, cx.beta, cx.a_max, (fl & 4) != 0, rb);
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
                                          const XWarpState<PM, NS>& ws, unsigned vmask,
                                          XBest& best) {
  const int lane = threadIdx.x & 31;
  uint2 rec[K];
#pragma unroll
  for (int k = 0; k < K; ++k) rec[k] = pack[lane + 32 * k];
  // fixed slot pairs (2j, 2j+1): a slot that is not a swept leaf prefix holds
  // subtrahends no record passes, so only pairs with no swept slot are skipped
  static_assert(NS % 2 == 0, "slot pairs");
#pragma unroll 1
  for (int j0 = 0; j0 < NS; j0 += 2) {
    if (!((vmask >> j0) & 3u)) continue;  // warp-uniform
    const int j1 = j0 + 1;
    const uint4 bb = *reinterpret_cast<const uint4*>(&ws.sw[j0]);
    const uint2 b0 = make_uint2(bb.x, bb.y), b1 = make_uint2(bb.z, bb.w);
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
                                            const XWarpState<PM, NS>& ws, unsigned vmask, int rpl,
                                            XBest& best) {
  switch (rpl) {
#define JSV_XSW(K) \
  case K: x_sweep_k<PM, NS, K>(cx, pack, ws, vmask, best); break;
    JSV_XSW(1) JSV_XSW(2) JSV_XSW(3) JSV_XSW(4) JSV_XSW(5) JSV_XSW(6) JSV_XSW(7) JSV_XSW(8)
    JSV_XSW(9) JSV_XSW(10) JSV_XSW(11) JSV_XSW(12) JSV_XSW(13) JSV_XSW(14) JSV_XSW(15) JSV_XSW(16)
#undef JSV_XSW
    default: break;
  }
}

// Persistent blocks (one per resident slot of the SMs) take chunks -- warp-round
// ranges [cstart[o], cstart[o + 1]) of the concatenation of every probe's rounds
// (a round = x_slots(P) consecutive prefixes), sized large-first by the host --
// from a counter.  Per probe segment of a chunk the block stages that probe's
// sink pool into shared memory, its warps take the segment's rounds from a
// shared counter (dynamic balance inside the block), and the block's best of the
// segment is reduced into part slot o + probe.
template <int PM, bool RANK, bool REG>
__global__ void __launch_bounds__(XBLOCK, (RANK && REG) ? 2 : 1)
    k_s2_exh(const __grid_constant__ XArgs a) {
  constexpr int NS = x_slots(PM);
  using WS = XWarpState<PM, NS>;
  extern __shared__ __align__(16) unsigned char x_smem[];
  __shared__ __align__(8) unsigned long long s_bar;
  __shared__ XBest s_warp[XBLOCK / 32];
  __shared__ unsigned long long s_leaves;
  __shared__ long long s_round;  // next round of the segment (warps take rounds dynamically)
  __shared__ __align__(16) DGraph s_g;  // the graph, read by every prefix derivation
  const S2Args& s = a.s;
  {
    const int2* src = reinterpret_cast<const int2*>(s.g);
    int2* dst = reinterpret_cast<int2*>(&s_g);
    for (int i = threadIdx.x; i < (int)(sizeof(DGraph) / 8); i += blockDim.x) dst[i] = src[i];
    static_assert(sizeof(DGraph) % 8 == 0, "DGraph copy granularity");
  }
  if (threadIdx.x == 0) {
    s_leaves = 0;
    if (RANK && a.tma) mbar_init(&s_bar, 1);
  }
  __syncthreads();
  const DGraph& g = s_g;
  const int T = s.T, P = g.P;
  const int tl = g.topo[T - 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int max_np = x_pad(a.max_pn_last);  // shared-memory layout is fixed for the launch
  XRankView rv;
  double2* s_lc = nullptr;  // float: (2 L, capacity)
  double2* s_as = nullptr;  // float: (accuracy, slices)
  unsigned char* tail;
  if (RANK) {
    uint4* s_rank = reinterpret_cast<uint4*>(x_smem);
    double* s_scap = reinterpret_cast<double*>(s_rank + max_np);
    double* s_sacc = s_scap + max_np;
    double* s_slat = s_sacc + max_np;
    uint2* s_pack = reinterpret_cast<uint2*>(s_slat + max_np);
    tail = reinterpret_cast<unsigned char*>(s_pack + max_np);
    rv.rank = s_rank; rv.scap = s_scap; rv.sacc = s_sacc; rv.slat2 = s_slat; rv.pack = s_pack;
  } else {
    s_lc = reinterpret_cast<double2*>(x_smem);
    s_as = s_lc + max_np;
    tail = reinterpret_cast<unsigned char*>(s_as + max_np);
  }
  WS& ws = reinterpret_cast<WS*>(tail)[wid];
  double frac[PM];
  unsigned thru = 0;
#pragma unroll
  for (int p = 0; p < PM; ++p) {
    frac[p] = (p < P) ? g.path_frac[p] : 0.0;
    if (p < P && ((g.path_mask[p] >> tl) & 1u)) thru |= 1u << p;
  }
  const int S = s.rq->S;
  volatile int* found = s.active;
  __shared__ long long s_chunk;
  long long chunk = -1, r_cur = 0, r_end = 0;

  int probe = -1;
  unsigned stage_phase = 0;
  XBest best;
  best.has = 0; best.sl = 0; best.obj = 0.0; best.idx = 0;
  unsigned long long leaves = 0;

  // block reduction of the current probe segment into part slot blockIdx.x + probe
  auto flush = [&]() {
    const XProbe& xp = a.xp[probe];
    if (a.mode == LEAF_ANY && best.has) found[probe] = 1;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const XBest o = x_shfl_down(best, d);
      if (x_better(a, xp, probe, o, best)) best = o;
    }
    for (int d = 16; d > 0; d >>= 1) leaves += __shfl_down_sync(0xffffffffu, leaves, d);
    if (lane == 0) {
      s_warp[wid] = best;
      atomicAdd(&s_leaves, leaves);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      XBest b = s_warp[0];
      for (int w = 1; w < XBLOCK / 32; ++w)
        if (x_better(a, xp, probe, s_warp[w], b)) b = s_warp[w];
      XPart& o = a.part[chunk + probe];
      o.has = b.has; o.sl = b.sl; o.obj = b.obj; o.idx = b.idx; o.leaves = s_leaves;
      s_leaves = 0;
    }
    best.has = 0; best.sl = 0; best.obj = 0.0; best.idx = 0;
    leaves = 0;
  };

  while (true) {
    if (r_cur >= r_end) {
      // next chunk (the previous chunk's last segment ended with a block barrier)
      if (threadIdx.x == 0) s_chunk = (long long)atomicAdd(a.work, 1ull);
      __syncthreads();
      chunk = s_chunk;
      if (chunk >= a.n_chunks) break;
      r_cur = a.cstart[chunk];
      r_end = a.cstart[chunk + 1];
    }
    probe = find_probe(a.roff, s.n_probes, r_cur);
    const long long seg_end = min(r_end, a.roff[probe + 1]);
    {
      // ---- stage the sink task's pool in shared memory (TMA bulk copies + mbarrier)
      const int pn = a.xp[probe].pn[T - 1];
      const int npad = x_pad(pn);
      const long long q = (long long)(probe * T + tl) * s.W;
      rv.n = pn;
      if (RANK) {
        const long long o = (long long)probe * s.W;
        uint4* s_rank = const_cast<uint4*>(rv.rank);
        uint2* s_pack = const_cast<uint2*>(rv.pack);
        double* s_scap = const_cast<double*>(rv.scap);
        double* s_sacc = const_cast<double*>(rv.sacc);
        double* s_slat = const_cast<double*>(rv.slat2);
        if (a.tma && pn > 0) {
          const unsigned b16 = (unsigned)pn * 16u, b8 = (unsigned)((pn * 8 + 15) & ~15);
          if (threadIdx.x == 0) {
            mbar_expect_tx(&s_bar, b16 + 4 * b8);
            bulk_g2s(s_rank, a.xrank + o, b16, &s_bar);
            bulk_g2s(s_pack, a.xpack + o, b8, &s_bar);
            bulk_g2s(s_scap, a.scap + o, b8, &s_bar);
            bulk_g2s(s_sacc, a.sacc + o, b8, &s_bar);
            bulk_g2s(s_slat, a.slat2 + o, b8, &s_bar);
          }
          mbar_wait(&s_bar, stage_phase);
          stage_phase ^= 1u;
        } else {
          for (int i = threadIdx.x; i < pn; i += blockDim.x) {
            s_rank[i] = a.xrank[o + i];
            s_scap[i] = a.scap[o + i];
            s_sacc[i] = a.sacc[o + i];
            s_slat[i] = a.slat2[o + i];
            s_pack[i] = a.xpack[o + i];
          }
        }
        __syncthreads();
        // padding records always fail (rank(2L) = max) so the sweep needs no bound test;
        // written after the copies land (the bulk sizes round up to 16 bytes)
        for (int i = pn + threadIdx.x; i < npad; i += blockDim.x) {
          s_rank[i] = make_uint4(0u, 0u, 0xFFFFFFFFu, 0xFFFFFFFFu);
          s_pack[i] = make_uint2(0x80008000u, 0x80008000u);  // rank(2L) field 0x7FFF fails
        }
      } else {
        for (int i = threadIdx.x; i < pn; i += blockDim.x) {
          s_lc[i] = make_double2(2.0 * s.p_lat[q + i], s.p_cap[q + i]);
          s_as[i] = make_double2(s.p_acc[q + i],
                                 __longlong_as_double((long long)(unsigned)s.p_sl[q + i]));
        }
      }
      if (threadIdx.x == 0) s_round = r_cur;
      __syncthreads();
    }

    const XProbe& xp = a.xp[probe];
    const DProbe& pr = s.probes[probe];
    const int pn = xp.pn[T - 1];
    const long long q = (long long)(probe * T + tl) * s.W;
    const int glog = xp.glog, G = 1 << glog;
    const int gw = 32 >> glog;  // prefix groups per warp
    const int gi = lane >> glog, lane_g = lane & (G - 1);
    const long long r_probe = a.roff[probe];
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
    const int rpl = xp.rpl;
    unsigned nswept = 0;  // register sweeps: leaf prefixes swept by the whole warp

    // rounds of NS prefixes, taken by the warps from the block counter (balance)
    while (true) {
      long long rd = 0;
      if (lane == 0) rd = (long long)atomicAdd((unsigned long long*)&s_round, 1ull);
      rd = __shfl_sync(0xffffffffu, rd, 0);
      if (rd >= seg_end) break;
      const long long qw = (rd - r_probe) * NS;
      if (a.mode == LEAF_ANY && __shfl_sync(0xffffffffu, lane == 0 ? found[probe] : 0, 0)) break;
      // ---- one prefix per lane -> shared memory
      if (lane < NS) {
        const long long qi = qw + lane;
        if (qi < xp.nq)
          x_prefix<PM, NS, RANK>(s, g, xp, pr, probe, xp.q0 + qi, frac, thru, lane, a.lat2_max, rv, ws);
        else {
          ws.flags[lane] = 0;
          if (RANK) ws.sw[lane] = make_uint2(0u, 0x80000000u);  // fails every record
        }
      }
      __syncwarp();
      if constexpr (RANK && REG && NS == 32) {
        // NS == 32 here: lane j derived prefix j
        const int myfl = ws.flags[lane];
        const unsigned vmask = __ballot_sync(0xffffffffu, (myfl & 9) == 1);
        const unsigned zmask = __ballot_sync(0xffffffffu, (myfl & 9) == 9);
        nswept += (unsigned)__popc(vmask);
        x_sweep_reg<PM, NS>(cx, rv.pack, ws, vmask, rpl, best);
        // sink demand 0: the only child is "no instances" (planner.py:868-875)
        if (zmask && lane == 0) leaves += x_zero_reg<PM, NS>(cx, pr, S, ws, zmask, best);
      } else {
      // ---- groups of G lanes sweep the sink pool for each prefix
      for (int j = gi; j < NS; j += gw) {
        const int fl = ws.flags[j];
        if (!(fl & 1)) continue;  // not a leaf prefix (group-uniform)
        // prefix state, read from shared memory
        const long long qp = ws.q[j];
        const double need = ws.need[j];
        const int sl_pre = ws.sl[j];
        const bool ok_pre = (fl & 2) != 0, later = (fl & 4) != 0;
        double f[PM], c[PM], pp[PM];
#pragma unroll
        for (int p = 0; p < PM; ++p) {
          f[p] = ws.s0[p][j];
          c[p] = ws.s1[p][j];
          pp[p] = ws.s2[p][j];
        }
        XBest rb;
        rb.has = 0; rb.sl = 0; rb.obj = 0.0; rb.idx = 0;
        if (fl & 8) {
          // sink demand 0: its only child is "no instances" (planner.py:868-875)
          if (lane_g == 0) {
            ++leaves;
            if (x_sink_eval<PM, RANK>(0.0, 0.0, 1.0, 0, need, sl_pre, ok_pre, f, c, pp, frac, thru,
                                      P, slo, S, pr, a_max))
              x_take<PM>(a, probe, tl, qp, R, pn, 1.0, sl_pre, 0, f, pp, frac, thru, P, alpha, beta,
                         a_max, later, rb);
          }
        } else if (RANK) {
          if (lane_g < pn) leaves += (unsigned)((pn - lane_g + G - 1) >> glog);
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
              const uint4 r = rv.rank[b0 + u * G];
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
                                frac, thru, P, alpha, beta, a_max, later, rb);
            }
            if (stop) break;
          }
        } else {
          if (lane_g < pn) leaves += (unsigned)((pn - lane_g + G - 1) >> glog);
          for (int b = lane_g; b < pn; b += G) {
            const double2 lc = s_lc[b], as = s_as[b];
            const int sl = (int)(unsigned)__double_as_longlong(as.y);
            if (!x_sink_eval<PM, false>(lc.x, lc.y, as.x, sl, need, sl_pre, ok_pre, f, c, pp, frac,
                                        thru, P, slo, S, pr, a_max))
              continue;
            if (x_take<PM>(a, probe, tl, qp, R, b, as.x, sl_pre, sl, f, pp, frac, thru, P, alpha,
                           beta, a_max, later, rb))
              break;
          }
        }
        if (rb.has && x_better(a, xp, probe, rb, best)) best = rb;
      }
      }
      __syncwarp();
    }
    if (RANK && REG && lane < pn) leaves += (unsigned long long)nswept * ((pn - lane + 31) >> 5);
    __syncthreads();  // the segment's rounds are done before its pool / s_round are rewritten
    flush();
    r_cur = seg_end;
  }
}

// per-probe fold of the block partials into BestRec (choices by topo position)
__global__ void __launch_bounds__(XBLOCK) k_s2_xreduce(const __grid_constant__ XArgs a) {
  __shared__ XBest s_warp[XBLOCK / 32];
  __shared__ unsigned long long s_leaves;
  const int probe = blockIdx.x;
  const long long b0 = a.boff[probe], b1 = a.boff[a.s.n_probes + 1 + probe];
  if (b0 == b1) return;
  const XProbe& xp = a.xp[probe];
  if (threadIdx.x == 0) s_leaves = 0;
  __syncthreads();
  XBest best;
  best.has = 0; best.sl = 0; best.obj = 0.0; best.idx = 0;
  unsigned long long leaves = 0;
  // LEAF_FULL: first the best (objective, slices) key over the parts -- no m
  // comparisons -- then only the parts holding exactly that key are folded by
  // x_better (m ties).  Usually one part holds it and no m comparison runs.
  // (A NaN objective keeps the plain fold: x_better's order is not total then.)
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
      c.has = p.has; c.sl = p.sl; c.obj = p.obj; c.idx = p.idx;
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
#define XRANK_PAR_MAX 2048
__device__ __host__ inline int x_rank_keys_per_pass(int n2) { return n2 <= XRANK_PAR_MAX ? 3 : 1; }

__global__ void __launch_bounds__(512) k_x_rank(const __grid_constant__ XArgs a, int n2) {
  extern __shared__ __align__(16) unsigned char k_smem[];
  const int nk = x_rank_keys_per_pass(n2);
  double* v = reinterpret_cast<double*>(k_smem);  // [nk][n2]
  int* ix = reinterpret_cast<int*>(v + nk * n2);  // [nk][n2]
  const int probe = blockIdx.x;
  const XProbe& xp = a.xp[probe];
  if (xp.rounds == 0) return;  // not an exhaustive probe
  const S2Args& s = a.s;
  const int T = s.T;
  const int tl = s.g->topo[T - 1];
  const int n = xp.pn[T - 1];
  const long long q = (long long)(probe * T + tl) * s.W;
  const long long o = (long long)probe * s.W;
  unsigned* rk = reinterpret_cast<unsigned*>(a.xrank + o);
  const int m = nk * n2;
  for (int key0 = 0; key0 < 3; key0 += nk) {
    for (int t = threadIdx.x; t < m; t += blockDim.x) {
      const int key = key0 + t / n2, i = t % n2;
      double x = INFINITY;
      if (i < n) x = key == 0 ? s.p_cap[q + i] : key == 1 ? s.p_acc[q + i] : 2.0 * s.p_lat[q + i];
      v[t] = x;
      ix[t] = i;
    }
    __syncthreads();
    for (int k = 2; k <= n2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = threadIdx.x; t < m; t += blockDim.x) {
          const int i = t & (n2 - 1);  // (n2 is a power of two)
          const int l = i ^ j;
          if (l > i) {
            const int tl2 = t - i + l;
            const bool up = (i & k) == 0;
            const double x = v[t], y = v[tl2];
            if ((x > y) == up) {
              v[t] = y; v[tl2] = x;
              const int tt = ix[t]; ix[t] = ix[tl2]; ix[tl2] = tt;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int t = threadIdx.x; t < nk * n; t += blockDim.x) {
      const int kk = t / n, i = t % n, key = key0 + kk;
      const double* vk = v + kk * n2;
      double* out = key == 0 ? a.scap : key == 1 ? a.sacc : a.slat2;
      const double x = vk[i];
      out[o + i] = x;
      const int r = x_first(n, [&](int k) { return vk[k] >= x; });  // #{values < x}
      rk[4 * ix[kk * n2 + i] + key] = (unsigned)r;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) rk[4 * i + 3] = (unsigned)s.p_sl[q + i];
  __syncthreads();
  // SWAR records (used when every field fits 15 bits: pool <= 32767, slices <= 32767)
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint4 r = a.xrank[o + i];
    const unsigned sl = r.w < 0x7FFFu ? r.w : 0x7FFFu;
    a.xpack[o + i] = make_uint2(0x80008000u | (r.x << 16) | r.y,
                                0x80008000u | ((0x7FFFu - r.z) << 16) | (0x7FFFu - sl));
  }
}

size_t x_smem_bytes(int max_pn_last, int P, bool rank) {
  const size_t n = (size_t)x_pad(max_pn_last);
  size_t ws;
  if (P <= 1) ws = sizeof(XWarpState<1, x_slots(1)>);
  else if (P <= 2) ws = sizeof(XWarpState<2, x_slots(2)>);
  else if (P <= 4) ws = sizeof(XWarpState<4, x_slots(4)>);
  else if (P <= 8) ws = sizeof(XWarpState<8, x_slots(8)>);
  else if (P <= 16) ws = sizeof(XWarpState<16, x_slots(16)>);
  else ws = sizeof(XWarpState<MAXP, x_slots(MAXP)>);
  const size_t per = rank ? (sizeof(uint4) + 3 * sizeof(double) + sizeof(uint2)) : 2 * sizeof(double2);
  return n * per + (XBLOCK / 32) * ws;
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
      cudaFuncSetAttribute(k_s2_exh<PMV, F, RP>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)smem);                                                        \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_s2_exh<PMV, F, RP>, XBLOCK, smem); \
  } while (0)
#define JSV_XLAUNCH(PMV, F, RP)                                                                \
  do {                                                                                        \
    if (smem > 40 * 1024)                                                                     \
      cudaFuncSetAttribute(k_s2_exh<PMV, F, RP>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)smem);                                                        \
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
  const size_t sm2 = (sizeof(double) + sizeof(int)) * n2 * x_rank_keys_per_pass(n2);
  cudaFuncSetAttribute(k_x_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  PROF_BEGIN(K_S2_XSORT);
  k_x_rank<<<a.s.n_probes, 512, sm2, st>>>(a, n2);
  PROF_END();
  return 1;
}

int launch_stage2_exhaustive(const XArgs& a, long long grid, int P, size_t smem,
                             cudaStream_t st, bool rank_done) {
  if (grid <= 0) return 0;
  int launches = 0;
  if (a.fast && !rank_done) {
    int n2 = 1;
    while (n2 < a.max_pn_last) n2 <<= 1;
    const size_t sm2 = (sizeof(double) + sizeof(int)) * n2 * x_rank_keys_per_pass(n2);
    cudaFuncSetAttribute(k_x_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    PROF_BEGIN(K_S2_XSORT);
    k_x_rank<<<a.s.n_probes, 512, sm2, st>>>(a, n2);
    PROF_END();
    ++launches;
  }
  PROF_BEGIN(K_S2_EXH);
  JSV_XDISPATCH(JSV_XLAUNCH);
  PROF_END();
  PROF_BEGIN(K_S2_XREDUCE);
  k_s2_xreduce<<<a.s.n_probes, XBLOCK, 0, st>>>(a);
  PROF_END();
  return launches + 2;
}
#undef JSV_XDISPATCH
#undef JSV_XD
#undef JSV_XDN
#undef JSV_XOCC
#undef JSV_XLAUNCH
