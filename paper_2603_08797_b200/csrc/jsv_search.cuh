// jsv_search.cuh -- level-synchronous branch-and-bound over the Stage-1 pools
// (included by jsv_stage2.cu).
//
// Per level L (task t = topo[L]):
//   k_s2_prefix  one thread per frontier slot: demand reaching t (_demand_at,
//                planner.py:821-833), slices used, the partial path latency and
//                accuracy products of the chosen prefix, and the number of pool
//                bundles that can pass the resource filter (the pool is sorted by
//                slices, so they form a prefix: "budget trimming").  In the
//                diagnostic re-run nothing is trimmed so kill counts are exact.
//   (scan)       exclusive scan of the per-slot widths -> work offsets.
//   k_s2_level   intermediate level: one work item = (slot, bundle); applies the
//                _visit filters (planner.py:876-903) in the reference order and
//                appends survivors to the next frontier.
//   k_s2_leaf    last level: same filters, then derive + validate of every
//                reached leaf (planner.py:835-855) and a per-thread, per-block
//                (shared memory) and per-probe (k_s2_reduce) lexicographic
//                reduction -- lock free.

#define ST_SKIP (-2)
#define ST_PASS (-1)
#define ST_BOUND 5

__device__ __forceinline__ unsigned long long obj_bits(double x) {
  if (x == 0.0) x = 0.0;  // -0.0 -> +0.0
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double bits_obj(unsigned long long b) {
  b = (b >> 63) ? (b & 0x7FFFFFFFFFFFFFFFull) : ~b;
  return __longlong_as_double((long long)b);
}

// largest slot s in [lo, hi) with pfx[s] <= w
__device__ __forceinline__ long long find_slot(const long long* pfx, long long lo, long long hi,
                                               long long w) {
  --hi;
  while (lo < hi) {
    const long long mid = (lo + hi + 1) >> 1;
    if (pfx[mid] <= w) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// ------------------------------------------------------------ prefix state

__global__ void __launch_bounds__(256) k_s2_prefix(const __grid_constant__ S2Args a) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= a.n_slots) return;
  const DGraph& g = *a.g;
  const DReq& rq = *a.rq;
  const int T = a.T, L = a.level, P = g.P;
  const int t = g.topo[L];
  const int probe = find_probe(a.foff, a.n_probes, s);
  const long long local = s - a.foff[probe];
  if (local >= a.fcap[probe] || local >= (long long)a.fcnt[probe]) {
    a.pr_width[s] = 0;
    a.pr_flag[s] = 0;
    return;
  }
  a.pr_probe[s] = probe;
  uint16_t ch[MAXT];
  for (int k = 0; k < L; ++k) ch[k] = a.cur[s * T + k];
  const DProbe& pr = a.probes[probe];
  const int jb = probe * T;
  double r[MAXT];
  int used = 0;
  for (int k = 0; k <= L; ++k) {
    const int u = g.topo[k];
    double ru;
    if (u == g.entry) {
      ru = pr.demand;
    } else {
      ru = 0.0;
      for (int qq = g.pred_off[u]; qq < g.pred_off[u + 1]; ++qq) {
        const int e = g.pred_edge[qq];
        const int src = g.edge_src[e];
        const int cs = ch[g.pos_of[src]];
        if (cs == NONE16 || r[src] == 0.0) continue;  // empty bundles carry no demand
        const double fan = rq.has_ov[e] ? rq.ov[e]
                                        : a.p_fan[((long long)(jb + src) * a.W + cs) * a.maxout +
                                                  (e - g.succ_off[src])];
        ru += r[src] * fan;
      }
    }
    r[u] = ru;
    if (k < L && ch[k] != NONE16) used += a.p_sl[(long long)(jb + u) * a.W + ch[k]];
  }
  const double rt = r[t];
  a.pr_r[s] = rt;
  a.pr_used[s] = used;
  int width, flag;
  if (rt == 0.0) {
    width = 1;  // the empty assignment is the only child (planner.py:868-875)
    flag = 0;
  } else {
    flag = 1;
    const int Pt = a.pool_n[jb + t];
    if (a.diag) {
      width = Pt;
    } else {
      // bundles passing `used + s + future > S + eps` form a prefix of the slices-sorted pool
      const int* psl = a.p_sl + (long long)(jb + t) * a.W;
      const int fut = a.future[probe * (T + 1) + L + 1];
      const double lim = (double)rq.S + rq.eps;
      int lo = 0, hi = Pt;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((double)(used + psl[mid] + fut) > lim) hi = mid;
        else lo = mid + 1;
      }
      width = lo;
    }
  }
  a.pr_width[s] = width;
  a.pr_flag[s] = flag;
  if (a.diag && flag) atomicOr(&a.cur_flag[s], 1);
  if (flag) {
    // partial path sums / products of the chosen prefix (path order, planner.py:805-819,
    // model.py:267-282); tasks after t on a path are descendants, hence still open
    for (int pp = 0; pp < P; ++pp) {
      const bool through = (g.path_mask[pp] >> t) & 1u;
      double lat = 0.0, prod = 1.0;
      for (int k = g.path_off[pp]; k < g.path_off[pp + 1]; ++k) {
        const int u = g.path_task[k];
        if (through && u == t) break;
        const int pu = g.pos_of[u];
        if (pu < L) {
          const int c = ch[pu];
          if (c != NONE16) {
            const long long q = (long long)(jb + u) * a.W + c;
            lat += 2.0 * a.p_lat[q];
            prod *= a.p_acc[q];
          } else {
            lat += 0.0;
            prod *= 1.0;
          }
        } else {
          prod *= a.acc_ub[jb + u];
        }
      }
      a.pr_lat[s * P + pp] = lat;
      a.pr_acc[s * P + pp] = prod;
    }
  }
  atomicAdd(&a.ptot[probe], (unsigned long long)width);
}

// Filters of one (slot, bundle) item.  Returns ST_PASS (child survives; ub set),
// a JSV_BIND_* kill reason, ST_BOUND (objective bound prune) or ST_SKIP.
__device__ __forceinline__ int filter_item(const S2Args& a, int probe, long long s, int b,
                                           bool check_bound, double& ub_out) {
  const DGraph& g = *a.g;
  const DReq& rq = *a.rq;
  const int T = a.T, L = a.level, P = g.P;
  const int t = g.topo[L];
  if (!(a.pr_flag[s] & 1)) return b == 0 ? ST_PASS : ST_SKIP;
  const int jb = probe * T;
  const DProbe& pr = a.probes[probe];
  const long long q = (long long)(jb + t) * a.W + b;
  const double eps = rq.eps;
  const int used = a.pr_used[s];
  const int fut = a.future[probe * (T + 1) + L + 1];
  const int bsl = a.p_sl[q];
  if (a.p_cap[q] + eps < a.pr_r[s] * (1.0 + rq.slack)) return JSV_BIND_THROUGHPUT;
  if ((double)(used + bsl + fut) > (double)rq.S + eps) return JSV_BIND_RESOURCES;
  const double lat2 = 2.0 * a.p_lat[q];
  const double accb = a.p_acc[q];
  for (int pp = 0; pp < P; ++pp) {
    if (!((g.path_mask[pp] >> t) & 1u)) continue;
    double x = a.pr_lat[s * P + pp] + lat2;
    bool after = false;
    for (int k = g.path_off[pp]; k < g.path_off[pp + 1]; ++k) {
      const int u = g.path_task[k];
      if (after) x += a.min_lat2[jb + u];
      if (u == t) after = true;
    }
    if (x > pr.slo_eff + eps) return JSV_BIND_LATENCY;
  }
  double total = 0.0;
  for (int pp = 0; pp < P; ++pp) {
    double A = a.pr_acc[s * P + pp];
    if ((g.path_mask[pp] >> t) & 1u) {
      A *= accb;
      bool after = false;
      for (int k = g.path_off[pp]; k < g.path_off[pp + 1]; ++k) {
        const int u = g.path_task[k];
        if (after) A *= a.acc_ub[jb + u];
        if (u == t) after = true;
      }
    }
    total += g.path_frac[pp] * A;
  }
  const double ub = total / g.a_max;
  if (ub < pr.acc_slo - eps) return JSV_BIND_ACCURACY;
  ub_out = ub;
  if (check_bound) {
    const unsigned long long ib = ((volatile unsigned long long*)a.inc)[probe];
    if (ib) {
      const double obj_ub = pr.alpha * ub - pr.beta * (double)(used + bsl + fut);
      if (obj_ub < bits_obj(ib) - eps) return ST_BOUND;
    }
  }
  return ST_PASS;
}

__global__ void __launch_bounds__(256) k_s2_level(const __grid_constant__ S2Args a) {
  const int T = a.T, L = a.level;
  const long long total = a.pfx[a.n_slots];
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < total; w += stride) {
    const long long s = find_slot(a.pfx, 0, a.n_slots, w);
    const int probe = a.pr_probe[s];
    const int b = (int)(w - a.pfx[s]);
    double ub = 0.0;
    // the objective bound against the probe's incumbent (planner.py:897-903) prunes
    // internal levels too once a leaf has set one (depth-first frontier chunks do early)
    const int st = filter_item(a, probe, s, b, a.mode == LEAF_FULL && !a.diag, ub);
    if (st == ST_SKIP) continue;
    const bool rpos = a.pr_flag[s] & 1;
    if (a.diag && rpos) {
      if (st >= 0 && st < 5) atomicAdd(&a.best[probe].kills[L][st], 1);
      else atomicOr(&a.cur_flag[s], 2);
    }
    if (st != ST_PASS) continue;
    const unsigned long long pos = atomicAdd(&a.nxt_cnt[probe], 1ull);
    if ((long long)pos >= a.nxt_cap[probe]) {
      atomicExch(a.err, 3);
      continue;
    }
    if (a.nxt_key) {
      const DProbe& pr = a.probes[probe];
      const int used = a.pr_used[s] + (rpos ? a.p_sl[(long long)(probe * T + a.g->topo[L]) * a.W + b] : 0);
      const int fut = a.future[probe * (T + 1) + L + 1];
      a.nxt_key[a.nxt_off[probe] + (long long)pos] = pr.alpha * ub - pr.beta * (double)(used + fut);
    }
    uint16_t* dst = a.nxt + (a.nxt_off[probe] + (long long)pos) * T;
    for (int k = 0; k < L; ++k) dst[k] = a.cur[s * T + k];
    dst[L] = rpos ? (uint16_t)b : (uint16_t)NONE16;
  }
}

// ---------------------------------------------------------------- leaves

struct Cand {
  int has, sl;
  double obj;
  long long code;
  int has_leaf;
  long long leaf;
};

__device__ __forceinline__ void code_choices(const S2Args& a, long long code, uint16_t* ch) {
  const long long s = code >> 16;
  for (int k = 0; k < a.level; ++k) ch[k] = a.cur[s * a.T + k];
  ch[a.level] = (uint16_t)(code & 0xFFFF);
}

__device__ inline int cmp_leaf(const S2Args& a, long long c1, long long c2) {
  uint16_t x[MAXT], y[MAXT];
  code_choices(a, c1, x);
  code_choices(a, c2, y);
  for (int k = 0; k < a.T; ++k) {
    const unsigned u = x[k] == NONE16 ? 0u : x[k], v = y[k] == NONE16 ? 0u : y[k];
    if (u != v) return u < v ? -1 : 1;
  }
  return 0;
}

// m(leaf c1) vs m(leaf c2) as Python tuple comparison (planner.py:852)
__device__ inline int cmp_tie(const S2Args& a, int probe, long long c1, long long c2) {
  uint16_t x[MAXT], y[MAXT];
  code_choices(a, c1, x);
  code_choices(a, c2, y);
  MCursor cx{&a, probe, x, 0, 0, 0, 0}, cy{&a, probe, y, 0, 0, 0, 0};
  cx.open_task();
  cy.open_task();
  while (true) {
    unsigned long long ex = 0, ey = 0;
    const bool hx = cx.next(ex), hy = cy.next(ey);
    if (!hx || !hy) return hx == hy ? 0 : (hx ? 1 : -1);  // a strict prefix is smaller
    if (ex != ey) return ex < ey ? -1 : 1;
  }
}

// is A a better feasible candidate than B?
__device__ inline bool better(const S2Args& a, int probe, const Cand& A, const Cand& B) {
  if (!A.has) return false;
  if (!B.has) return true;
  if (a.mode == LEAF_FULL) {
    if (A.obj != B.obj) return A.obj > B.obj;
    if (A.sl != B.sl) return A.sl < B.sl;
    return cmp_tie(a, probe, A.code, B.code) < 0;
  }
  if (a.mode == LEAF_FIRST) return cmp_leaf(a, A.code, B.code) < 0;
  return false;
}

__device__ inline void merge(const S2Args& a, int probe, Cand& X, const Cand& Y) {
  if (better(a, probe, Y, X)) {
    X.has = Y.has; X.sl = Y.sl; X.obj = Y.obj; X.code = Y.code;
  }
  if (a.diag && Y.has_leaf && (!X.has_leaf || cmp_leaf(a, Y.leaf, X.leaf) > 0)) {
    X.has_leaf = 1;
    X.leaf = Y.leaf;
  }
}

__global__ void __launch_bounds__(256) k_s2_leaf(const __grid_constant__ S2Args a) {
  __shared__ int sk[5];
  __shared__ Cand sc[256];
  __shared__ unsigned long long s_leaves;
  if (threadIdx.x < 5) sk[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_leaves = 0;
  __syncthreads();
  const long long blk = blockIdx.x;
  const int probe = find_probe(a.boff, a.n_probes, blk);
  const long long chunk = blk - a.boff[probe];
  const long long w_begin = a.pstart[probe];
  const long long w_end = w_begin + (long long)a.ptot[probe];
  const long long s_lo = a.foff[probe], s_hi = a.foff[probe] + a.fcap[probe];
  const long long w0 = w_begin + chunk * (long long)blockDim.x * a.ipt;
  const DGraph& g = *a.g;
  const DReq& rq = *a.rq;
  const DProbe& pr = a.probes[probe];
  const bool check_bound = (a.mode == LEAF_FULL);
  const int L = a.level;
  Cand best;
  best.has = 0; best.sl = 0; best.obj = 0.0; best.code = 0; best.has_leaf = 0; best.leaf = 0;
  unsigned long long leaves = 0;
  volatile int* found = a.active;  // per-probe "found" flags of feasible-only probes
  uint16_t ch[MAXT];
  for (int k = 0; k < a.ipt; ++k) {
    const long long w = w0 + (long long)k * blockDim.x + threadIdx.x;
    if (w >= w_end) break;
    if (a.mode == LEAF_ANY && found[probe]) break;
    const long long s = find_slot(a.pfx, s_lo, s_hi, w);
    const int b = (int)(w - a.pfx[s]);
    double ub = 0.0;
    const int st = filter_item(a, probe, s, b, check_bound, ub);
    if (st == ST_SKIP) continue;
    const bool rpos = a.pr_flag[s] & 1;
    if (a.diag && rpos) {
      if (st >= 0 && st < 5) atomicAdd(&sk[st], 1);
      else atomicOr(&a.cur_flag[s], 2);
    }
    if (st != ST_PASS) continue;
    for (int q = 0; q < L; ++q) ch[q] = a.cur[s * a.T + q];
    ch[L] = rpos ? (uint16_t)b : (uint16_t)NONE16;
    // leaf: derive_configuration + validate_configuration from scratch
    double lat[MAXT], cap[MAXT], acc[MAXT], fan[MAXE];
    int sl[MAXT];
    uint32_t present;
    load_leaf(a, probe, ch, lat, cap, acc, sl, fan, present);
    EvalOut ev;
    evaluate<false>(g, rq, pr, lat, cap, acc, sl, fan, present, ev, nullptr, nullptr, nullptr,
                    nullptr);
    ++leaves;
    const long long code = (s << 16) | (long long)ch[L];
    if (a.diag && (!best.has_leaf || cmp_leaf(a, code, best.leaf) > 0)) {
      best.has_leaf = 1;
      best.leaf = code;
    }
    if (!ev.feasible) continue;
    if (a.mode == LEAF_ANY) {
      best.has = 1;
      best.obj = ev.objective;
      best.sl = ev.total_sl;
      best.code = code;
      found[probe] = 1;
      break;
    }
    Cand c;
    c.has = 1; c.sl = ev.total_sl; c.obj = ev.objective; c.code = code; c.has_leaf = 0; c.leaf = 0;
    if (better(a, probe, c, best)) {
      best.has = 1; best.sl = c.sl; best.obj = c.obj; best.code = c.code;
      if (a.mode == LEAF_FULL) {
        const unsigned long long ob = obj_bits(c.obj);
        if (ob > ((volatile unsigned long long*)a.inc)[probe]) atomicMax(&a.inc[probe], ob);
      }
    }
  }
  sc[threadIdx.x] = best;
  atomicAdd(&s_leaves, leaves);
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      Cand x = sc[threadIdx.x];
      merge(a, probe, x, sc[threadIdx.x + st]);
      sc[threadIdx.x] = x;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    LeafPart& P = a.part[blk];
    P.has = sc[0].has;
    P.sl = sc[0].sl;
    P.obj = sc[0].obj;
    P.code = sc[0].code;
    P.has_leaf = sc[0].has_leaf;
    P.leaf = sc[0].leaf;
    P.leaves = s_leaves;
  }
  if (a.diag && threadIdx.x < 5 && sk[threadIdx.x])
    atomicAdd(&a.best[probe].kills[L][threadIdx.x], sk[threadIdx.x]);
}

// m(choices x) vs m(choices y), both by topo position (planner.py:852)
__device__ inline int cmp_choice_m(const S2Args& a, int probe, const uint16_t* x, const uint16_t* y) {
  MCursor cx{&a, probe, x, 0, 0, 0, 0}, cy{&a, probe, y, 0, 0, 0, 0};
  cx.open_task();
  cy.open_task();
  while (true) {
    unsigned long long ex = 0, ey = 0;
    const bool hx = cx.next(ex), hy = cy.next(ey);
    if (!hx || !hy) return hx == hy ? 0 : (hx ? 1 : -1);  // a strict prefix is smaller
    if (ex != ey) return ex < ey ? -1 : 1;
  }
}

// DFS order of two choice vectors (cmp_leaf's order)
__device__ inline int cmp_choice_dfs(int T, const uint16_t* x, const uint16_t* y) {
  for (int k = 0; k < T; ++k) {
    const unsigned u = x[k] == NONE16 ? 0u : x[k], v = y[k] == NONE16 ? 0u : y[k];
    if (u != v) return u < v ? -1 : 1;
  }
  return 0;
}

// per-probe fold of the leaf-block partials into BestRec (merged with what an earlier
// frontier chunk of the same probe left there: the chunks of a split level)
__global__ void __launch_bounds__(256) k_s2_reduce(const __grid_constant__ S2Args a) {
  __shared__ Cand sc[256];
  __shared__ unsigned long long s_leaves;
  const int probe = blockIdx.x;
  const long long b0 = a.boff[probe], b1 = a.boff[probe + 1];
  if (b0 == b1) return;
  if (threadIdx.x == 0) s_leaves = 0;
  __syncthreads();
  Cand best;
  best.has = 0; best.sl = 0; best.obj = 0.0; best.code = 0; best.has_leaf = 0; best.leaf = 0;
  unsigned long long leaves = 0;
  for (long long i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const LeafPart& P = a.part[i];
    Cand c;
    c.has = P.has; c.sl = P.sl; c.obj = P.obj; c.code = P.code; c.has_leaf = P.has_leaf;
    c.leaf = P.leaf;
    merge(a, probe, best, c);
    leaves += P.leaves;
  }
  sc[threadIdx.x] = best;
  atomicAdd(&s_leaves, leaves);
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      Cand x = sc[threadIdx.x];
      merge(a, probe, x, sc[threadIdx.x + s]);
      sc[threadIdx.x] = x;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    BestRec* B = a.best + probe;
    B->leaves += s_leaves;
    const Cand& c = sc[0];
    if (c.has) {
      uint16_t ch[MAXT];
      code_choices(a, c.code, ch);
      bool take = !B->has;
      if (!take && a.mode == LEAF_FULL) {
        if (c.obj != B->obj) take = c.obj > B->obj;
        else if (c.sl != B->sl) take = c.sl < B->sl;
        else take = cmp_choice_m(a, probe, ch, B->choice) < 0;
      } else if (!take && a.mode == LEAF_FIRST) {
        take = cmp_choice_dfs(a.T, ch, B->choice) < 0;
      }
      if (take) {
        for (int k = 0; k < a.T; ++k) B->choice[k] = ch[k];
        B->obj = c.obj;
        B->sl = c.sl;
      }
      B->has = 1;
      B->found = 1;
    }
    if (c.has_leaf) {
      uint16_t ch[MAXT];
      code_choices(a, c.leaf, ch);
      if (!B->has_leaf || cmp_choice_dfs(a.T, ch, B->leaf_choice) > 0) {
        for (int k = 0; k < a.T; ++k) B->leaf_choice[k] = ch[k];
        B->has_leaf = 1;
      }
    }
  }
}

// deepest blocked level: a prefix with r > 0 whose children all died (planner.py:910-911)
__global__ void k_s2_blocked(const __grid_constant__ S2Args a) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= a.n_slots) return;
  const int f = a.cur_flag[s];
  if ((f & 1) && !(f & 2)) atomicMax(&a.best[a.pr_probe[s]].deepest, a.level);
}

int launch_stage2_prep(const S2Args& a, double* min_lat2, int* min_sl, double* acc_ub, int* future,
                       cudaStream_t st) {
  // on entry S2Args.min_lat2 / min_sl / acc_ub point at the Stage-1 per-pool values
  PROF_BEGIN(K_S2_PREP);
  k_s2_prep<<<(a.n_probes + 127) / 128, 128, 0, st>>>(a, min_lat2, min_sl, acc_ub, future,
                                                       a.min_lat2, a.min_sl, a.acc_ub);
  PROF_END();
  return 1;
}

int launch_stage2_prefix(const S2Args& a, cudaStream_t st) {
  if (a.n_slots <= 0) return 0;
  PROF_BEGIN(K_S2_PREFIX);
  k_s2_prefix<<<(unsigned)((a.n_slots + 255) / 256), 256, 0, st>>>(a);
  PROF_END();
  return 1;
}

int launch_stage2_level(const S2Args& a, long long total, cudaStream_t st) {
  if (total <= 0) return 0;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  PROF_BEGIN(K_S2_LEVEL);
  k_s2_level<<<(unsigned)blocks, 256, 0, st>>>(a);
  PROF_END();
  return 1;
}

// ---------------------------------------------------------------- best-first
// A frontier about to be split into depth-first halves is first ordered by its
// children's objective upper bound (descending, per probe): the first half then
// holds the most promising prefixes, its leaves set an incumbent early and the
// bound prunes every later chunk.  The order changes only the traversal (every
// filter is admissible and the chunk merges are order-free), never a result; it
// also makes the traversal independent of the atomic slot order of k_s2_level.

__global__ void k_fr_keys(const double* key, double* kout, int* perm, const long long* foff,
                          const long long* fcap, const unsigned long long* fcnt) {
  const int i = blockIdx.y;
  const long long cap = fcap[i];
  const long long m = min((long long)fcnt[i], cap);
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < cap;
       k += (long long)gridDim.x * blockDim.x) {
    const long long s = foff[i] + k;
    kout[s] = k < m ? key[s] : -INFINITY;
    perm[s] = (int)s;
  }
}

__global__ void k_fr_gather(const uint16_t* src, uint16_t* dst, const int* perm, const long long* foff,
                            const long long* fcap, int T) {
  const int i = blockIdx.y;
  const long long cap = fcap[i];
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < cap;
       k += (long long)gridDim.x * blockDim.x) {
    const long long s = foff[i] + k;
    const long long f = perm[s];
    for (int q = 0; q < T; ++q) dst[s * T + q] = src[f * T + q];
  }
}

int launch_frontier_best_first(const double* key, uint16_t* rows, uint16_t* rows_tmp, double* k_tmp,
                               double* k_out, int* perm, int* perm_out, void* sort_tmp,
                               size_t* sort_bytes, const long long* foff, const long long* fcap,
                               const long long* seg_end, const unsigned long long* fcnt, int n,
                               long long n_slots, long long max_cap, int T, cudaStream_t st) {
  // sort_tmp == nullptr: only report the scratch the segmented sort needs
  if (!sort_tmp) {
    return (int)cub::DeviceSegmentedRadixSort::SortPairsDescending(
        nullptr, *sort_bytes, k_tmp, k_out, perm, perm_out, (int)n_slots, n, foff, seg_end, 0, 64, st);
  }
  if (n <= 0 || n_slots <= 0 || max_cap <= 0) return (int)cudaSuccess;
  const dim3 grid((unsigned)std::min<long long>(64, (max_cap + 255) / 256), (unsigned)n);
  k_fr_keys<<<grid, 256, 0, st>>>(key, k_tmp, perm, foff, fcap, fcnt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  e = cub::DeviceSegmentedRadixSort::SortPairsDescending(
      sort_tmp, *sort_bytes, k_tmp, k_out, perm, perm_out, (int)n_slots, n, foff, seg_end, 0, 64, st);
  if (e != cudaSuccess) return (int)e;
  k_fr_gather<<<grid, 256, 0, st>>>(rows, rows_tmp, perm_out, foff, fcap, T);
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  return (int)cudaMemcpyAsync(rows, rows_tmp, sizeof(uint16_t) * (size_t)n_slots * T,
                              cudaMemcpyDeviceToDevice, st);
}

int launch_stage2_leaf(const S2Args& a, long long n_blocks, cudaStream_t st) {
  if (n_blocks <= 0) return 0;
  PROF_BEGIN(K_S2_LEAF);
  k_s2_leaf<<<(unsigned)n_blocks, 256, 0, st>>>(a);
  PROF_END();
  PROF_BEGIN(K_S2_REDUCE);
  k_s2_reduce<<<a.n_probes, 256, 0, st>>>(a);
  PROF_END();
  return 2;
}

int launch_stage2_blocked(const S2Args& a, cudaStream_t st) {
  if (a.n_slots <= 0) return 0;
  k_s2_blocked<<<(unsigned)((a.n_slots + 255) / 256), 256, 0, st>>>(a);
  return 1;
}
