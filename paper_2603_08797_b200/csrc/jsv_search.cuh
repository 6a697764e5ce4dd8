// jsv_search.cuh -- level-synchronous branch-and-bound expansion and the
// lock-free leaf reduction (included by jsv_stage2.cu).
//
// A work item (prefix, b) applies the reference _visit filters
// (planner.py:876-903) in order.  Intermediate levels append surviving
// children to the next frontier; the last level derives + validates each
// reached leaf (planner.py:835-855) and reduces it per thread, per block
// (shared memory) and finally per probe (k_s2_reduce) -- no locks, so
// thousands of concurrent feasible leaves never serialise.

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

// Per-thread scratch of expand_item.  Declared once at kernel scope by the
// callers: with the arrays local to the inlined callee, nvcc 12.9's stack
// slot colouring overlapped the callee's acc[] with the caller's ch[].
struct ExpScratch {
  double r[MAXT];
  double acc[MAXT];
  uint16_t ch[MAXT];
};

// Apply the node filters to child b of prefix pidx; fills xs.ch[0..L].
__device__ __forceinline__ int expand_item(const S2Args& a, int probe, long long pidx, int b,
                                           ExpScratch& xs, bool& rpos, bool check_bound) {
  const DGraph& g = *a.g;
  const DReq& rq = *a.rq;
  const int T = a.T, L = a.level;
  const int t = g.topo[L];
  uint16_t* ch = xs.ch;
  for (int k = 0; k < L; ++k) ch[k] = a.cur[pidx * T + k];
  const DProbe& pr = a.probes[probe];
  const int jb = probe * T;
  double* r = xs.r;
  int used = 0;
  for (int k = 0; k <= L; ++k) {
    const int u = g.topo[k];
    double ru;
    if (u == g.entry) {
      ru = pr.demand;
    } else {
      // _demand_at (planner.py:821-833)
      ru = 0.0;
      for (int qq = g.pred_off[u]; qq < g.pred_off[u + 1]; ++qq) {
        const int e = g.pred_edge[qq];
        const int s = g.edge_src[e];
        const int cs = ch[g.pos_of[s]];
        if (cs == NONE16 || r[s] == 0.0) continue;
        const double fan = rq.has_ov[e] ? rq.ov[e]
                                        : a.p_fan[((long long)(jb + s) * a.W + cs) * a.maxout +
                                                  (e - g.succ_off[s])];
        ru += r[s] * fan;
      }
    }
    r[u] = ru;
    if (k < L && ch[k] != NONE16) used += a.p_sl[(long long)(jb + u) * a.W + ch[k]];
  }
  const double rt = r[t];
  if (rt == 0.0) {
    rpos = false;
    if (b != 0) return ST_SKIP;
    ch[L] = NONE16;
    return ST_PASS;
  }
  rpos = true;
  const int P = a.pool_n[jb + t];
  if (b >= P) return ST_SKIP;
  const long long q = (long long)(jb + t) * a.W + b;
  const int* fut = a.future + probe * (T + 1);
  const double need = rt * (1.0 + rq.slack);
  const double eps = rq.eps;
  const int bsl = a.p_sl[q];
  if (a.p_cap[q] + eps < need) return JSV_BIND_THROUGHPUT;
  if ((double)(used + bsl + fut[L + 1]) > (double)rq.S + eps) return JSV_BIND_RESOURCES;
  // partial-path latency (_latency_ok, planner.py:805-819)
  const double lat2 = 2.0 * a.p_lat[q];
  for (int pp = 0; pp < g.P; ++pp) {
    if (!((g.path_mask[pp] >> t) & 1u)) continue;
    double tot = 0.0;
    for (int k = g.path_off[pp]; k < g.path_off[pp + 1]; ++k) {
      const int u = g.path_task[k];
      if (u == t) {
        tot += lat2;
      } else if (g.pos_of[u] < L) {
        const int c = ch[g.pos_of[u]];
        tot += (c == NONE16) ? 0.0 : 2.0 * a.p_lat[(long long)(jb + u) * a.W + c];
      } else {
        tot += a.min_lat2[jb + u];
      }
    }
    if (tot > pr.slo_eff + eps) return JSV_BIND_LATENCY;
  }
  // accuracy upper bound (planner.py:889-894)
  double* acc = xs.acc;
  for (int u = 0; u < T; ++u) {
    const int pu = g.pos_of[u];
    if (pu < L) {
      const int c = ch[pu];
      acc[u] = (c == NONE16) ? 1.0 : a.p_acc[(long long)(jb + u) * a.W + c];
    } else if (u == t) {
      acc[u] = a.p_acc[q];
    } else {
      acc[u] = a.acc_ub[jb + u];
    }
  }
  const double ub = weighted_paths(g, acc) / g.a_max;
  if (ub < pr.acc_slo - eps) return JSV_BIND_ACCURACY;
  ch[L] = (uint16_t)b;
  if (check_bound) {
    // objective bound against the incumbent (planner.py:895-902)
    const unsigned long long ib = ((volatile unsigned long long*)a.inc)[probe];
    if (ib) {
      const double obj_ub = pr.alpha * ub - pr.beta * (double)(used + bsl + fut[L + 1]);
      if (obj_ub < bits_obj(ib) - eps) return ST_BOUND;
    }
  }
  return ST_PASS;
}

__global__ void __launch_bounds__(256) k_s2_level(S2Args a) {
  const int T = a.T, L = a.level;
  const long long stride = (long long)gridDim.x * blockDim.x;
  ExpScratch xs;
  const uint16_t* ch = xs.ch;
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < a.total_work;
       w += stride) {
    int lo = 0, hi = a.n_probes - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.woff[mid] <= w) lo = mid;
      else hi = mid - 1;
    }
    const int probe = lo;
    const long long lw = w - a.woff[probe];
    const int width = a.width[probe];
    const long long pidx = a.foff[probe] + lw / width;
    const int b = (int)(lw % width);
    bool rpos = false;
    const int st = expand_item(a, probe, pidx, b, xs, rpos, false);
    if (st == ST_SKIP) continue;
    if (a.diag && rpos) {
      if (b == 0) atomicOr(&a.cur_flag[pidx], 1);
      if (st >= 0 && st < 5) atomicAdd(&a.best[probe].kills[L][st], 1);
      else atomicOr(&a.cur_flag[pidx], 2);
    }
    if (st != ST_PASS) continue;
    const unsigned long long pos = atomicAdd(&a.nxt_cnt[probe], 1ull);
    if ((long long)pos >= a.nxt_cap[probe]) {
      atomicExch(a.err, 3);
      continue;
    }
    uint16_t* dst = a.nxt + (a.nxt_off[probe] + (long long)pos) * T;
    for (int k = 0; k <= L; ++k) dst[k] = ch[k];
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
  const long long pidx = code >> 16;
  for (int k = 0; k < a.level; ++k) ch[k] = a.cur[pidx * a.T + k];
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

__device__ inline int cmp_tie(const S2Args& a, int probe, long long c1, long long c2) {
  const DGraph& g = *a.g;
  uint16_t x[MAXT], y[MAXT], cx[MAXT], cy[MAXT];
  code_choices(a, c1, x);
  code_choices(a, c2, y);
  for (int u = 0; u < a.T; ++u) {
    cx[u] = x[g.pos_of[u]];
    cy[u] = y[g.pos_of[u]];
  }
  unsigned long long kx[4], ky[4];
  tie_key(a, probe, cx, kx);
  tie_key(a, probe, cy, ky);
  return cmp_words(kx, ky, 4);
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

__device__ __forceinline__ int probe_of_block(const S2Args& a, long long blk) {
  int lo = 0, hi = a.n_probes - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.boff[mid] <= blk) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(256) k_s2_leaf(S2Args a) {
  __shared__ int sk[5];
  __shared__ Cand sc[256];
  __shared__ unsigned long long s_leaves;
  if (threadIdx.x < 5) sk[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_leaves = 0;
  __syncthreads();
  const long long blk = blockIdx.x;
  const int probe = probe_of_block(a, blk);
  const long long chunk = blk - a.boff[probe];
  const long long work = a.woff[probe + 1] - a.woff[probe];
  const int width = a.width[probe];
  const long long per_block = (long long)blockDim.x * a.ipt;
  const long long w0 = chunk * per_block;
  const DGraph& g = *a.g;
  const DReq& rq = *a.rq;
  const DProbe& pr = a.probes[probe];
  const bool check_bound = (a.mode == LEAF_FULL);
  Cand best;
  best.has = 0; best.sl = 0; best.obj = 0.0; best.code = 0; best.has_leaf = 0; best.leaf = 0;
  unsigned long long leaves = 0;
  volatile int* found = a.active;  // reused as the per-probe "found" flags
  ExpScratch xs;
  for (int k = 0; k < a.ipt; ++k) {
    const long long lw = w0 + (long long)k * blockDim.x + threadIdx.x;
    if (lw >= work) break;
    if (a.mode == LEAF_ANY && found[probe]) break;
    const long long pidx = a.foff[probe] + lw / width;
    const int b = (int)(lw % width);
    bool rpos = false;
    const int st = expand_item(a, probe, pidx, b, xs, rpos, check_bound);
    const uint16_t* ch = xs.ch;
    if (st == ST_SKIP) continue;
    if (a.diag && rpos) {
      if (b == 0) atomicOr(&a.cur_flag[pidx], 1);
      if (st >= 0 && st < 5) atomicAdd(&sk[st], 1);
      else atomicOr(&a.cur_flag[pidx], 2);
    }
    if (st != ST_PASS) continue;
    // leaf: derive_configuration + validate_configuration from scratch
    double lat[MAXT], cap[MAXT], acc[MAXT], fan[MAXE];
    int sl[MAXT];
    uint32_t present;
    load_leaf(a, probe, ch, lat, cap, acc, sl, fan, present);
    EvalOut ev;
    evaluate<false>(g, rq, pr, lat, cap, acc, sl, fan, present, ev, nullptr, nullptr, nullptr,
                    nullptr);
    ++leaves;
    const long long code = (pidx << 16) | (long long)ch[a.level];
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
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      Cand x = sc[threadIdx.x];
      merge(a, probe, x, sc[threadIdx.x + s]);
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
    atomicAdd(&a.best[probe].kills[a.level][threadIdx.x], sk[threadIdx.x]);
}

// per-probe fold of the leaf-block partials into BestRec
__global__ void __launch_bounds__(256) k_s2_reduce(S2Args a) {
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
      for (int k = 0; k < a.T; ++k) B->choice[k] = ch[k];
      B->has = 1;
      B->found = 1;
      B->obj = c.obj;
      B->sl = c.sl;
    }
    if (c.has_leaf) {
      uint16_t ch[MAXT];
      code_choices(a, c.leaf, ch);
      for (int k = 0; k < a.T; ++k) B->leaf_choice[k] = ch[k];
      B->has_leaf = 1;
    }
  }
}

// debug: every frontier entry must hold valid pool indices
__global__ void k_s2_check(S2Args a, long long n_prefix, int depth, const int* prefix_probe) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n_prefix) return;
  const int probe = prefix_probe[i];
  for (int k = 0; k < depth; ++k) {
    const int c = a.cur[i * a.T + k];
    const int t = a.g->topo[k];
    if (c != NONE16 && c >= a.pool_n[probe * a.T + t])
      printf("bad frontier entry %lld pos %d value %d (pool %d)\n", i, k, c,
             a.pool_n[probe * a.T + t]);
  }
}

int launch_stage2_check(const S2Args& a, long long n, int depth, const int* pp, cudaStream_t st) {
  if (n <= 0) return 0;
  k_s2_check<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a, n, depth, pp);
  return 1;
}

// deepest blocked level: a prefix with r > 0 whose children all died (planner.py:910-911)
__global__ void k_s2_blocked(S2Args a, long long n_prefix, const int* prefix_probe) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n_prefix) return;
  const int f = a.cur_flag[i];
  if ((f & 1) && !(f & 2)) atomicMax(&a.best[prefix_probe[i]].deepest, a.level);
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

int launch_stage2_level(const S2Args& a, cudaStream_t st) {
  if (a.total_work <= 0) return 0;
  long long blocks = (a.total_work + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  PROF_BEGIN(K_S2_LEVEL);
  k_s2_level<<<(unsigned)blocks, 256, 0, st>>>(a);
  PROF_END();
  return 1;
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

int launch_stage2_blocked(const S2Args& a, long long n_prefix_total, const int* prefix_probe,
                          cudaStream_t st) {
  if (n_prefix_total <= 0) return 0;
  k_s2_blocked<<<(unsigned)((n_prefix_total + 255) / 256), 256, 0, st>>>(a, n_prefix_total,
                                                                         prefix_probe);
  return 1;
}
