// jsv_fanout.cuh -- exact Stage 2 for fan-out graphs too large to sweep
// (included by jsv_stage2.cu).  BASELINE configs[3]: the 12-task star, whose
// cross-product (~459^12) neither the reference's DFS (it does not finish,
// SURVEY.md a12) nor the exhaustive sweep can cover.
//
// Graph class: one entry task e and k leaves, each leaf's only predecessor is e
// and it has no successors (one path (e, leaf) per leaf, graph.paths order).
// Once e's bundle b0 is fixed, every leaf's verdicts are independent
// (throughput: cap - r0 * fan(b0, leaf) * (1 + slack) >= 0; latency: the
// two-term CPython sum 2 L(b0) + 2 L(leaf) <= slo_eff), and the rest couples
// the leaves only through sums: slices (resources) and the path-weighted
// accuracy W = sum_leaf frac * ((1.0 * acc0) * acc_leaf) (model.py:267-282),
// which the objective alpha * W / a_max - beta * slices increases.
//
//   k_fo_prep   one block per (probe, b0): per leaf the distinct (slices,
//               accuracy) classes of its feasible bundles (bitonic sort +
//               unique), then a suffix DP over the leaves
//               F[j][s] = max sum of leaf accuracy terms of leaves j.. using
//               exactly s slices, and b0's best objective over s (real arith.)
//   k_fo_tau    per probe: tau = best over b0 - delta
//   k_fo_enum   one thread per (probe, b0, total slices) whose DP optimum
//               reaches tau: depth-first enumeration of every class vector
//               whose real objective reaches tau (DP suffix bounds prune)
//   k_fo_eval   one thread per enumerated class vector: each leaf takes the
//               m-smallest feasible bundle of its class (bundles of one class
//               tie on objective and slices, so only m separates them), then
//               derive_configuration + validate_configuration exactly in the
//               reference's order; the (objective, slices, m) argmax is
//               folded per probe under a lock.
//
// Exactness: a feasible candidate X with float objective >= the returned
// optimum F' has real objective >= F' - eps, and every such X is enumerated
// while tau <= F' - eps; the host lowers tau and repeats until that holds.
// Dropping nothing but identical-class duplicates (resolved by m) keeps the
// reference's tie-breaks.

__device__ __forceinline__ long long fo_cls_base(const FoArgs& a, int probe, int b0, int j) {
  return (((long long)probe * a.P0max + b0) * a.k + j) * a.s.W;
}
__device__ __forceinline__ long long fo_F_base(const FoArgs& a, int probe, int b0, int j) {
  return (((long long)probe * a.P0max + b0) * (a.k + 1) + j) * (long long)(a.SB + 1);
}

// leaf demand r_leaf = 0.0 + r0 * fan (model.py:239-264, evaluate() order)
__device__ __forceinline__ double fo_leaf_demand(const FoArgs& a, int probe, int b0, int j) {
  const S2Args& s = a.s;
  const DGraph& g = *s.g;
  const int e = a.edge[j];
  const double fan = s.rq->has_ov[e]
                         ? s.rq->ov[e]
                         : s.p_fan[((long long)(probe * s.T + a.entry) * s.W + b0) * s.maxout +
                                   (e - g.succ_off[a.entry])];
  double d = 0.0;
  d += s.probes[probe].demand * fan;
  return d;
}

// throughput + latency verdicts of leaf bundle b given the entry bundle b0
__device__ __forceinline__ bool fo_leaf_ok(const FoArgs& a, int probe, int b0, int j, int b,
                                           double need) {
  const S2Args& s = a.s;
  const long long q = (long long)(probe * s.T + a.leaf[j]) * s.W + b;
  if (!(s.p_cap[q] - need >= 0)) return false;
  PySum ps;
  ps.add(2.0 * s.p_lat[(long long)(probe * s.T + a.entry) * s.W + b0]);
  ps.add(2.0 * s.p_lat[q]);
  return s.probes[probe].slo_eff - ps.result() >= 0;
}

__global__ void __launch_bounds__(256) k_fo_prep(const __grid_constant__ FoArgs a) {
  __shared__ double sacc[1024];  // feasible bundles of one leaf as (slices, accuracy) pairs
  __shared__ int ssl[1024];
  __shared__ int msl[1024];       // DP classes: per slices value, the largest accuracy
  __shared__ double mac[1024];
  __shared__ int scount, smcount;
  typedef cub::BlockScan<int, 256> FoScan;
  __shared__ typename FoScan::TempStorage ftmp;
  const S2Args& s = a.s;
  const int probe = blockIdx.x / a.P0max, b0 = blockIdx.x % a.P0max;
  const int T = s.T;
  const int P0 = s.pool_n[probe * T + a.entry];
  const long long bq = ((long long)probe * a.P0max + b0);
  // (sharded solve: this rank's block of entry bundles)
  const int lo0 = (int)((long long)P0 * a.shard_rank / a.shard_world);
  const int hi0 = (int)((long long)P0 * (a.shard_rank + 1) / a.shard_world);
  if (!a.act[probe] || b0 >= P0 || b0 < lo0 || b0 >= hi0) {
    if (threadIdx.x == 0) a.b0best[bq] = -INFINITY;
    return;
  }
  const DProbe& pr = s.probes[probe];
  const DGraph& g = *s.g;
  const double sf = 1.0 + s.rq->slack;
  const long long q0 = (long long)(probe * T + a.entry) * s.W + b0;
  const double acc0 = s.p_acc[q0];
  const int s0 = s.p_sl[q0];
  // entry throughput verdict; the budget must leave room for the entry itself
  const bool b0_ok = (s.p_cap[q0] - pr.demand * sf >= 0) && (s0 <= a.SB);
  // Leaves in reverse order: each leaf's class list is built (global, for
  // k_fo_enum) and its suffix-DP step taken at once.  The DP only needs, per
  // slices value, the class of largest accuracy (w is monotone in it and the
  // rest term depends on slices alone), so the step runs over <= SB + 1
  // classes held in shared memory -- the same maxima as over every class.
  const int SB = a.SB;
  for (int sv = threadIdx.x; sv <= SB; sv += blockDim.x)
    a.F[fo_F_base(a, probe, b0, a.k) + sv] = (sv == 0) ? 0.0 : -INFINITY;
  for (int j = a.k - 1; j >= 0; --j) {
    const int lt = a.leaf[j];
    const int Pl = s.pool_n[probe * T + lt];
    const double r = fo_leaf_demand(a, probe, b0, j);
    const long long cb = fo_cls_base(a, probe, b0, j);
    __syncthreads();
    if (r == 0.0) {
      // only "no instances" (planner.py:868-875): slices 0, accuracy 1.0
      if (threadIdx.x == 0) {
        a.cls[cb].acc = 1.0; a.cls[cb].s = 0;
        a.ncls[bq * a.k + j] = 1;
        msl[0] = 0; mac[0] = 1.0;
        smcount = 1;
      }
    } else {
      const double need = r * sf;
      int n2 = 1;
      while (n2 < Pl) n2 <<= 1;
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        if (i < Pl && fo_leaf_ok(a, probe, b0, j, i, need)) {
          const long long q = (long long)(probe * T + lt) * s.W + i;
          ssl[i] = s.p_sl[q];
          sacc[i] = s.p_acc[q];
        } else {
          ssl[i] = 0x7FFFFFFF;
          sacc[i] = INFINITY;
        }
      }
      __syncthreads();
      // bitonic sort by (slices, accuracy)
      for (int kk = 2; kk <= n2; kk <<= 1) {
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
          for (int i = threadIdx.x; i < n2; i += blockDim.x) {
            const int l = i ^ jj;
            if (l > i) {
              const bool up = (i & kk) == 0;
              const bool gt = ssl[i] > ssl[l] || (ssl[i] == ssl[l] && sacc[i] > sacc[l]);
              if (gt == up) {
                const int ts = ssl[i]; ssl[i] = ssl[l]; ssl[l] = ts;
                const double ta = sacc[i]; sacc[i] = sacc[l]; sacc[l] = ta;
              }
            }
          }
          __syncthreads();
        }
      }
      // unique -> class list (global), and the last class of each slices value
      // -> DP classes (shared); block scans over chunks of the sorted list
      if (threadIdx.x == 0) { scount = 0; smcount = 0; }
      __syncthreads();
      for (int i0 = 0; i0 < n2; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        const bool valid = i < n2 && ssl[i] != 0x7FFFFFFF;
        const int fu = valid && (i == 0 || ssl[i] != ssl[i - 1] || !(sacc[i] == sacc[i - 1]));
        const int fm = valid && (i + 1 == n2 || ssl[i + 1] != ssl[i]);
        int ou, tu, om, tm;
        FoScan(ftmp).ExclusiveSum(fu, ou, tu);
        __syncthreads();
        FoScan(ftmp).ExclusiveSum(fm, om, tm);
        if (fu) {
          a.cls[cb + scount + ou].acc = sacc[i];
          a.cls[cb + scount + ou].s = ssl[i];
        }
        if (fm) {
          msl[smcount + om] = ssl[i];
          mac[smcount + om] = sacc[i];
        }
        __syncthreads();
        if (threadIdx.x == 0) { scount += tu; smcount += tm; }
        __syncthreads();
      }
      if (threadIdx.x == 0) a.ncls[bq * a.k + j] = scount;
    }
    __syncthreads();
    // suffix DP step (real arithmetic: a bound, not a verdict)
    const int nm = smcount;
    const double frac = g.path_frac[j];
    const double* Fn = a.F + fo_F_base(a, probe, b0, j + 1);
    double* Fj = a.F + fo_F_base(a, probe, b0, j);
    for (int sv = threadIdx.x; sv <= SB; sv += blockDim.x) {
      double best = -INFINITY;
      for (int c = 0; c < nm; ++c) {
        const int sc = msl[c];
        if (sc > sv) break;  // classes sorted by slices
        const double rest = Fn[sv - sc];
        if (rest == -INFINITY) continue;
        const double w = frac * ((1.0 * acc0) * mac[c]);
        const double v = w + rest;
        best = v > best ? v : best;
      }
      Fj[sv] = best;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double best = -INFINITY;
    if (b0_ok) {
      const double* F0 = a.F + fo_F_base(a, probe, b0, 0);
      const double wmin = pr.acc_slo * g.a_max - FO_DELTA_W;
      for (int sv = 0; sv + s0 <= SB; ++sv) {
        const double W = F0[sv];
        if (W == -INFINITY || W < wmin) continue;
        const double obj = pr.alpha * (W / g.a_max) - pr.beta * (double)(s0 + sv);
        best = obj > best ? obj : best;
      }
    }
    a.b0best[bq] = best;
  }
}

__global__ void __launch_bounds__(256) k_fo_tau(const __grid_constant__ FoArgs a, double delta) {
  __shared__ double sb[256];
  const int probe = blockIdx.x;
  double best = -INFINITY;
  for (int b = threadIdx.x; b < a.P0max; b += blockDim.x) {
    const double v = a.b0best[(long long)probe * a.P0max + b];
    best = v > best ? v : best;
  }
  sb[threadIdx.x] = best;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st && sb[threadIdx.x + st] > sb[threadIdx.x]) sb[threadIdx.x] = sb[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) a.tau[probe] = sb[0] - delta;
}

// one thread per (probe, b0, total leaf slices); DFS stacks in shared memory
#define FO_ENUM_THREADS 128
__global__ void __launch_bounds__(FO_ENUM_THREADS) k_fo_enum(const __grid_constant__ FoArgs a) {
  __shared__ double s_part[MAXT + 1][FO_ENUM_THREADS];
  __shared__ int s_rem[MAXT + 1][FO_ENUM_THREADS];
  __shared__ int s_cur[MAXT][FO_ENUM_THREADS];
  const int tx = threadIdx.x;
  const long long id = blockIdx.x * (long long)blockDim.x + tx;
  const int SB = a.SB;
  const long long per_probe = (long long)a.P0max * (SB + 1);
  const int probe = (int)(id / per_probe);
  if (probe >= a.s.n_probes || !a.act[probe]) return;
  const int b0 = (int)((id % per_probe) / (SB + 1));
  const int stot = (int)(id % (SB + 1));
  const long long bq = (long long)probe * a.P0max + b0;
  if (a.b0best[bq] == -INFINITY || a.b0best[bq] < a.tau[probe]) return;
  const S2Args& s = a.s;
  const DProbe& pr = s.probes[probe];
  const DGraph& g = *s.g;
  const long long q0 = (long long)(probe * s.T + a.entry) * s.W + b0;
  const double acc0 = s.p_acc[q0];
  const int s0 = s.p_sl[q0];
  if (s0 + stot > SB) return;
  const double* F0 = a.F + fo_F_base(a, probe, b0, 0);
  if (F0[stot] == -INFINITY) return;
  // W must reach both the accuracy SLO and the objective threshold (real arithmetic)
  const double w_obj = (a.tau[probe] + pr.beta * (double)(s0 + stot)) * g.a_max / pr.alpha;
  double wneed = pr.acc_slo * g.a_max;
  wneed = (w_obj > wneed ? w_obj : wneed) - FO_DELTA_W;
  if (F0[stot] < wneed) return;
  const int k = a.k;
  int j = 0;
  s_rem[0][tx] = stot;
  s_part[0][tx] = 0.0;
  s_cur[0][tx] = -1;
  while (j >= 0) {
    const long long cb = fo_cls_base(a, probe, b0, j);
    const int nc = a.ncls[bq * k + j];
    const double frac = g.path_frac[j];
    const double* Fn = a.F + fo_F_base(a, probe, b0, j + 1);
    const int rj = s_rem[j][tx];
    const double pj = s_part[j][tx];
    int c = s_cur[j][tx] + 1;
    int found = -1;
    for (; c < nc; ++c) {
      const int sc = a.cls[cb + c].s;
      if (sc > rj) break;
      const double rest = Fn[rj - sc];
      if (rest == -INFINITY) continue;
      const double w = frac * ((1.0 * acc0) * a.cls[cb + c].acc);
      if (pj + w + rest < wneed) continue;
      found = c;
      s_rem[j + 1][tx] = rj - sc;
      s_part[j + 1][tx] = pj + w;
      break;
    }
    if (found < 0) {
      --j;
      continue;
    }
    s_cur[j][tx] = found;
    if (j + 1 == k) {
      if (s_rem[k][tx] == 0) {
        const unsigned long long slot = atomicAdd(a.ncand, 1ull);
        if ((long long)slot >= a.cand_cap) {
          atomicExch(a.overflow, 1);
          return;
        }
        FoCand& o = a.cand[slot];
        o.probe = probe;
        o.b0 = b0;
        for (int t = 0; t < k; ++t) o.cls[t] = (uint16_t)s_cur[t][tx];
      }
      continue;  // next class at this leaf
    }
    ++j;
    s_cur[j][tx] = -1;
  }
}

// item-list order of two bundles of one task inside otherwise equal m tuples
// (planner.py:852): first differing item, else the shorter list is smaller iff
// no later task (larger id) holds instances
__device__ inline int fo_items_cmp(const S2Args& a, int probe, int t, int b1, int b2, bool later) {
  const long long jq = (long long)(probe * a.T + t) * a.W;
  const long long base = (long long)probe * a.C_probe + a.task_base[t];
  const long long c1 = base + a.pool_cand[jq + b1], c2 = base + a.pool_cand[jq + b2];
  const int n1 = a.nitems[c1], n2 = a.nitems[c2];
  const int n = n1 < n2 ? n1 : n2;
  for (int k = 0; k < n; ++k) {
    const uint32_t e1 = a.items[c1 * a.maxi + k], e2 = a.items[c2 * a.maxi + k];
    if (e1 != e2) return e1 < e2 ? -1 : 1;
  }
  if (n1 == n2) return 0;
  const int shorter = (n1 < n2) ? -1 : 1;
  return later ? -shorter : shorter;
}

// m of two full choice vectors (by topo position), Python tuple order
__device__ inline int fo_cmp_m(const S2Args& a, int probe, const uint16_t* x, const uint16_t* y) {
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

__global__ void __launch_bounds__(128) k_fo_eval(const __grid_constant__ FoArgs a, long long n) {
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= n) return;
  const FoCand& cd = a.cand[id];
  const int probe = cd.probe, b0 = cd.b0;
  const S2Args& s = a.s;
  const DGraph& g = *s.g;
  const int T = s.T;
  const double sf = 1.0 + s.rq->slack;
  const long long bq = (long long)probe * a.P0max + b0;
  uint16_t ch[MAXT];  // by topo position
  for (int k = 0; k < T; ++k) ch[k] = NONE16;
  ch[g.pos_of[a.entry]] = (uint16_t)b0;
  bool nonempty[MAXT];
  for (int t = 0; t < T; ++t) nonempty[t] = (t == a.entry);
  for (int j = 0; j < a.k; ++j) nonempty[a.leaf[j]] = fo_leaf_demand(a, probe, b0, j) != 0.0;
  for (int j = 0; j < a.k; ++j) {
    const int lt = a.leaf[j];
    const double r = fo_leaf_demand(a, probe, b0, j);
    if (r == 0.0) continue;  // no instances
    const FoCls c = a.cls[fo_cls_base(a, probe, b0, j) + cd.cls[j]];
    bool later = false;
    for (int t = lt + 1; t < T; ++t) later = later || nonempty[t];
    // the m-smallest feasible bundle of the class
    const int Pl = s.pool_n[probe * T + lt];
    const double need = r * sf;
    int pick = -1;
    for (int b = 0; b < Pl; ++b) {
      const long long q = (long long)(probe * T + lt) * s.W + b;
      if (s.p_sl[q] != c.s || !(s.p_acc[q] == c.acc)) continue;
      if (!fo_leaf_ok(a, probe, b0, j, b, need)) continue;
      if (pick < 0 || fo_items_cmp(s, probe, lt, b, pick, later) < 0) pick = b;
    }
    if (pick < 0) return;  // cannot happen: classes come from feasible bundles
    ch[g.pos_of[lt]] = (uint16_t)pick;
  }
  double lat[MAXT], cap[MAXT], acc[MAXT], fan[MAXE];
  int sl[MAXT];
  uint32_t present;
  load_leaf(s, probe, ch, lat, cap, acc, sl, fan, present);
  EvalOut ev;
  evaluate<false>(g, *s.rq, s.probes[probe], lat, cap, acc, sl, fan, present, ev, nullptr, nullptr,
                  nullptr, nullptr);
  (void)bq;
  if (!ev.feasible) return;
  BestRec* B = s.best + probe;
  spin_lock(&B->lock);
  bool take = !B->has;
  if (!take) {
    const volatile BestRec* vb = B;
    if (ev.objective != vb->obj) take = ev.objective > vb->obj;
    else if (ev.total_sl != vb->sl) take = ev.total_sl < vb->sl;
    else {
      uint16_t cb[MAXT];
      for (int k = 0; k < T; ++k) cb[k] = vb->choice[k];
      take = fo_cmp_m(s, probe, ch, cb) < 0;
    }
  }
  if (take) {
    B->has = 1;
    B->found = 1;
    B->obj = ev.objective;
    B->sl = ev.total_sl;
    for (int k = 0; k < T; ++k) B->choice[k] = ch[k];
  }
  atomicAdd(&B->leaves, 1ull);
  atomicAdd(&B->nodes, 1ull);  // (stats.nodes: candidates evaluated one by one)
  spin_unlock(&B->lock);
}

int launch_fanout_prep(const FoArgs& a, cudaStream_t st) {
  PROF_BEGIN(K_FO_PREP);
  k_fo_prep<<<(unsigned)(a.s.n_probes * a.P0max), 256, 0, st>>>(a);
  PROF_END();
  return 1;
}

int launch_fanout_tau(const FoArgs& a, double delta, cudaStream_t st) {
  k_fo_tau<<<a.s.n_probes, 256, 0, st>>>(a, delta);
  return 1;
}

int launch_fanout_round(const FoArgs& a, long long* n_cand_host, cudaStream_t st) {
  cudaMemsetAsync(a.ncand, 0, sizeof(unsigned long long), st);
  const long long work = (long long)a.s.n_probes * a.P0max * (a.SB + 1);
  PROF_BEGIN(K_FO_ENUM);
  k_fo_enum<<<(unsigned)((work + FO_ENUM_THREADS - 1) / FO_ENUM_THREADS), FO_ENUM_THREADS, 0, st>>>(a);
  PROF_END();
  unsigned long long nc = 0;
  cudaMemcpyAsync(&nc, a.ncand, sizeof(nc), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  int ovf = 0;
  cudaMemcpy(&ovf, a.overflow, sizeof(int), cudaMemcpyDeviceToHost);
  if (ovf) {
    *n_cand_host = -1;
    return 3;
  }
  *n_cand_host = (long long)nc;
  if (nc > 0) {
    PROF_BEGIN(K_FO_EVAL);
    k_fo_eval<<<(unsigned)((nc + 127) / 128), 128, 0, st>>>(a, (long long)nc);
    PROF_END();
  }
  return 3;
}
