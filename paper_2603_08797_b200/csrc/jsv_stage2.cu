// jsv_stage2.cu -- Stage 2 on sm_100a: exact search over the Stage-1 pools.
//
// Replaces reference planner.py:731-912 (_Search), 243-361 (derive +
// validate at every leaf) and 973-1110 (plan_uninformed's per-task argmax).
//
// The reference explores a depth-first branch-and-bound tree over tasks in
// topological order.  Here the same tree is expanded level-synchronously: a
// work item is (surviving prefix, pool bundle) and applies exactly the
// reference's filters in its order (throughput, resources, partial-path
// latency, accuracy upper bound, objective bound against the incumbent).
// Leaves are derived from scratch and validated in the reference's float
// order, then folded into a per-probe lexicographic reduction
//   (objective desc, total slices asc, m asc)                 full plans
//   (first leaf in DFS order)                                  feasible_only
// which equals the reference's answer because every filter is admissible and
// ties are broken on the canonical m.  For an
// infeasible plan there is no incumbent, so the set of visited prefixes is
// order-independent and the diagnostic re-run reproduces the reference's kill
// counts, deepest blocked level and last failed leaf (H5).
#include <cub/block/block_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>
#include <algorithm>
#include "jsv_internal.cuh"
#include "jsv_kernels.h"

__global__ void k_s2_prep(const __grid_constant__ S2Args a, double* min_lat2, int* min_sl, double* acc_ub, int* future,
                          const double* s1_lat2, const int* s1_sl, const double* s1_acc) {
  const int probe = blockIdx.x * blockDim.x + threadIdx.x;
  if (probe >= a.n_probes) return;
  const DGraph& g = *a.g;
  const DProbe& pr = a.probes[probe];
  const int T = a.T;
  for (int t = 0; t < T; ++t) {
    const int job = probe * T + t;
    const bool cz = (pr.could_zero >> t) & 1u;
    min_lat2[job] = cz ? 0.0 : s1_lat2[job];
    min_sl[job] = cz ? 0 : s1_sl[job];
    acc_ub[job] = cz ? 1.0 : s1_acc[job];
  }
  int* fut = future + probe * (T + 1);
  fut[T] = 0;
  for (int i = T - 1; i >= 0; --i) fut[i] = fut[i + 1] + min_sl[probe * T + g.topo[i]];
  BestRec* B = a.best + probe;
  B->lock = 0;
  B->has = 0;
  B->found = 0;
  B->has_leaf = 0;
  B->deepest = -1;
  for (int i = 0; i < MAXT; ++i)
    for (int k = 0; k < 5; ++k) B->kills[i][k] = 0;
  B->nodes = 0;
  B->leaves = 0;
  B->live = 0;
}

#include "jsv_s2common.cuh"

#include "jsv_search.cuh"


__device__ void write_config(const FinArgs& a, int probe, const uint16_t* cb_task,
                             jsv_plan_out& o) {
  const DGraph& g = *a.g;
  const int T = a.T;
  double lat[MAXT], cap[MAXT], acc[MAXT], fan[MAXE];
  int sl[MAXT];
  uint32_t present = 0;
  for (int u = 0; u < T; ++u) {
    const int c = cb_task[u];
    const int job = probe * T + u;
    const int outd = g.succ_off[u + 1] - g.succ_off[u];
    o.n_items[u] = 0;
    if (c == NONE16) {
      lat[u] = 0.0; cap[u] = 0.0; acc[u] = 1.0; sl[u] = 0;
      for (int j = 0; j < outd; ++j) fan[g.succ_off[u] + j] = 0.0;
      continue;
    }
    const long long q = (long long)job * a.W + c;
    lat[u] = a.p_lat[q]; cap[u] = a.p_cap[q]; acc[u] = a.p_acc[q]; sl[u] = a.p_sl[q];
    for (int j = 0; j < outd; ++j) fan[g.succ_off[u] + j] = a.p_fan[q * a.maxout + j];
    present |= 1u << u;
    const long long cand = (long long)probe * a.C_probe + a.task_base[u] + a.pool_cand[q];
    const int n = a.nitems[cand];
    o.n_items[u] = n;
    const int kb = g.key_off[u];
    for (int k = 0; k < n; ++k) {
      const uint32_t w = a.items[cand * a.maxi + k];
      o.items[u][k] = w;
      o.hput[u][k] = (double)(w & 0xFFFFu) * a.tb.key_thr[kb + (w >> 16)];
    }
  }
  EvalOut ev;
  evaluate<true>(g, *a.rq, a.probes[probe], lat, cap, acc, sl, fan, present, ev, o.lat_margin,
                 o.thr_margin, &o.res_margin, &o.acc_margin);
  for (int u = 0; u < T; ++u) {
    o.latency[u] = lat[u];
    o.capacity[u] = cap[u];
    o.accuracy[u] = acc[u];
    o.slices[u] = sl[u];
    o.demand[u] = ev.dem[u];
  }
  for (int e = 0; e < g.E; ++e) o.fanout[e] = ev.fan[e];
  for (int p = 0; p < g.P; ++p) {
    double prod = 1.0;
    for (int k = g.path_off[p]; k < g.path_off[p + 1]; ++k) prod *= acc[g.path_task[k]];
    o.path_acc[p] = prod;
  }
  o.total_slices = ev.total_sl;
  o.a_obj = ev.a_obj;
  o.objective = ev.objective;
  o.uncovered_mask = ev.uncovered;
  o.has_config = 1;
  o.feasible = ev.feasible ? 1 : 0;
  o.binding = ev.first_fail;
}

__device__ int binding_from_kills(const int* k) {
  int best = 0;
  for (int n = 1; n < 5; ++n)
    if (k[n] > k[best]) best = n;
  return k[best] ? best : JSV_BIND_THROUGHPUT;
}

__global__ void k_finalize(const __grid_constant__ FinArgs a) {
  const int probe = blockIdx.x * blockDim.x + threadIdx.x;
  if (probe >= a.n_probes) return;
  const DGraph& g = *a.g;
  const int T = a.T;
  jsv_plan_out& o = a.out[probe];
  o.has_config = 0;
  o.feasible = 0;
  o.binding = JSV_BIND_THROUGHPUT;
  o.objective = 0.0;
  o.a_obj = 0.0;
  o.dead = a.dead[probe];
  for (int t = 0; t < T; ++t) {
    o.pool_size[t] = a.pool_n[probe * T + t];
    o.truncated[t] = a.pool_trunc[probe * T + t];
    o.pool_present[t] = 1;
  }
  const BestRec& B = a.best[probe];
  o.nodes = (long long)B.nodes;
  o.leaves = (long long)B.leaves;
  if (a.uninformed) {
    uint16_t cb[MAXT];
    for (int t = 0; t < T; ++t) cb[t] = NONE16;
    for (int i = 0; i < T; ++i) {
      const int t = g.topo[i];
      const int pk = a.pick[probe * T + t];
      if (pk == -2) continue;  // demand_star == 0: no instances
      if (pk < 0) {
        for (int k = i + 1; k < T; ++k) o.pool_present[g.topo[k]] = 0;
        o.binding = binding_from_kills(a.uni_kills + (probe * T + t) * 5);
        return;
      }
      cb[t] = (uint16_t)pk;
    }
    write_config(a, probe, cb, o);
    if (o.feasible) o.binding = JSV_BIND_NONE;
    return;
  }
  if (o.dead) {
    o.binding = JSV_BIND_RESOURCES;
    return;
  }
  if (B.has) {
    uint16_t cb[MAXT];
    for (int u = 0; u < T; ++u) cb[u] = B.choice[g.pos_of[u]];
    write_config(a, probe, cb, o);
    o.binding = JSV_BIND_NONE;
    return;
  }
  if (B.deepest >= 0) {
    o.binding = binding_from_kills(B.kills[B.deepest]);
  } else if (B.has_leaf) {
    uint16_t cb[MAXT];
    for (int u = 0; u < T; ++u) cb[u] = B.leaf_choice[g.pos_of[u]];
    jsv_plan_out tmp;
    write_config(a, probe, cb, tmp);
    o.binding = tmp.binding < 0 ? JSV_BIND_THROUGHPUT : tmp.binding;
  } else {
    o.binding = JSV_BIND_THROUGHPUT;
  }
  o.has_config = 0;
  o.feasible = 0;
}

int launch_finalize(const FinArgs& a, cudaStream_t st) {
  PROF_BEGIN(K_FINALIZE);
  // one thread per probe, spread over the SMs: each thread writes its ~5 KB
  // record with scattered stores, so few lanes per SM keep the LSUs from
  // serialising (64 probes: 64 one-thread blocks)
  int tpb = 1;
  while (tpb * 148 < a.n_probes && tpb < 64) tpb <<= 1;
  k_finalize<<<(a.n_probes + tpb - 1) / tpb, tpb, 0, st>>>(a);
  PROF_END();
  return 1;
}

// ------------------------------------------------------- plan_uninformed picks

// One block per (probe, task): exact per-task filters + argmax of
// (alpha*w_t*acc - beta*s, -s), ties on items (planner.py:1064-1100).
__global__ void __launch_bounds__(256) k_uni_pick(const __grid_constant__ S2Args a, FinArgs f, int* pick, int* kills) {
  __shared__ int sk[5];
  __shared__ double s_score[256];
  __shared__ int s_sl[256];
  __shared__ int s_idx[256];
  const int job = blockIdx.x;
  const int probe = job / a.T, t = job % a.T;
  const DProbe& pr = a.probes[probe];
  const DReq& rq = *a.rq;
  if (threadIdx.x < 5) sk[threadIdx.x] = 0;
  if (pr.star[t] == 0.0) {
    if (threadIdx.x == 0) {
      pick[job] = -2;
      for (int k = 0; k < 5; ++k) kills[job * 5 + k] = 0;
    }
    return;
  }
  __syncthreads();
  const double need = pr.star[t] * (1.0 + rq.slack);
  const int P = a.pool_n[job];
  const double wa = pr.alpha * pr.weight[t];
  double bscore = 0.0;
  int bsl = 0, bidx = -1;
  const long long cbase = (long long)probe * f.C_probe + f.task_base[t];
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    const long long q = (long long)job * a.W + k;
    int why = -1;
    if (a.p_cap[q] < need) why = JSV_BIND_THROUGHPUT;
    else if (2.0 * a.p_lat[q] > pr.lat_budget[t]) why = JSV_BIND_LATENCY;
    else if ((double)a.p_sl[q] > pr.slice_budget[t]) why = JSV_BIND_RESOURCES;
    else if (a.p_acc[q] < pr.floor_[t]) why = JSV_BIND_ACCURACY;
    if (why >= 0) {
      atomicAdd(&sk[why], 1);
      continue;
    }
    const double score = wa * a.p_acc[q] - pr.beta * (double)a.p_sl[q];
    bool better;
    if (bidx < 0) better = true;
    else if (score != bscore) better = score > bscore;
    else if (a.p_sl[q] != bsl) better = a.p_sl[q] < bsl;
    else {
      const long long c1 = cbase + f.pool_cand[q], c2 = cbase + f.pool_cand[(long long)job * a.W + bidx];
      const int n1 = f.nitems[c1], n2 = f.nitems[c2];
      int r = 0;
      for (int i = 0; i < (n1 < n2 ? n1 : n2) && r == 0; ++i) {
        uint32_t x = f.items[c1 * f.maxi + i], y = f.items[c2 * f.maxi + i];
        if (x != y) r = x < y ? -1 : 1;
      }
      if (r == 0) r = n1 < n2 ? -1 : (n1 > n2 ? 1 : 0);
      better = r < 0;
    }
    if (better) { bscore = score; bsl = a.p_sl[q]; bidx = k; }
  }
  s_score[threadIdx.x] = bscore;
  s_sl[threadIdx.x] = bsl;
  s_idx[threadIdx.x] = bidx;
  __syncthreads();
  if (threadIdx.x == 0) {
    int bi = -1;
    double bs = 0.0;
    int bl = 0;
    for (int x = 0; x < blockDim.x; ++x) {
      const int k = s_idx[x];
      if (k < 0) continue;
      bool better;
      if (bi < 0) better = true;
      else if (s_score[x] != bs) better = s_score[x] > bs;
      else if (s_sl[x] != bl) better = s_sl[x] < bl;
      else {
        const long long c1 = cbase + f.pool_cand[(long long)job * a.W + k];
        const long long c2 = cbase + f.pool_cand[(long long)job * a.W + bi];
        const int n1 = f.nitems[c1], n2 = f.nitems[c2];
        int r = 0;
        for (int i = 0; i < (n1 < n2 ? n1 : n2) && r == 0; ++i) {
          uint32_t xx = f.items[c1 * f.maxi + i], yy = f.items[c2 * f.maxi + i];
          if (xx != yy) r = xx < yy ? -1 : 1;
        }
        if (r == 0) r = n1 < n2 ? -1 : (n1 > n2 ? 1 : 0);
        better = r < 0;
      }
      if (better) { bi = k; bs = s_score[x]; bl = s_sl[x]; }
    }
    pick[job] = bi;
    for (int k = 0; k < 5; ++k) kills[job * 5 + k] = sk[k];
  }
}

int launch_uninformed(const S2Args& a, const FinArgs& f, int* pick, int* kills, cudaStream_t st) {
  PROF_BEGIN(K_UNINFORMED);
  k_uni_pick<<<a.n_probes * a.T, 256, 0, st>>>(a, f, pick, kills);
  PROF_END();
  return 1;
}

// ---------------------------------------------------------- derive / validate

__global__ void k_derive(const __grid_constant__ DeriveArgs a) {
  const DGraph& g = *a.g;
  const int T = g.T;
  jsv_plan_out& o = *a.out;
  double lat[MAXT], cap[MAXT], acc[MAXT], fan[MAXE];
  int sl[MAXT];
  uint32_t present = 0;
  for (int u = 0; u < T; ++u) {
    const int n = a.n_items[u];
    Stat s;
    bundle_stats(g, a.tb, u, a.items + u * MAXI, n, s);
    lat[u] = s.lat; cap[u] = s.cap; acc[u] = s.acc; sl[u] = s.sl;
    const int outd = g.succ_off[u + 1] - g.succ_off[u];
    for (int j = 0; j < outd; ++j) fan[g.succ_off[u] + j] = s.fan[j];
    o.n_items[u] = n;
    const int kb = g.key_off[u];
    for (int k = 0; k < n; ++k) {
      const uint32_t w = a.items[u * MAXI + k];
      o.items[u][k] = w;
      o.hput[u][k] = (double)(w & 0xFFFFu) * a.tb.key_thr[kb + (w >> 16)];
    }
    if (n) present |= 1u << u;
  }
  EvalOut ev;
  evaluate<true>(g, *a.rq, *a.probe, lat, cap, acc, sl, fan, present, ev, o.lat_margin,
                 o.thr_margin, &o.res_margin, &o.acc_margin);
  for (int u = 0; u < T; ++u) {
    o.latency[u] = lat[u];
    o.capacity[u] = cap[u];
    o.accuracy[u] = acc[u];
    o.slices[u] = sl[u];
    o.demand[u] = ev.dem[u];
  }
  for (int e = 0; e < g.E; ++e) o.fanout[e] = ev.fan[e];
  for (int p = 0; p < g.P; ++p) {
    double prod = 1.0;
    for (int k = g.path_off[p]; k < g.path_off[p + 1]; ++k) prod *= acc[g.path_task[k]];
    o.path_acc[p] = prod;
  }
  o.total_slices = ev.total_sl;
  o.a_obj = ev.a_obj;
  o.objective = ev.objective;
  o.uncovered_mask = ev.uncovered;
  o.has_config = 1;
  o.feasible = ev.feasible ? 1 : 0;
  o.binding = ev.first_fail;
}

int launch_derive(const DeriveArgs& a, cudaStream_t st) {
  k_derive<<<1, 1, 0, st>>>(a);
  return 1;
}

// validate_configuration on caller-supplied fields (planner.py:329-361)
__global__ void k_validate(const __grid_constant__ ValidateArgs a) {
  const DGraph& g = *a.g;
  const DReq& rq = *a.rq;
  const DProbe& pr = *a.probe;
  jsv_plan_out& o = *a.out;
  bool ok = true;
  for (int p = 0; p < g.P; ++p) {
    PySum ps;
    for (int k = g.path_off[p]; k < g.path_off[p + 1]; ++k) ps.add(2.0 * a.lat[g.path_task[k]]);
    o.lat_margin[p] = pr.slo_eff - ps.result();
    ok = ok && o.lat_margin[p] >= 0;
  }
  for (int t = 0; t < g.T; ++t) {
    o.thr_margin[t] = a.cap[t] - a.dem[t] * (1.0 + rq.slack);
    ok = ok && o.thr_margin[t] >= 0;
  }
  o.res_margin = (double)(rq.S - a.total_sl);
  o.acc_margin = a.a_obj - pr.acc_slo;
  o.uncovered_mask = a.uncovered;
  o.feasible = ok && o.res_margin >= 0 && o.acc_margin >= 0 && a.uncovered == 0;
}

int launch_validate(const ValidateArgs& a, cudaStream_t st) {
  k_validate<<<1, 1, 0, st>>>(a);
  return 1;
}
