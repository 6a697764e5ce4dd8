// jsv_stage1.cu -- Stage 1 on sm_100a: candidate bundles per (probe, task).
//
// Replaces reference planner.py:406-635 (_tuples_for, _enumeration_size,
// _exhaustive_counts, _structured_counts, _stats_for_counts, _pareto_filter,
// _candidate_pool).  A "job" is one (probe, task) pair; all jobs of a batch run
// in the same launches:
//
//   k_generate   one thread per enumeration unit: exhaustive count vectors are
//                unranked from a suffix-ways table; structured covers and
//                2-variant mixes are decoded from the unit index.
//   k_stats      one thread per candidate: latency / capacity / slices /
//                weighted accuracy + fan-out (all-equal short circuit).
//   k_pairs_l    both skyline passes (same slices; survivors with fewer
//                slices), one thread per candidate over list-ordered
//                coordinates with a float shadow quick reject (k_pairs_a: tiled
//                form, for rows of more than 16 coordinates):
//   k_pairs_a    tiled all-pairs skyline: candidate i dies if another
//                candidate weakly dominates it with a different row, or has an
//                identical row and smaller items (the reference's dedup).  By
//                transitivity this equals the reference's sequential
//                "not dominated by an earlier kept row" filter.
//   k_compact    survivors -> frontier list.
//   k_pairs_b    frontier position (lexicographic row order) and capacity
//                rank (-cap, slices, items) by counting.
//   k_truncate   frontier order, pareto_width truncation (planner.py:574-583),
//                pool SoA + per-pool bounds for Stage 2.
//   (ties on m are resolved in Stage 2 directly on the bundles' item lists)
#include <algorithm>
#include <cstdlib>
#include <cub/block/block_scan.cuh>
#include "jsv_internal.cuh"
#include "jsv_kernels.h"

__constant__ double c_grid[N_LEVELS] = {1.0,    0.75,    0.5,       0.375,    0.25,
                                        0.1875, 0.125,   0.09375,   0.0625,   0.046875,
                                        0.03125, 0.0234375, 0.015625, 0.01171875};

// cover(i, dem) of planner.py:503-508: max(1, ceil(dem / H - 1e-12)) if it fits.
__device__ __forceinline__ int cover_count(double dem, double h, int cost, int S) {
  double q = dem / h - 1e-12;
  if (!(q <= (double)S)) return 0;
  double cq = ceil(q);
  long long c = (long long)cq;
  if (c < 1) c = 1;
  if (c * (long long)cost > S) return 0;
  return (int)c;
}

__device__ __forceinline__ long long job_base(const S1Args& a, int probe, int t) {
  return (long long)probe * a.C_probe + a.task_base[t];
}

// Slots for the m candidates of this thread in its job's slab: one atomicAdd per
// (warp, job) group instead of one per candidate (the slab counter is hot).
__device__ __forceinline__ int reserve_slots(const S1Args& a, int job, int m, bool active) {
  const unsigned full = 0xffffffffu;
  const int key = active ? job : -1;
  const unsigned grp = __match_any_sync(full, key);
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(grp) - 1;
  // exclusive prefix of m over the group's lanes below this one
  int pre = 0, tot = 0;
  unsigned g = grp;
  while (g) {
    const int l = __ffs(g) - 1;
    g &= g - 1;
    const int v = __shfl_sync(grp, m, l);
    if (l < lane) pre += v;
    tot += v;
  }
  int basepos = 0;
  if (lane == leader && active && tot > 0) basepos = atomicAdd(&a.cnt[job], tot);
  basepos = __shfl_sync(grp, basepos, leader);
  return basepos + pre;
}

__device__ __forceinline__ void store_candidate(const S1Args& a, int probe, int t, int pos,
                                                const uint32_t* it, int n) {
  if (pos >= a.task_cap[t]) {
    atomicExch(a.err, 1);
    return;
  }
  const long long c = job_base(a, probe, t) + pos;
  a.nitems[c] = n;
  for (int k = 0; k < n; ++k) a.items[c * a.maxi + k] = it[k];
}

// One enumeration unit lu of descriptor D for one probe: either one item list
// (it[0 .. n), m = 1) or m singletons / homogeneous covers of one key (key1 >= 0,
// counts[0 .. m)); m = 0: no candidate.
struct GenOut {
  uint32_t it[MAXI];
  int n, m, key1;
  int counts[N_LEVELS + 1];
};

__device__ __forceinline__ void gen_unit(const S1Args& a, int probe, const GenDesc& D, int lu,
                                         GenOut& o, const unsigned* W) {
  const DGraph& g = *a.g;
  const DReq& rq = *a.rq;
  const int t = D.task;
  const int S = rq.S;
  const int kb = g.key_off[t];
  const int* tup = a.tb.sub_key + D.key_base;
  o.n = 0;
  o.m = 0;
  o.key1 = -1;
  if (D.mode == 0) {
    // unrank count vector lu+1 (0 is the empty vector) -- _exhaustive_counts
    unsigned long long idx = (unsigned long long)lu + 1ull;
    int left = S;
    bool ok = true;
    for (int i = 0; i < D.n_tuples && ok; ++i) {
      const int cost = a.tb.key_cost[kb + tup[i]];
      int c = 0;
      while (true) {
        unsigned long long w = W[(i + 1) * (S + 1) + (left - c * cost)];
        if (idx < w) break;
        idx -= w;
        ++c;
      }
      if (c > 0) {
        if (o.n >= MAXI) { atomicExch(a.err, 2); ok = false; break; }
        o.it[o.n++] = ((uint32_t)tup[i] << 16) | (uint32_t)c;
      }
      left -= c * cost;
    }
    o.m = ok ? 1 : 0;
    return;
  }
  const DProbe& pr = a.probes[probe];
  const double target = pr.r_upper[D.a][t] * (1.0 + rq.slack);
  const bool has_lv = target > 0;
  if (lu < D.n_tuple_units) {
    // singleton + homogeneous covers of one tuple, distinct counts only
    o.key1 = tup[lu];
    const int cost = a.tb.key_cost[kb + o.key1];
    const double h = a.tb.key_thr[kb + o.key1];
    int cnt[N_LEVELS + 1];
    int mm = 0;
    if (cost <= S) cnt[mm++] = 1;
    if (has_lv) {
      for (int k = 0; k < N_LEVELS; ++k) {
        int c = cover_count(target * c_grid[k], h, cost, S);
        if (c > 0) cnt[mm++] = c;
      }
    }
    for (int x = 0; x < mm; ++x) {
      bool dup = false;
      for (int y = 0; y < o.m; ++y) dup |= o.counts[y] == cnt[x];
      if (!dup) o.counts[o.m++] = cnt[x];
    }
  } else if (has_lv) {
    // two-variant mix unit: (pair, phi, level, rep_a, rep_b)
    int mu = lu - D.n_tuple_units;
    const int per_pair = rq.n_mix * N_LEVELS * 4;
    int pi = mu / per_pair;
    int rem = mu % per_pair;
    const int rsel = rem & 3;
    rem >>= 2;
    const int lvk = rem % N_LEVELS;
    const int ph = rem / N_LEVELS;
    int ga = 0, gb = 1;
    {
      // pair index -> (ga < gb) in row-major order
      int G = D.n_groups;
      int acc = 0;
      for (ga = 0; ga < G; ++ga) {
        int cnt = G - 1 - ga;
        if (pi < acc + cnt) { gb = ga + 1 + (pi - acc); break; }
        acc += cnt;
      }
    }
    const int ia = a.tb.grp_rep[2 * (D.grp_base + ga) + (rsel & 1)];
    const int ib = a.tb.grp_rep[2 * (D.grp_base + gb) + (rsel >> 1)];
    if (ia >= 0 && ib >= 0) {
      const double phi = rq.mix[ph];
      const double lvl = target * c_grid[lvk];
      const int ka = tup[ia], kbb = tup[ib];
      const int costa = a.tb.key_cost[kb + ka], costb = a.tb.key_cost[kb + kbb];
      const int ca = cover_count(phi * lvl, a.tb.key_thr[kb + ka], costa, S);
      const int cb = cover_count((1.0 - phi) * lvl, a.tb.key_thr[kb + kbb], costb, S);
      if (ca != 0 && cb != 0 && ca * costa + cb * costb <= S) {
        o.it[0] = ((uint32_t)ka << 16) | (uint32_t)ca;
        o.it[1] = ((uint32_t)kbb << 16) | (uint32_t)cb;
        o.n = 2;
        o.m = 1;
      }
    }
  }
}

__global__ void k_generate(const __grid_constant__ S1Args a) {
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool in = gtid < (long long)a.n_probes * a.U;
  const int probe = in ? (int)(gtid / a.U) : 0;
  const int u = in ? (int)(gtid % a.U) : 0;
  // the last descriptor whose first unit is <= u (unit_off is non-decreasing):
  // binary search instead of a scan of dependent loads
  int d = 0, step = 1;
  while (step * 2 < a.n_desc) step <<= 1;
  for (; step > 0; step >>= 1)
    if (d + step < a.n_desc && a.desc[d + step].unit_off <= u) d += step;
  const GenDesc D = a.desc[d];
  const int t = D.task;
  GenOut o;
  o.m = 0;
  o.n = 0;
  o.key1 = -1;
  if (in) gen_unit(a, probe, D, u - D.unit_off, o, a.ways + D.w_off);
  const int job = probe * a.T + t;
  const int pos = reserve_slots(a, job, o.m, in);
  if (o.key1 >= 0) {
    for (int x = 0; x < o.m; ++x) {
      const uint32_t one = ((uint32_t)o.key1 << 16) | (uint32_t)o.counts[x];
      store_candidate(a, probe, t, pos + x, &one, 1);
    }
  } else if (o.m > 0) {
    store_candidate(a, probe, t, pos, o.it, o.n);
  }
}

__device__ __forceinline__ int locate_task(const S1Args& a, long long local) {
  int t = 0;
  while (t + 1 < a.T && a.task_base[t + 1] <= local) ++t;
  return t;
}

__global__ void k_stats(const __grid_constant__ S1Args a) {
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long tot = (long long)a.n_probes * a.C_probe;
  if (c >= tot) return;
  const int probe = (int)(c / a.C_probe);
  const long long local = c % a.C_probe;
  const int t = locate_task(a, local);
  const int pos = (int)(local - a.task_base[t]);
  if (pos >= a.cnt[probe * a.T + t]) return;
  const DGraph& g = *a.g;
  Stat s;
  uint32_t it[MAXI];
  const int n = a.nitems[c];
  for (int k = 0; k < n; ++k) it[k] = a.items[c * a.maxi + k];
  bundle_stats(g, a.tb, t, it, n, s);
  const int outd = g.succ_off[t + 1] - g.succ_off[t];
  a.sl[c] = s.sl;
  a.arr[0 * tot + c] = (double)s.sl;
  a.arr[1 * tot + c] = -s.cap;
  a.arr[2 * tot + c] = -s.acc;
  a.arr[3 * tot + c] = s.lat;
  for (int j = 0; j < a.D - 4; ++j) a.arr[(4 + j) * tot + c] = j < outd ? s.fan[j] : 0.0;
  a.flag[c] = 0u;
}

// Append the work items of one job: i tiles of 256, j chunks of jchunk over
// [0, jend(i0)).  Called by every thread of the block: one atomicAdd reserves
// the job's whole range, the threads write it tile by tile.  Lists the launch
// will not consume (wl_mask) are skipped.
__device__ __forceinline__ int items_of_tile(int tl, int n, int jchunk, bool triangular) {
  const int jend = triangular ? min(n, tl * 256 + 256) : n;
  return max(1, (jend + jchunk - 1) / jchunk);
}
__device__ void push_items(const S1Args& a, int k, int job, int n, int jchunk, bool triangular) {
  __shared__ int s_at;
  if (!((a.wl_mask >> k) & 1)) return;  // (block-uniform)
  const int tiles = (n + 255) / 256;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int tl = 0; tl < tiles; ++tl) tot += items_of_tile(tl, n, jchunk, triangular);
    s_at = tot ? atomicAdd(a.wn + k, tot) : 0;
  }
  __syncthreads();
  const int at = s_at;
  for (int tl = threadIdx.x; tl < tiles; tl += blockDim.x) {
    int off = 0;
    if (triangular) {
      for (int u = 0; u < tl; ++u) off += items_of_tile(u, n, jchunk, true);
    } else {
      off = tl * items_of_tile(0, n, jchunk, false);
    }
    const int nj = items_of_tile(tl, n, jchunk, triangular);
    for (int c = 0; c < nj; ++c) a.wl[k][at + off + c] = make_int4(job, tl * 256, c * jchunk, 0);
  }
}

// Counting sort of a job's candidates by slice count: order[] and bucket starts
// bstart[s] = #candidates with fewer than s slices (s = 0 .. S+1).
#define BUCKET_SMEM_MAX 12288
// (JOB_BS threads: two job blocks per SM at <= 64 registers, so a batch's
// jobs run in one wave)
#define JOB_BS 512
__global__ void __launch_bounds__(JOB_BS, 2) k_bucket(const __grid_constant__ S1Args a) {
  extern __shared__ int hist[];
  const int job = a.job_map ? a.job_map[a.job_off + blockIdx.x] : blockIdx.x;
  const int probe = job / a.T, t = job % a.T;
  const int n = a.cnt[job];
  const int NB = a.S + 2;
  const long long tot = (long long)a.n_probes * a.C_probe;
  const long long base = job_base(a, probe, t);
  int* bst = a.bstart + (long long)job * NB;
  if (NB > BUCKET_SMEM_MAX) {
    // huge budgets: identity order, every candidate scanned
    push_items(a, 0, job, n, 1024, false);
    for (int s = threadIdx.x; s < NB; s += blockDim.x) bst[s] = (s == 0) ? 0 : n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      a.order[base + i] = i;
      for (int d = 0; d < a.D; ++d) a.arrl[d * tot + base + i] = a.arr[d * tot + base + i];
    }
    return;
  }
  for (int s = threadIdx.x; s < NB; s += blockDim.x) hist[s] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    atomicAdd(&hist[(int)a.arr[base + i] + 1], 1);  // arr[0] = slices
  __syncthreads();
  {
    // inclusive block scan of the bucket counts, JOB_BS buckets per step (840-slice
    // budgets: 842 buckets -- a thread-0 loop was most of this kernel there)
    typedef cub::BlockScan<int, JOB_BS> BScan;
    __shared__ typename BScan::TempStorage btmp;
    __shared__ int bcarry;
    if (threadIdx.x == 0) bcarry = 0;
    __syncthreads();
    for (int s0 = 0; s0 < NB; s0 += JOB_BS) {
      const int s = s0 + threadIdx.x;
      const int v = s < NB ? hist[s] : 0;
      int inc, total;
      BScan(btmp).InclusiveSum(v, inc, total);
      const int c0 = bcarry;
      if (s < NB) {
        hist[s] = c0 + inc;
        bst[s] = c0 + inc;
      }
      __syncthreads();
      if (threadIdx.x == 0) bcarry = c0 + total;
      __syncthreads();
    }
  }
  // same-bucket pass items: j chunks of 1024 (a tile's bucket range can be long)
  push_items(a, 0, job, n, 1024, false);
  __syncthreads();
  // hist[s] is now the start of bucket s; scatter (order inside a bucket is irrelevant)
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int s = (int)a.arr[base + i];
    const int pos = atomicAdd(&hist[s], 1);
    a.order[base + pos] = i;
    for (int d = 0; d < a.D; ++d) a.arrl[d * tot + base + pos] = a.arr[d * tot + base + i];
    // float shadow of coordinates 1..4 (the same-slices pass's quick reject)
    if (a.D >= 5)
      a.arrf[base + pos] = make_float4((float)a.arr[1 * tot + base + i], (float)a.arr[2 * tot + base + i],
                                       (float)a.arr[3 * tot + base + i], (float)a.arr[4 * tot + base + i]);
  }
}

// items(c1) < items(c2) lexicographically over ((key, count), ...) tuples
__device__ __forceinline__ int cmp_items(const S1Args& a, long long c1, long long c2) {
  const int n1 = a.nitems[c1], n2 = a.nitems[c2];
  const int n = n1 < n2 ? n1 : n2;
  for (int k = 0; k < n; ++k) {
    uint32_t x = a.items[c1 * a.maxi + k], y = a.items[c2 * a.maxi + k];
    if (x != y) return x < y ? -1 : 1;
  }
  return n1 < n2 ? -1 : (n1 > n2 ? 1 : 0);
}

#define TJ 128

// Skyline test in two passes (the dominance relation is transitive, so a
// candidate is dominated iff some skyline candidate dominates it):
//   mode 0  every candidate against the candidates of its own slices bucket
//           (>90% of dominated candidates have a same-slices dominator);
//   mode 1  the survivors of mode 0 against the survivors with fewer slices.
// A candidate dies if another weakly dominates it with a different row, or has
// an identical row and smaller items (the reference's dedup); by transitivity
// this equals the reference's sequential "not dominated by an earlier kept
// row" filter.  i runs over the slices-sorted list so a block's candidates
// have similar slices and the j range a block stages in shared memory is short.
template <int D>
__device__ __forceinline__ void pairs_a_tile(const S1Args& a, int job, int i0, int j0, int jchunk,
                                             int mode, double* sh, int* shj, int& s_lo, int& s_hi) {
  const int probe = job / a.T, t = job % a.T;
  const int n = mode == 0 ? a.cnt[job] : a.scnt[job];
  if (i0 >= n || j0 >= n) return;  // (block-uniform)
  const long long tot = (long long)a.n_probes * a.C_probe;
  const long long base = job_base(a, probe, t);
  const int* list = (mode == 0 ? a.order : a.surv) + base;
  const int* bst = a.bstart + (long long)job * (a.S + 2);
  const int* sbst = a.sbst + (long long)job * (a.S + 2);
  const bool act = i0 + (int)threadIdx.x < n;
  const int i = act ? list[i0 + threadIdx.x] : 0;
  double xi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) xi[d] = act ? a.arr[d * tot + base + i] : 0.0;
  int lo_i = 0, hi_i = 0;
  if (act) {
    const int si = (int)xi[0];
    if (mode == 0) {
      lo_i = bst[si];
      hi_i = bst[si + 1];
    } else {
      hi_i = sbst[si];
    }
  }
  if (threadIdx.x == 0) {
    s_lo = 0x7FFFFFFF;
    s_hi = 0;
  }
  __syncthreads();
  if (act && hi_i > lo_i) {
    atomicMin(&s_lo, lo_i);
    atomicMax(&s_hi, hi_i);
  }
  __syncthreads();
  const int jbeg = max(j0, s_lo);
  const int j1 = min(min(n, j0 + jchunk), s_hi);
  unsigned fl = 0;
  for (int jt = jbeg; jt < j1; jt += TJ) {
    const int nj = min(TJ, j1 - jt);
    for (int x = threadIdx.x; x < TJ; x += blockDim.x) shj[x] = x < nj ? list[jt + x] : 0;
    __syncthreads();
    for (int x = threadIdx.x; x < D * TJ; x += blockDim.x) {
      int d = x / TJ, jj = x % TJ;
      sh[x] = jj < nj ? a.arr[d * tot + base + shj[jj]] : 0.0;
    }
    __syncthreads();
    if (act && !fl) {
      const int jlo = max(0, lo_i - jt), jhi = min(nj, hi_i - jt);
      for (int jj = jlo; jj < jhi; ++jj) {
        bool le = true, eq = true;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          double xj = sh[d * TJ + jj];
          le = le && (xj <= xi[d]);
          eq = eq && (xj == xi[d]);
        }
        if (le) {
          if (!eq) {
            fl |= 1u;
            break;
          }
          const int j = shj[jj];
          if (j != i) {
            int c = cmp_items(a, base + j, base + i);
            if (c < 0 || (c == 0 && j < i)) {
              fl |= 2u;
              break;
            }
          }
        }
      }
    }
    __syncthreads();
  }
  if (act && fl) atomicOr(&a.flag[base + i], fl);
}

// Work items {job, i0, j0} of a pass come from a device list built by the
// kernel that knew the job's count (k_bucket / k_surv / k_compact), so no block
// is launched for the empty tail of a job's candidate capacity.
template <int D>
__global__ void __launch_bounds__(256) k_pairs_a(const __grid_constant__ S1Args a,
                                                 const int4* items, const int* n_items, int jchunk,
                                                 int mode) {
  __shared__ double sh[D * TJ];
  __shared__ int shj[TJ];
  __shared__ int s_lo, s_hi;
  const int nw = *n_items;
  for (int w = blockIdx.x; w < nw; w += gridDim.x) {
    const int4 it = items[w];
    pairs_a_tile<D>(a, it.x, it.y, it.z, jchunk, mode, sh, shj, s_lo, s_hi);
    __syncthreads();
  }
}

// The same skyline test without shared-memory staging or barriers: one thread
// per list position i scans its own j range straight from the list-ordered
// coordinates (arrl, L1-resident).  Lanes of a warp hold neighbouring list
// positions -- the same or adjacent slices buckets -- so they read the same j
// in step (broadcast loads) and each leaves its loop at its first dominator.
template <int D, bool SKIP0>
__global__ void __launch_bounds__(256) k_pairs_l(const __grid_constant__ S1Args a, int mode) {
  const long long tot = (long long)a.n_probes * a.C_probe;
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= tot) return;
  const int probe = (int)(gid / a.C_probe);
  const long long local = gid % a.C_probe;
  const int t = locate_task(a, local);
  const int p = (int)(local - a.task_base[t]);
  const int job = probe * a.T + t;
  const int n = mode == 0 ? a.cnt[job] : a.scnt[job];
  if (p >= n) return;
  const long long base = job_base(a, probe, t);
  const double* __restrict__ xl = a.arrl + base;
  double xi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) xi[d] = xl[d * tot + p];
  const int si = (int)xi[0];
  int lo, hi;
  if (mode == 0) {
    const int* bst = a.bstart + (long long)job * (a.S + 2);
    lo = bst[si];
    hi = bst[si + 1];
  } else {
    lo = 0;
    hi = a.sbst[(long long)job * (a.S + 2) + si];
  }
  const int* list = (mode == 0 ? a.order : a.surv) + base;
  // quick reject on the float shadow: rounding to float is monotone, so
  // float(x_j) > float(x_i) in any coordinate proves x_j > x_i there (j cannot
  // dominate i); otherwise the exact double test below decides
  constexpr bool FQ = SKIP0 && D >= 5;
  float4 fi = make_float4(0.f, 0.f, 0.f, 0.f);
  if (FQ) fi = a.arrf[base + p];
  unsigned fl = 0;
  // exact weak-dominance / dedup test of j against i; true when i dies
  auto exact = [&](int j) -> bool {
    bool le = true, eq = true;
    // (SKIP0: a same-slices bucket -- coordinate 0 is equal for every j)
#pragma unroll
    for (int d = SKIP0 ? 1 : 0; d < D; ++d) {
      const double xj = xl[d * tot + j];
      le = le && (xj <= xi[d]);
      eq = eq && (xj == xi[d]);
    }
    if (!le) return false;
    // (survivors pass: j has fewer slices, so its row differs from i's)
    if (!eq || (SKIP0 && mode != 0)) {
      fl = 1u;
      return true;
    }
    if (j != p) {
      const int ci = list[p], cj = list[j];
      const int c = cmp_items(a, base + cj, base + ci);
      if (c < 0 || (c == 0 && cj < ci)) {
        fl = 2u;
        return true;
      }
    }
    return false;
  };
  constexpr int XJ = 8;
  if (FQ) {
    // XJ shadow loads in flight per step; the j's that survive the quick
    // reject get the exact test, in j order
    bool dead = false;
    for (int j = lo; j < hi && !dead; j += XJ) {
      unsigned keep = 0;
#pragma unroll
      for (int u = 0; u < XJ; ++u) {
        if (j + u < hi) {
          const float4 fj = a.arrf[base + j + u];
          const bool rej = (fj.x > fi.x) | (fj.y > fi.y) | (fj.z > fi.z) | (fj.w > fi.w);
          keep |= (rej ? 0u : 1u) << u;
        }
      }
      while (keep && !dead) {
        const int u = __ffs(keep) - 1;
        keep &= keep - 1;
        dead = exact(j + u);
      }
    }
  } else {
    for (int j = lo; j < hi; ++j)
      if (exact(j)) break;
  }
  if (fl) atomicOr(&a.flag[base + list[p]], fl);
}

// Survivors of the same-bucket pass, in slices order, and their bucket starts
// sbst[s] = #survivors with fewer than s slices.
#define SURV_KC 24
#define JOB_W (JOB_BS / 32)
__device__ __forceinline__ void surv_write(const S1Args& a, long long base, long long tot, int pos, int i) {
  a.surv[base + pos] = i;
  for (int d = 0; d < a.D; ++d) a.arrl[d * tot + base + pos] = a.arr[d * tot + base + i];
  if (a.D >= 5)
    a.arrf[base + pos] = make_float4((float)a.arr[1 * tot + base + i], (float)a.arr[2 * tot + base + i],
                                     (float)a.arr[3 * tot + base + i], (float)a.arr[4 * tot + base + i]);
}

__global__ void __launch_bounds__(JOB_BS, 2) k_surv(const __grid_constant__ S1Args a) {
  typedef cub::BlockScan<int, JOB_BS> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  __shared__ int woff[SURV_KC * JOB_W];
  const int job = blockIdx.x;
  const int probe = job / a.T, t = job % a.T;
  const int n = a.cnt[job];
  const long long base = job_base(a, probe, t);
  const long long tot = (long long)a.n_probes * a.C_probe;
  const int* order = a.order + base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (n <= SURV_KC * JOB_BS) {
    // every chunk's list entries and flags loaded up front (no load latency
    // between chunks), survivor offsets from per-(chunk, warp) ballot counts
    // and ONE block scan over them
    unsigned bal[SURV_KC];
#pragma unroll
    for (int c = 0; c < SURV_KC; ++c) {
      const int p = c * JOB_BS + threadIdx.x;
      const bool alive = p < n && a.flag[base + order[p]] == 0u;
      bal[c] = __ballot_sync(0xffffffffu, alive);
    }
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < SURV_KC; ++c) woff[c * JOB_W + warp] = __popc(bal[c]);
    }
    __syncthreads();
    // (c, warp) slots in list order: chunk-major, warp-minor
    const int x = threadIdx.x < SURV_KC * JOB_W ? woff[threadIdx.x] : 0;
    int xo, total;
    Scan(tmp).ExclusiveSum(x, xo, total);
    __syncthreads();
    if (threadIdx.x < SURV_KC * JOB_W) woff[threadIdx.x] = xo;
    if (threadIdx.x == 0) carry = total;
    __syncthreads();
    const unsigned below = (1u << lane) - 1u;
#pragma unroll
    for (int c = 0; c < SURV_KC; ++c) {
      const int p = c * JOB_BS + threadIdx.x;
      if (p < n) {
        const int pos = woff[c * JOB_W + warp] + __popc(bal[c] & below);
        a.pcnt[base + p] = pos;
        if ((bal[c] >> lane) & 1u) surv_write(a, base, tot, pos, order[p]);
      }
    }
  } else {
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int s0 = 0; s0 < n; s0 += JOB_BS) {
      const int p = s0 + threadIdx.x;
      const int i = p < n ? order[p] : 0;
      const int alive = (p < n && a.flag[base + i] == 0u) ? 1 : 0;
      int off, total;
      Scan(tmp).ExclusiveSum(alive, off, total);
      if (p < n) a.pcnt[base + p] = carry + off;
      if (alive) surv_write(a, base, tot, carry + off, i);
      __syncthreads();
      if (threadIdx.x == 0) carry += total;
      __syncthreads();
    }
  }
  __syncthreads();
  const int total = carry;
  const int NB = a.S + 2;
  const int* bst = a.bstart + (long long)job * NB;
  int* sb = a.sbst + (long long)job * NB;
  for (int s = threadIdx.x; s < NB; s += blockDim.x) sb[s] = bst[s] >= n ? total : a.pcnt[base + bst[s]];
  if (threadIdx.x == 0) a.scnt[job] = total;
  // survivors with fewer slices precede i in the list: j < i0 + 256
  push_items(a, 1, job, total, 1024, true);
}

__global__ void __launch_bounds__(JOB_BS, 2) k_compact(const __grid_constant__ S1Args a) {
  typedef cub::BlockScan<int, JOB_BS> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  __shared__ int woff[SURV_KC * JOB_W];
  const int job = blockIdx.x;
  const int probe = job / a.T, t = job % a.T;
  const int n = a.cnt[job];
  const long long base = job_base(a, probe, t);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (n <= SURV_KC * JOB_BS) {
    // every chunk's flags loaded up front; offsets from ballot counts and one
    // block scan (as k_surv)
    unsigned bal[SURV_KC];
#pragma unroll
    for (int c = 0; c < SURV_KC; ++c) {
      const int i = c * JOB_BS + threadIdx.x;
      bal[c] = __ballot_sync(0xffffffffu, i < n && a.flag[base + i] == 0u);
    }
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < SURV_KC; ++c) woff[c * JOB_W + warp] = __popc(bal[c]);
    }
    __syncthreads();
    const int x = threadIdx.x < SURV_KC * JOB_W ? woff[threadIdx.x] : 0;
    int xo, total;
    Scan(tmp).ExclusiveSum(x, xo, total);
    __syncthreads();
    if (threadIdx.x < SURV_KC * JOB_W) woff[threadIdx.x] = xo;
    if (threadIdx.x == 0) carry = total;
    __syncthreads();
    const unsigned below = (1u << lane) - 1u;
#pragma unroll
    for (int c = 0; c < SURV_KC; ++c) {
      if ((bal[c] >> lane) & 1u) {
        const int pos = woff[c * JOB_W + warp] + __popc(bal[c] & below);
        a.front[base + pos] = c * JOB_BS + threadIdx.x;
        a.fpos[base + pos] = 0;
        a.fcr[base + pos] = 0;
      }
    }
  } else {
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int s0 = 0; s0 < n; s0 += JOB_BS) {
      int i = s0 + threadIdx.x;
      int alive = (i < n && a.flag[base + i] == 0u) ? 1 : 0;
      int off, total;
      Scan(tmp).ExclusiveSum(alive, off, total);
      if (alive) {
        a.front[base + carry + off] = i;
        a.fpos[base + carry + off] = 0;
        a.fcr[base + carry + off] = 0;
      }
      __syncthreads();
      if (threadIdx.x == 0) carry += total;
      __syncthreads();
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) a.fcnt[job] = carry;
  push_items(a, 2, job, carry, 1024, false);
}

// Frontier order and capacity ranks by sorting instead of counting (jobs whose
// frontier has at most FSORT_MAX bundles and finite coordinates; the others keep
// k_pairs_b's pair counts).  One block per job, bitonic sort of frontier
// indices in shared memory: (1) by the row, lexicographically -- rows are
// distinct here, so a bundle's sorted rank is the number of rows below it, the
// position k_pairs_b counts (planner.py:556-559); (2) when the frontier will be
// truncated, by (-capacity, slices, items) (planner.py:576), distinct keys too.
#define FSORT_MAX 2048
template <int D>
__global__ void __launch_bounds__(512) k_front_sort(const __grid_constant__ S1Args a) {
  extern __shared__ __align__(16) unsigned char fs_smem[];
  __shared__ int s_ok;
  const int job = blockIdx.x;
  const int probe = job / a.T, t = job % a.T;
  const int F = a.fcnt[job];
  const long long tot = (long long)a.n_probes * a.C_probe;
  const long long base = job_base(a, probe, t);
  // (rows of 16 coordinates: half the frontier fits the shared-memory keys)
  constexpr int FMAX = D <= 12 ? FSORT_MAX : FSORT_MAX / 2;
  if (F > FMAX || F == 0) {
    if (threadIdx.x == 0) a.fsorted[job] = 0;
    return;
  }
  int F2 = 1;
  while (F2 < F) F2 <<= 1;
  double* key = reinterpret_cast<double*>(fs_smem);  // [D][F2]
  int* ix = reinterpret_cast<int*>(key + D * F2);
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  for (int k = threadIdx.x; k < F2; k += blockDim.x) {
    ix[k] = k;
    if (k < F) {
      const int c = a.front[base + k];
      for (int d = 0; d < D; ++d) {
        const double v = a.arr[d * tot + base + c];
        if (!isfinite(v)) s_ok = 0;
        key[d * F2 + k] = v;
      }
    } else {
      for (int d = 0; d < D; ++d) key[d * F2 + k] = INFINITY;
    }
  }
  __syncthreads();
  if (!s_ok) {
    if (threadIdx.x == 0) a.fsorted[job] = 0;
    return;
  }
  // sort 1: rows, lexicographic (padding rows +inf, ties by index)
  for (int kk = 2; kk <= F2; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < F2; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const int x = ix[i], y = ix[l];
          int c = 0;
#pragma unroll
          for (int d = 0; d < D; ++d) {
            if (c == 0) {
              const double u = key[d * F2 + x], v = key[d * F2 + y];
              c = u < v ? -1 : (u > v ? 1 : 0);
            }
          }
          if (c == 0) c = x < y ? -1 : 1;
          const bool up = (i & kk) == 0;
          if ((c > 0) == up) {
            ix[i] = y;
            ix[l] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int r = threadIdx.x; r < F; r += blockDim.x) a.fpos[base + ix[r]] = r;
  if (F > a.W) {
    __syncthreads();
    for (int k = threadIdx.x; k < F2; k += blockDim.x) ix[k] = k;
    __syncthreads();
    // sort 2: (-capacity, slices, items); padding -capacity = +inf
    for (int kk = 2; kk <= F2; kk <<= 1) {
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < F2; i += blockDim.x) {
          const int l = i ^ j;
          if (l > i) {
            const int x = ix[i], y = ix[l];
            const double cx = key[1 * F2 + x], cy = key[1 * F2 + y];
            int c;
            if (cx != cy) c = cx < cy ? -1 : 1;
            else if (x >= F || y >= F) c = x < y ? -1 : 1;
            else if (key[x] != key[y]) c = key[x] < key[y] ? -1 : 1;
            else c = cmp_items(a, base + a.front[base + x], base + a.front[base + y]);
            if (c == 0) c = x < y ? -1 : 1;
            const bool up = (i & kk) == 0;
            if ((c > 0) == up) {
              ix[i] = y;
              ix[l] = x;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int r = threadIdx.x; r < F; r += blockDim.x) a.fcr[base + ix[r]] = r;
  }
  if (threadIdx.x == 0) a.fsorted[job] = 1;
}

template <int D>
__device__ __forceinline__ void pairs_b_tile(const S1Args& a, int job, int i0, int j0, int jchunk,
                                             double* sh, int* shc) {
  const int probe = job / a.T, t = job % a.T;
  if (a.fsorted[job]) return;  // ranks already computed by k_front_sort
  const int F = a.fcnt[job];
  if (i0 >= F || j0 >= F) return;  // (block-uniform)
  const int j1 = min(F, j0 + jchunk);
  const bool need_cap = F > a.W;
  const long long tot = (long long)a.n_probes * a.C_probe;
  const long long base = job_base(a, probe, t);
  const int i = i0 + threadIdx.x;
  const bool act = i < F;
  const int ci = act ? a.front[base + i] : 0;
  double xi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) xi[d] = act ? a.arr[d * tot + base + ci] : 0.0;
  int pos = 0, cr = 0;
  for (int jt = j0; jt < j1; jt += TJ) {
    const int nj = min(TJ, j1 - jt);
    for (int x = threadIdx.x; x < TJ; x += blockDim.x) shc[x] = x < nj ? a.front[base + jt + x] : 0;
    __syncthreads();
    for (int x = threadIdx.x; x < D * TJ; x += blockDim.x) {
      int d = x / TJ, jj = x % TJ;
      sh[x] = jj < nj ? a.arr[d * tot + base + shc[jj]] : 0.0;
    }
    __syncthreads();
    if (act) {
      for (int jj = 0; jj < nj; ++jj) {
        // lexicographic row order (planner.py:556-559; rows are distinct here)
        int lt = 0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          double xj = sh[d * TJ + jj];
          if (lt == 0) {
            if (xj < xi[d]) lt = 1;
            else if (xj > xi[d]) lt = -1;
          }
        }
        pos += lt == 1;
        if (need_cap) {
          // (-capacity, slices, items) order (planner.py:576)
          double cj = sh[1 * TJ + jj], c0 = xi[1];
          bool less;
          if (cj != c0) less = cj < c0;
          else if (sh[jj] != xi[0]) less = sh[jj] < xi[0];
          else less = cmp_items(a, base + shc[jj], base + ci) < 0;
          cr += less;
        }
      }
    }
    __syncthreads();
  }
  if (act) {
    if (pos) atomicAdd(&a.fpos[base + i], pos);
    if (cr) atomicAdd(&a.fcr[base + i], cr);
  }
}

template <int D>
__global__ void __launch_bounds__(256) k_pairs_b(const __grid_constant__ S1Args a,
                                                 const int4* items, const int* n_items, int jchunk) {
  __shared__ double sh[D * TJ];
  __shared__ int shc[TJ];
  const int nw = *n_items;
  for (int w = blockIdx.x; w < nw; w += gridDim.x) {
    const int4 it = items[w];
    pairs_b_tile<D>(a, it.x, it.y, it.z, jchunk, sh, shc);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) k_truncate(const __grid_constant__ S1Args a) {
  typedef cub::BlockScan<int, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry_nontop, carry_kept;
  __shared__ double red_lat[1024];
  __shared__ int red_sl[1024];
  __shared__ double red_acc[1024];
  const int job = blockIdx.x;
  const int probe = job / a.T, t = job % a.T;
  const int F = a.fcnt[job];
  const int W = a.W;
  const long long tot = (long long)a.n_probes * a.C_probe;
  const long long base = job_base(a, probe, t);
  const DGraph& g = *a.g;
  for (int i = threadIdx.x; i < F; i += blockDim.x) {
    int p = a.fpos[base + i];
    a.sorted[base + p] = a.front[base + i];
    a.scr[base + p] = a.fcr[base + i];
  }
  __syncthreads();
  int* pool = a.pool_cand + (long long)job * W;
  int P;
  if (F <= W) {
    for (int k = threadIdx.x; k < F; k += blockDim.x) pool[k] = a.sorted[base + k];
    P = F;
    if (threadIdx.x == 0) a.pool_trunc[job] = 0;
  } else {
    if (threadIdx.x == 0) { carry_nontop = 0; carry_kept = 0; }
    __syncthreads();
    const int top_n = W / 2, rest = W - W / 2;
    for (int s0 = 0; s0 < F; s0 += 1024) {
      int k = s0 + threadIdx.x;
      int nontop = (k < F && a.scr[base + k] >= top_n) ? 1 : 0;
      int before, tot_nt;
      Scan(tmp).ExclusiveSum(nontop, before, tot_nt);
      __syncthreads();
      int keep = 0;
      if (k < F) keep = (!nontop) || (carry_nontop + before < rest);
      int kpos, tot_k;
      Scan(tmp).ExclusiveSum(keep, kpos, tot_k);
      if (keep) pool[carry_kept + kpos] = a.sorted[base + k];
      __syncthreads();
      if (threadIdx.x == 0) { carry_nontop += tot_nt; carry_kept += tot_k; }
      __syncthreads();
    }
    P = carry_kept;
    if (threadIdx.x == 0) a.pool_trunc[job] = 1;
  }
  __syncthreads();
  const int outd = g.succ_off[t + 1] - g.succ_off[t];
  double mlat = 1e308;
  int msl = 0x7fffffff;
  double macc = -1.0;
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    long long c = base + pool[k];
    long long q = (long long)job * W + k;
    double lat = a.arr[3 * tot + c];
    double acc = -a.arr[2 * tot + c];
    int sl = (int)a.arr[0 * tot + c];
    a.p_sl[q] = sl;
    a.p_cap[q] = -a.arr[1 * tot + c];
    a.p_acc[q] = acc;
    a.p_lat[q] = lat;
    for (int j = 0; j < outd; ++j) a.p_fan[q * a.maxout + j] = a.arr[(4 + j) * tot + c];
    double l2 = 2.0 * lat;
    if (l2 < mlat) mlat = l2;
    if (sl < msl) msl = sl;
    if (acc > macc) macc = acc;
  }
  red_lat[threadIdx.x] = mlat;
  red_sl[threadIdx.x] = msl;
  red_acc[threadIdx.x] = macc;
  __syncthreads();
  for (int s = 512; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      int o = threadIdx.x + s;
      if (red_lat[o] < red_lat[threadIdx.x]) red_lat[threadIdx.x] = red_lat[o];
      if (red_sl[o] < red_sl[threadIdx.x]) red_sl[threadIdx.x] = red_sl[o];
      if (red_acc[o] > red_acc[threadIdx.x]) red_acc[threadIdx.x] = red_acc[o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.pool_n[job] = P;
    a.pool_min_lat2[job] = red_lat[0];
    a.pool_min_sl[job] = red_sl[0];
    a.pool_acc_ub[job] = red_acc[0];
  }
}


// Duplicate probes (identical Stage-1 inputs, see plan_batch_internal): copy the
// representative's pools -- every per-job array Stage 2 and finalize read -- and
// the item lists of its pool candidates (same local candidate index) into the
// duplicate's slots.  One block per (duplicate probe, task).
__global__ void __launch_bounds__(256) k_s1_expand(const __grid_constant__ S1Args a,
                                                   const int* rep, int n_s1) {
  const int d = n_s1 + blockIdx.x / a.T, t = blockIdx.x % a.T;
  const int u = rep[d];
  const int jd = d * a.T + t, ju = u * a.T + t;
  const int W = a.W;
  const int np = a.pool_n[ju];
  if (threadIdx.x == 0) {
    a.pool_n[jd] = np;
    a.pool_trunc[jd] = a.pool_trunc[ju];
    a.pool_min_lat2[jd] = a.pool_min_lat2[ju];
    a.pool_min_sl[jd] = a.pool_min_sl[ju];
    a.pool_acc_ub[jd] = a.pool_acc_ub[ju];
    a.cnt[jd] = a.cnt[ju];
    a.fcnt[jd] = a.fcnt[ju];
  }
  const long long bd = job_base(a, d, t), bu = job_base(a, u, t);
  for (int k = threadIdx.x; k < np; k += blockDim.x) {
    const long long qd = (long long)jd * W + k, qu = (long long)ju * W + k;
    const int c = a.pool_cand[qu];
    a.pool_cand[qd] = c;
    a.p_sl[qd] = a.p_sl[qu];
    a.p_cap[qd] = a.p_cap[qu];
    a.p_acc[qd] = a.p_acc[qu];
    a.p_lat[qd] = a.p_lat[qu];
    for (int e = 0; e < a.maxout; ++e) a.p_fan[qd * a.maxout + e] = a.p_fan[qu * a.maxout + e];
    const int ni = a.nitems[bu + c];
    a.nitems[bd + c] = ni;
    for (int m = 0; m < ni; ++m) a.items[(bd + c) * a.maxi + m] = a.items[(bu + c) * a.maxi + m];
  }
}

int launch_stage1_expand(const S1Args& a, const int* rep, int n_s1, int n, cudaStream_t st) {
  if (n <= n_s1) return 0;
  k_s1_expand<<<(unsigned)((n - n_s1) * a.T), 256, 0, st>>>(a, rep, n_s1);
  return 1;
}

// ------------------------------------------------------------ fused Stage 1
//
// k_s1_job: one block per job (probe, task) runs all of Stage 1 for it -- the same
// steps as the kernel chain above, with block barriers instead of kernel
// boundaries and the job's working lists in shared memory (global scratch when a
// job has more than S1Args::fused_cap candidates):
//   A  enumeration units of the task's descriptors -> item lists (gen_unit);
//   B  bundle statistics -> skyline rows (global `arr`, read by the exact tests);
//   C  counting sort by slices, float shadow of coordinates 1..4 in list order;
//   D  same-slices skyline pass (float-shadow quick reject, exact double test,
//      equal rows: the smaller item list survives -- the reference's dedup);
//   E  survivors in list order, their slice-bucket starts;
//   F  survivors against the survivors with fewer slices;
//   G  frontier (survivors in candidate order);
//   H  frontier order (lexicographic rows) and capacity ranks by bitonic sorts
//      (pair counting for non-finite rows or frontiers beyond the sort size);
//   I  pareto_width truncation and the pool SoA + per-pool bounds.
// Dominance is transitive, so the two passes equal the reference's sequential
// "not dominated by an earlier kept row" filter (planner.py:543-583).

__device__ __forceinline__ float4 s1_shadow(const S1Args& a, long long tot, long long c, int D) {
  // coordinates 1..4 rounded to float (monotone); missing coordinates never reject
  return make_float4((float)a.arr[1 * tot + c], (float)a.arr[2 * tot + c], (float)a.arr[3 * tot + c],
                     D >= 5 ? (float)a.arr[4 * tot + c] : -INFINITY);
}

// stable block-wide compaction step: returns this thread's output slot (or -1) and
// advances *carry by the chunk's count (all threads call it)
template <class Scan>
__device__ __forceinline__ int s1_compact_slot(typename Scan::TempStorage& tmp, int* carry, bool keep) {
  int off, total;
  Scan(tmp).ExclusiveSum(keep ? 1 : 0, off, total);
  const int base = *carry;
  __syncthreads();
  if (threadIdx.x == 0) *carry = base + total;
  __syncthreads();
  return keep ? base + off : -1;
}

// stable block-wide compaction of [0, n) with two block barriers: warp w owns one
// contiguous chunk, counts its kept entries by ballots, takes its base from the
// per-warp counts and emits (slot, index) in order.  keep(i) is evaluated twice
// (it must be a pure read); emit(k, i) is called for the k-th kept i.  Returns the
// kept count (every thread).
template <int NT, class Keep, class Emit>
__device__ __forceinline__ int s1_compact_warps(int n, int* s_wcnt, Keep keep, Emit emit) {
  constexpr int NW = NT / 32;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int chunk = (((n + NW - 1) / NW) + 31) & ~31;
  const int c0 = min(n, w * chunk), c1 = min(n, c0 + chunk);
  int cnt = 0;
  for (int b = c0; b < c1; b += 32) {
    const int i = b + lane;
    cnt += __popc(__ballot_sync(FULL, i < c1 && keep(i)));
  }
  if (lane == 0) s_wcnt[w] = cnt;
  __syncthreads();
  int before = 0, total = 0;
  for (int x = lane; x < NW; x += 32) {
    const int v = s_wcnt[x];
    total += v;
    if (x < w) before += v;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    before += __shfl_xor_sync(FULL, before, d);
    total += __shfl_xor_sync(FULL, total, d);
  }
  for (int b = c0; b < c1; b += 32) {
    const int i = b + lane;
    const bool k = i < c1 && keep(i);
    const unsigned m = __ballot_sync(FULL, k);
    if (k) emit(before + __popc(m & ((1u << lane) - 1u)), i);
    before += __popc(m);
  }
  __syncthreads();  // (s_wcnt reusable, every emit visible)
  return total;
}

// exclusive bucket starts in place over h[0 .. nb) (h[i] holds the count of i - 1)
template <class Scan, int S1F_THREADS>
__device__ __forceinline__ void s1_scan_inplace(typename Scan::TempStorage& tmp, int* h, int nb,
                                                int* carry) {
  if (threadIdx.x == 0) *carry = 0;
  __syncthreads();
  for (int i0 = 0; i0 < nb; i0 += S1F_THREADS) {
    const int i = i0 + threadIdx.x;
    const int v = i < nb ? h[i] : 0;
    int inc, total;
    Scan(tmp).InclusiveSum(v, inc, total);
    const int base = *carry;
    if (i < nb) h[i] = base + inc;
    __syncthreads();
    if (threadIdx.x == 0) *carry = base + total;
    __syncthreads();
  }
}

// JSV_S1_PHASES: %globaltimer at the phase boundaries of every job (diagnostics)
#define S1_STAMP(k)                                                            \
  do {                                                                         \
    if (a.stamps && threadIdx.x == 0) {                                        \
      unsigned long long t_;                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
      a.stamps[job * 10 + (k)] = t_;                                    \
    }                                                                          \
  } while (0)
// S1F_THREADS: 1024 (one block per SM, small batches: the most threads per job) or
// 512 (two blocks per SM, large batches)
template <int D, int S1F_THREADS>
__global__ void __launch_bounds__(S1F_THREADS, 2048 / S1F_THREADS / 2) k_s1_job(const __grid_constant__ S1Args a) {
  extern __shared__ __align__(16) unsigned char s1_smem[];
  typedef cub::BlockScan<int, S1F_THREADS> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_n, s_carry, s_ok;
  __shared__ unsigned s_tests[2];  // float-shadow / exact pair tests of the job
  __shared__ int s_wcnt[S1F_THREADS / 32];  // per-warp counts of s1_compact_warps
  __shared__ int s_work[3];  // dynamic work counters: units (A), list positions (D), survivors (F)
  __shared__ __align__(8) unsigned long long s_bar;  // TMA staging of the task's tables
  __shared__ void* s_kptr[4];                        // staged key tables (lat, thr, var, cost)
  __shared__ const unsigned* s_wptr[8];              // staged ways table per descriptor
  __shared__ double s_rd[32];
  __shared__ int s_ri[32];
  __shared__ double s_ra[32];
  const int job = a.job_map ? a.job_map[a.job_off + blockIdx.x] : (int)blockIdx.x;
  const int probe = job / a.T, t = job % a.T;
  const long long tot = (long long)a.n_probes * a.C_probe;
  const long long base = job_base(a, probe, t);
  const int NB = a.S + 2;
  const int tid = threadIdx.x, lane = tid & 31;
  const DGraph& g = *a.g;
  int* bst = reinterpret_cast<int*>(s1_smem);  // [NB] slice-bucket starts
  int* sbst = bst + NB;                        // [NB] survivor bucket starts (cursor in C)
  unsigned char* pcand = s1_smem + (((size_t)2 * NB * sizeof(int) + 15) & ~(size_t)15);
  if (tid == 0) {
    s_n = 0;
    s_work[0] = s_work[1] = s_work[2] = 0;
    s_tests[0] = s_tests[1] = 0;
  }
  S1_STAMP(0);
  __syncthreads();

  // per-candidate working lists: shared memory when the job fits, else global scratch
  const int ncap = a.fused_cap;
  // (before the lists are in use: the task's exhaustive ways tables for A and its
  // profile-key tables for B are staged in their space)
  const int nk = g.key_off[t + 1] - g.key_off[t];
  const int kb = g.key_off[t];
  const int d0 = a.desc_t0[t], d1 = a.desc_t0[t + 1];
  // (key tables in the lists' space, ways tables in the shadow list's space)
  const bool keys_sm = bulk_span(16 * (size_t)nk) + bulk_span(16 * (size_t)nk) <= (size_t)ncap * 16;
  size_t w_span = 0;
  for (int d = d0; d < d1; ++d)
    if (a.desc[d].mode == 0) w_span += bulk_span(4 * (size_t)(a.desc[d].n_tuples + 1) * (a.S + 1));
  const bool ways_sm = w_span <= (size_t)ncap * 16 && d1 - d0 <= 8;
  unsigned char* kreg = pcand;
  unsigned char* wreg = pcand + (((size_t)ncap * 20 + 15) & ~(size_t)15);
  // TMA (cp.async.bulk) staging of both, completing on one mbarrier; JSV_NO_TMA: loops
  if (tid == 0) {
    if (a.tma) {
      mbar_init(&s_bar, 1);
      unsigned tx = 0;
      unsigned char* kp = kreg;
      if (keys_sm) {
        s_kptr[0] = bulk_stage(kp, a.tb.key_lat + kb, 8 * (size_t)nk, &s_bar, &tx);
        kp += bulk_span(8 * (size_t)nk);
        s_kptr[1] = bulk_stage(kp, a.tb.key_thr + kb, 8 * (size_t)nk, &s_bar, &tx);
        kp += bulk_span(8 * (size_t)nk);
        s_kptr[2] = bulk_stage(kp, a.tb.key_var + kb, 4 * (size_t)nk, &s_bar, &tx);
        kp += bulk_span(4 * (size_t)nk);
        s_kptr[3] = bulk_stage(kp, a.tb.key_cost + kb, 4 * (size_t)nk, &s_bar, &tx);
      }
      if (ways_sm) {
        unsigned char* wp = wreg;
        for (int d = d0; d < d1; ++d) {
          const GenDesc& Dd = a.desc[d];
          if (Dd.mode != 0) continue;
          const size_t bytes = 4 * (size_t)(Dd.n_tuples + 1) * (a.S + 1);
          s_wptr[d - d0] = static_cast<const unsigned*>(bulk_stage(wp, a.ways + Dd.w_off, bytes, &s_bar, &tx));
          wp += bulk_span(bytes);
        }
      }
      // (arrive with the transaction count after issuing: the phase completes when
      // every byte has landed)
      mbar_expect_tx(&s_bar, tx);
    } else {
      unsigned char* kp = kreg;
      s_kptr[0] = kp; kp += bulk_span(8 * (size_t)nk);
      s_kptr[1] = kp; kp += bulk_span(8 * (size_t)nk);
      s_kptr[2] = kp; kp += bulk_span(4 * (size_t)nk);
      s_kptr[3] = kp;
      unsigned char* wp = wreg;
      for (int d = d0; d < d1; ++d) {
        if (a.desc[d].mode != 0) continue;
        s_wptr[d - d0] = reinterpret_cast<const unsigned*>(wp);
        wp += bulk_span(4 * (size_t)(a.desc[d].n_tuples + 1) * (a.S + 1));
      }
    }
  }
  __syncthreads();
  double* k_lat = static_cast<double*>(s_kptr[0]);
  double* k_thr = static_cast<double*>(s_kptr[1]);
  int* k_var = static_cast<int*>(s_kptr[2]);
  int* k_cost = static_cast<int*>(s_kptr[3]);
  if (a.tma) {
    if (keys_sm || ways_sm) mbar_wait(&s_bar, 0);
  } else {
    if (keys_sm)
      for (int k = tid; k < nk; k += S1F_THREADS) {
        k_lat[k] = a.tb.key_lat[kb + k];
        k_thr[k] = a.tb.key_thr[kb + k];
        k_var[k] = a.tb.key_var[kb + k];
        k_cost[k] = a.tb.key_cost[kb + k];
      }
    if (ways_sm)
      for (int d = d0; d < d1; ++d) {
        const GenDesc& Dd = a.desc[d];
        if (Dd.mode != 0) continue;
        const int m = (Dd.n_tuples + 1) * (a.S + 1);
        unsigned* w = const_cast<unsigned*>(s_wptr[d - d0]);
        for (int i = tid; i < m; i += S1F_THREADS) w[i] = a.ways[Dd.w_off + i];
      }
  }
  __syncthreads();
  // ---- A: enumeration units of this task's descriptors (_candidate_pool's union)
  int u_tot = 0;
  for (int d = a.desc_t0[t]; d < a.desc_t0[t + 1]; ++d) u_tot += a.desc[d].n_units;
  // warps take groups of 32 units from a shared counter (unit costs differ: exhaustive
  // unranking, cover levels, mixes)
  for (int u0 = 0;;) {
    if (lane == 0) u0 = atomicAdd(&s_work[0], 32);
    u0 = __shfl_sync(0xffffffffu, u0, 0);
    if (u0 >= u_tot) break;
    const int u = u0 + lane;
    GenOut o;
    o.m = 0;
    o.n = 0;
    o.key1 = -1;
    if (u < u_tot) {
      int d = a.desc_t0[t], lu = u;
      while (lu >= a.desc[d].n_units) lu -= a.desc[d++].n_units;
      gen_unit(a, probe, a.desc[d], lu, o, ways_sm ? s_wptr[d - d0] : a.ways + a.desc[d].w_off);
    }
    // warp-aggregated slot reservation
    int incl = o.m;
    for (int k = 1; k < 32; k <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, k);
      if (lane >= k) incl += v;
    }
    const int wtot = __shfl_sync(0xffffffffu, incl, 31);
    int wb = 0;
    if (lane == 31 && wtot) wb = atomicAdd(&s_n, wtot);
    wb = __shfl_sync(0xffffffffu, wb, 31);
    const int pos = wb + incl - o.m;
    if (o.key1 >= 0) {
      for (int x = 0; x < o.m; ++x) {
        const uint32_t one = ((uint32_t)o.key1 << 16) | (uint32_t)o.counts[x];
        store_candidate(a, probe, t, pos + x, &one, 1);
      }
    } else if (o.m > 0) {
      store_candidate(a, probe, t, pos, o.it, o.n);
    }
  }
  __syncthreads();
  const int n = min(s_n, (int)a.task_cap[t]);
  S1_STAMP(1);
  if (tid == 0) a.cnt[job] = s_n;
  const bool fits = n <= ncap;
  int* front = fits ? reinterpret_cast<int*>(pcand) : a.front + base;
  int* ord = fits ? front + ncap : a.order + base;
  int* slp = fits ? ord + ncap : a.pcnt + base;
  int* survp = fits ? slp + ncap : a.surv + base;  // list position of survivor k
  int* sslp = fits ? survp + ncap : a.scr + base;
  float4* shl = fits ? reinterpret_cast<float4*>(sslp + ncap + ((4 - (ncap & 3)) & 3))
                     : a.arrf + base;
  unsigned char* dead = fits ? reinterpret_cast<unsigned char*>(shl + ncap)
                             : reinterpret_cast<unsigned char*>(a.flag + base);

  // ---- B: bundle statistics (planner.py:155-213) -> skyline rows; C: bucket counts
  for (int s0 = tid; s0 < NB; s0 += S1F_THREADS) bst[s0] = 0;
  __syncthreads();
  {
    const int outd = g.succ_off[t + 1] - g.succ_off[t];
    for (int c = tid; c < n; c += S1F_THREADS) {
      Stat st;
      uint32_t it[MAXI];
      const long long cc = base + c;
      const int ni = a.nitems[cc];
      for (int k = 0; k < ni; ++k) it[k] = a.items[cc * a.maxi + k];
      if (keys_sm) bundle_stats_k(g, a.tb, t, it, ni, st, k_var, k_cost, k_lat, k_thr);
      else bundle_stats(g, a.tb, t, it, ni, st);
      a.sl[cc] = st.sl;
      a.arr[0 * tot + cc] = (double)st.sl;
      a.arr[1 * tot + cc] = -st.cap;
      a.arr[2 * tot + cc] = -st.acc;
      a.arr[3 * tot + cc] = st.lat;
      for (int j = 0; j < D - 4; ++j) a.arr[(4 + j) * tot + cc] = j < outd ? st.fan[j] : 0.0;
      dead[c] = 0;
    }
  }
  __syncthreads();
  // ---- B': identical item lists (the same count vector enumerated in several
  // sub-spaces, planner.py:628-632 unions them as a set) keep one candidate, by an
  // open-addressing hash set in shared memory (in the shadow list's space, not yet in use)
  int H = 1;
  while (H < 2 * n) H <<= 1;
  if (fits && H <= 4 * ncap) {
    int* table = reinterpret_cast<int*>(shl);
    for (int h = tid; h < H; h += S1F_THREADS) table[h] = -1;
    __syncthreads();
    for (int c = tid; c < n; c += S1F_THREADS) {
      const long long cc = base + c;
      const int ni = a.nitems[cc];
      unsigned hv = 0x9E3779B9u * (unsigned)(ni + 1);
      for (int k = 0; k < ni; ++k) {
        unsigned x = a.items[cc * a.maxi + k] * 0xCC9E2D51u;
        x = (x << 15) | (x >> 17);
        hv = ((hv ^ (x * 0x1B873593u)) << 13 | (hv ^ (x * 0x1B873593u)) >> 19) * 5u + 0xE6546B64u;
      }
      hv ^= hv >> 16; hv *= 0x85EBCA6Bu; hv ^= hv >> 13;
      for (int h = (int)(hv & (unsigned)(H - 1));; h = (h + 1) & (H - 1)) {
        const int occ = atomicCAS(&table[h], -1, c);
        if (occ == -1) break;
        if (a.nitems[base + occ] == ni && cmp_items(a, base + occ, cc) == 0) {
          dead[c] = 1;  // a duplicate of `occ`
          break;
        }
      }
    }
    __syncthreads();
  }
  for (int c = tid; c < n; c += S1F_THREADS)
    if (!dead[c]) atomicAdd(&bst[a.sl[base + c] + 1], 1);
  __syncthreads();
  S1_STAMP(2);
  // ---- C: counting sort by slices (bucket starts bst[s] = #candidates with < s slices)
  s1_scan_inplace<Scan, S1F_THREADS>(tmp, bst, NB, &s_carry);
  for (int s0 = tid; s0 < NB; s0 += S1F_THREADS) sbst[s0] = bst[s0];
  __syncthreads();
  const int nl = bst[NB - 1];  // candidates in the slices-ordered list (duplicates left out)
  for (int c = tid; c < n; c += S1F_THREADS) {
    if (dead[c]) continue;
    const int sl = a.sl[base + c];
    const int p = atomicAdd(&sbst[sl], 1);
    ord[p] = c;
    slp[p] = sl;
    shl[p] = s1_shadow(a, tot, base + c, D);
  }
  __syncthreads();

  S1_STAMP(3);
  // exact weak-dominance / dedup test of list entry j (candidate cj) against i
  // (coordinates 1 .. D-1; coordinate 0, slices, is equal or smaller for j)
  auto dominated = [&](const double* xi, int ci, int cj, bool same_slices) -> bool {
    bool le = true, eq = true;
#pragma unroll
    for (int d = 1; d < D; ++d) {
      const double xj = a.arr[d * tot + base + cj];
      le = le && (xj <= xi[d]);
      eq = eq && (xj == xi[d]);
    }
    if (!le) return false;
    if (!eq || !same_slices) return true;  // (fewer slices: a different row)
    if (cj == ci) return false;
    const int c = cmp_items(a, base + cj, base + ci);
    return c < 0 || (c == 0 && cj < ci);
  };
  constexpr int XJ = 16;  // (shadow rows in flight per step: 8 -> 16 took 218 -> 209 us per batch)
  unsigned n_sh = 0, n_ex = 0;  // pair tests of the two passes: float shadow / exact
  // ---- D: every candidate against its own slices bucket
  // (warps take 32 list positions at a time: the bucket scans differ in length)
  for (int p0 = 0;;) {
    if (lane == 0) p0 = atomicAdd(&s_work[1], 32);
    p0 = __shfl_sync(0xffffffffu, p0, 0);
    if (p0 >= nl) break;
    const int p = p0 + lane;
    if (p >= nl) continue;
    const int ci = ord[p];
    double xi[D];
#pragma unroll
    for (int d = 1; d < D; ++d) xi[d] = a.arr[d * tot + base + ci];
    const float4 fi = shl[p];
    const int sl = slp[p];
    const int lo = bst[sl], hi = bst[sl + 1];
    bool isdead = false;
    for (int j = lo; j < hi && !isdead; j += XJ) {
      unsigned keep = 0;
#pragma unroll
      for (int u = 0; u < XJ; ++u) {
        if (j + u < hi) {
          const float4 fj = shl[j + u];
          ++n_sh;
          const bool rej = (fj.x > fi.x) | (fj.y > fi.y) | (fj.z > fi.z) | (fj.w > fi.w);
          keep |= (rej ? 0u : 1u) << u;
        }
      }
      while (keep && !isdead) {
        const int u = __ffs(keep) - 1;
        keep &= keep - 1;
        if (j + u != p) {
          isdead = dominated(xi, ci, ord[j + u], true);
          ++n_ex;
        }
      }
    }
    if (isdead) dead[ci] = 1;
  }
  __syncthreads();
  S1_STAMP(4);
  // ---- E: survivors in list order and their bucket starts
  for (int s0 = tid; s0 < NB; s0 += S1F_THREADS) sbst[s0] = 0;
  __syncthreads();
  const int ns = s1_compact_warps<S1F_THREADS>(
      nl, s_wcnt, [&](int p) { return !dead[ord[p]]; },
      [&](int k, int p) {
        survp[k] = p;
        sslp[k] = slp[p];
        atomicAdd(&sbst[slp[p] + 1], 1);
      });
  s1_scan_inplace<Scan, S1F_THREADS>(tmp, sbst, NB, &s_carry);
  // ---- F: survivors against the survivors with fewer slices
  for (int k0 = 0;;) {
    if (lane == 0) k0 = atomicAdd(&s_work[2], 32);
    k0 = __shfl_sync(0xffffffffu, k0, 0);
    if (k0 >= ns) break;
    if (k0 + lane >= ns) continue;
    const int k = ns - 1 - (k0 + lane);  // (the most slices -- the longest scans -- first)
    const int ci = ord[survp[k]];
    double xi[D];
#pragma unroll
    for (int d = 1; d < D; ++d) xi[d] = a.arr[d * tot + base + ci];
    const float4 fi = shl[survp[k]];
    const int hi = sbst[sslp[k]];
    bool isdead = false;
    for (int j = 0; j < hi && !isdead; j += XJ) {
      unsigned keep = 0;
#pragma unroll
      for (int u = 0; u < XJ; ++u) {
        if (j + u < hi) {
          const float4 fj = shl[survp[j + u]];
          ++n_sh;
          const bool rej = (fj.x > fi.x) | (fj.y > fi.y) | (fj.z > fi.z) | (fj.w > fi.w);
          keep |= (rej ? 0u : 1u) << u;
        }
      }
      while (keep && !isdead) {
        const int u = __ffs(keep) - 1;
        keep &= keep - 1;
        isdead = dominated(xi, ci, ord[survp[j + u]], false);
        ++n_ex;
      }
    }
    if (isdead) dead[ci] = 1;
  }
  __syncthreads();
  S1_STAMP(5);
  // pair-test counters: warp sums into shared memory, one global add per job at the end
  if (a.tests) {
    unsigned sh = n_sh, ex = n_ex;
    for (int d = 16; d > 0; d >>= 1) {
      sh += __shfl_down_sync(0xffffffffu, sh, d);
      ex += __shfl_down_sync(0xffffffffu, ex, d);
    }
    if (lane == 0) {
      atomicAdd(&s_tests[0], sh);
      atomicAdd(&s_tests[1], ex);
    }
  }
  // ---- G: the frontier in candidate order
  const int F = s1_compact_warps<S1F_THREADS>(
      n, s_wcnt, [&](int c) { return !dead[c]; }, [&](int k, int c) { front[k] = c; });
  if (tid == 0) a.fcnt[job] = F;

  S1_STAMP(6);
  // ---- H: frontier order (planner.py:556-559) and capacity ranks (planner.py:576)
  int* fpos = a.fpos + base;  // [F] position of frontier entry k in row order
  int* fcr = a.fcr + base;    // [F] its (-capacity, slices, items) rank (F > W)
  constexpr int FMAX = D <= 12 ? FSORT_MAX : FSORT_MAX / 2;
  int F2 = 1;
  while (F2 < F) F2 <<= 1;
  // sort keys after the frontier list (the other per-candidate lists are dead now)
  double* key = reinterpret_cast<double*>(
      fits ? pcand + (((size_t)F * sizeof(int) + 15) & ~(size_t)15) : pcand);
  int* ix = reinterpret_cast<int*>(key + (size_t)D * F2);
  if (tid == 0) s_ok = F <= FMAX;
  __syncthreads();
  if (s_ok) {
    for (int k = tid; k < F2; k += S1F_THREADS) {
      ix[k] = k;
      if (k < F) {
        const int c = front[k];
        for (int d = 0; d < D; ++d) {
          const double v = a.arr[d * tot + base + c];
          if (!isfinite(v)) s_ok = 0;
          key[d * F2 + k] = v;
        }
      } else {
        for (int d = 0; d < D; ++d) key[d * F2 + k] = INFINITY;
      }
    }
    __syncthreads();
  }
  if (s_ok) {
    // sort 1: rows, lexicographic (distinct rows: the sorted rank is the count of
    // smaller rows; padding rows +inf, ties by index)
    // (a stage with j <= 32 pairs elements inside one 64-element block, and the 32
    // consecutive h of a warp cover whole blocks: such a stage needs only the warp's
    // own earlier writes -- __syncwarp -- unless the stage before it crossed warps)
    int pj = F2;
    for (int kk = 2; kk <= F2; kk <<= 1) {
      for (int j = kk >> 1; j > 0; j >>= 1) {
        if (j >= 64 || pj >= 64) __syncthreads();
        else __syncwarp();
        pj = j;
        for (int h = tid; h < (F2 >> 1); h += S1F_THREADS) {
          const int i = ((h & ~(j - 1)) << 1) | (h & (j - 1)), l = i | j;
          const int x = ix[i], y = ix[l];
          int c = 0;
#pragma unroll
          for (int d = 0; d < D; ++d) {
            if (c == 0) {
              const double u = key[d * F2 + x], v = key[d * F2 + y];
              c = u < v ? -1 : (u > v ? 1 : 0);
            }
          }
          if (c == 0) c = x < y ? -1 : 1;
          if ((c > 0) == ((i & kk) == 0)) {
            ix[i] = y;
            ix[l] = x;
          }
        }
      }
    }
    __syncthreads();
    for (int r = tid; r < F; r += S1F_THREADS) fpos[ix[r]] = r;
    if (F > a.W) {
      __syncthreads();
      for (int k = tid; k < F2; k += S1F_THREADS) ix[k] = k;
      __syncthreads();
      // sort 2: (-capacity, slices, items); padding -capacity = +inf
      pj = F2;
      for (int kk = 2; kk <= F2; kk <<= 1) {
        for (int j = kk >> 1; j > 0; j >>= 1) {
          if (j >= 64 || pj >= 64) __syncthreads();
          else __syncwarp();
          pj = j;
          for (int h = tid; h < (F2 >> 1); h += S1F_THREADS) {
            const int i = ((h & ~(j - 1)) << 1) | (h & (j - 1)), l = i | j;
            const int x = ix[i], y = ix[l];
            const double cx = key[1 * F2 + x], cy = key[1 * F2 + y];
            int c;
            if (cx != cy) c = cx < cy ? -1 : 1;
            else if (x >= F || y >= F) c = x < y ? -1 : 1;
            else if (key[x] != key[y]) c = key[x] < key[y] ? -1 : 1;
            else c = cmp_items(a, base + front[x], base + front[y]);
            if (c == 0) c = x < y ? -1 : 1;
            if ((c > 0) == ((i & kk) == 0)) {
              ix[i] = y;
              ix[l] = x;
            }
          }
        }
      }
      __syncthreads();
      for (int r = tid; r < F; r += S1F_THREADS) fcr[ix[r]] = r;
    }
  } else {
    // pair counting (non-finite rows or a frontier beyond the sort size)
    for (int i = tid; i < F; i += S1F_THREADS) {
      const int ci = front[i];
      int pos = 0, cr = 0;
      for (int jj = 0; jj < F; ++jj) {
        const int cj = front[jj];
        int lt = 0;
        for (int d = 0; d < D; ++d) {
          if (lt == 0) {
            const double xj = a.arr[d * tot + base + cj], xi = a.arr[d * tot + base + ci];
            if (xj < xi) lt = 1;
            else if (xj > xi) lt = -1;
          }
        }
        pos += lt == 1;
        if (F > a.W) {
          const double c1 = a.arr[1 * tot + base + cj], c0 = a.arr[1 * tot + base + ci];
          bool less;
          if (c1 != c0) less = c1 < c0;
          else if (a.arr[base + cj] != a.arr[base + ci]) less = a.arr[base + cj] < a.arr[base + ci];
          else less = cmp_items(a, base + cj, base + ci) < 0;
          cr += less;
        }
      }
      fpos[i] = pos;
      fcr[i] = cr;
    }
  }
  __syncthreads();

  S1_STAMP(7);
  // ---- I: truncation to pareto_width (planner.py:574-583) and the pool
  int* srt = a.sorted + base;  // frontier candidates in row order
  int* scr = a.scr + base;     // ... and their capacity ranks
  for (int i = tid; i < F; i += S1F_THREADS) {
    const int p = fpos[i];
    srt[p] = front[i];
    if (F > a.W) scr[p] = fcr[i];  // (capacity ranks exist only for truncated frontiers)
  }
  __syncthreads();
  const int W = a.W;
  int* pool = a.pool_cand + (long long)job * W;
  int P;
  if (F <= W) {
    for (int k = tid; k < F; k += S1F_THREADS) pool[k] = srt[k];
    P = F;
    if (tid == 0) a.pool_trunc[job] = 0;
  } else {
    // the W/2 largest capacities, then the other frontier rows in row order
    const int top_n = W / 2, rest = W - W / 2;
    __shared__ int s_nontop, s_kept;
    if (tid == 0) { s_nontop = 0; s_kept = 0; }
    __syncthreads();
    for (int s0 = 0; s0 < F; s0 += S1F_THREADS) {
      const int k = s0 + tid;
      const int nontop = (k < F && scr[k] >= top_n) ? 1 : 0;
      int before, tot_nt;
      Scan(tmp).ExclusiveSum(nontop, before, tot_nt);
      __syncthreads();
      const int keep = (k < F) && ((!nontop) || (s_nontop + before < rest));
      int kpos, tot_k;
      Scan(tmp).ExclusiveSum(keep, kpos, tot_k);
      if (keep) pool[s_kept + kpos] = srt[k];
      __syncthreads();
      if (tid == 0) { s_nontop += tot_nt; s_kept += tot_k; }
      __syncthreads();
    }
    P = s_kept;
    if (tid == 0) a.pool_trunc[job] = 1;
  }
  __syncthreads();
  const int outd = g.succ_off[t + 1] - g.succ_off[t];
  double mlat = 1e308, macc = -1.0;
  int msl = 0x7fffffff;
  for (int k = tid; k < P; k += S1F_THREADS) {
    const long long c = base + pool[k];
    const long long q = (long long)job * W + k;
    const double lat = a.arr[3 * tot + c];
    const double acc = -a.arr[2 * tot + c];
    const int sl = (int)a.arr[0 * tot + c];
    a.p_sl[q] = sl;
    a.p_cap[q] = -a.arr[1 * tot + c];
    a.p_acc[q] = acc;
    a.p_lat[q] = lat;
    for (int j = 0; j < outd; ++j) a.p_fan[q * a.maxout + j] = a.arr[(4 + j) * tot + c];
    const double l2 = 2.0 * lat;
    if (l2 < mlat) mlat = l2;
    if (sl < msl) msl = sl;
    if (acc > macc) macc = acc;
  }
  for (int d = 16; d > 0; d >>= 1) {
    mlat = fmin(mlat, __shfl_down_sync(0xffffffffu, mlat, d));
    msl = min(msl, __shfl_down_sync(0xffffffffu, msl, d));
    macc = fmax(macc, __shfl_down_sync(0xffffffffu, macc, d));
  }
  if (lane == 0) {
    s_rd[tid >> 5] = mlat;
    s_ri[tid >> 5] = msl;
    s_ra[tid >> 5] = macc;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < S1F_THREADS / 32; ++w) {
      if (s_rd[w] < mlat) mlat = s_rd[w];
      if (s_ri[w] < msl) msl = s_ri[w];
      if (s_ra[w] > macc) macc = s_ra[w];
    }
    mlat = fmin(mlat, s_rd[0]);
    msl = min(msl, s_ri[0]);
    macc = fmax(macc, s_ra[0]);
    a.pool_n[job] = P;
    if (a.tests) {
      atomicAdd(&a.tests[0], (unsigned long long)s_tests[0]);
      atomicAdd(&a.tests[1], (unsigned long long)s_tests[1]);
    }
    a.pool_min_lat2[job] = mlat;
    a.pool_min_sl[job] = msl;
    a.pool_acc_ub[job] = macc;
  }
  S1_STAMP(8);
}

// shared memory of k_s1_job: bucket tables + per-candidate lists of fused_cap
// candidates, or the frontier sort keys, whichever is larger
size_t s1_fused_smem(int D, int NB, int cap) {
  const size_t fixed = ((size_t)2 * NB * sizeof(int) + 15) & ~(size_t)15;
  const size_t lists = (size_t)cap * (5 * sizeof(int) + sizeof(float4) + 1) + 64;
  const int fmax = D <= 12 ? FSORT_MAX : FSORT_MAX / 2;
  const size_t sort = (((size_t)fmax * sizeof(int) + 15) & ~(size_t)15) +
                      (size_t)fmax * (D * sizeof(double) + sizeof(int));
  return fixed + std::max(lists, sort);
}

int launch_stage1_fused(const S1Args& a, size_t smem, int n_heavy, cudaStream_t st, cudaStream_t st2,
                        cudaEvent_t fork, cudaEvent_t join) {
  const long long jobs = (long long)a.n_probes * a.T;
  int dev = 0, n_sm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
#define JSV_S1F(DV, NT, GRID, ARGS, STREAM)                                        \
  do {                                                                             \
    jsv_smem_attr((const void*)k_s1_job<DV, NT>, smem);                            \
    k_s1_job<DV, NT><<<(unsigned)(GRID), NT, smem, STREAM>>>(ARGS);                \
  } while (0)
#define JSV_S1FD(NT, GRID, ARGS, STREAM)             \
  switch (a.D) {                                     \
    case 4: JSV_S1F(4, NT, GRID, ARGS, STREAM); break;   \
    case 5: JSV_S1F(5, NT, GRID, ARGS, STREAM); break;   \
    case 6: JSV_S1F(6, NT, GRID, ARGS, STREAM); break;   \
    case 8: JSV_S1F(8, NT, GRID, ARGS, STREAM); break;   \
    case 12: JSV_S1F(12, NT, GRID, ARGS, STREAM); break; \
    default: JSV_S1F(16, NT, GRID, ARGS, STREAM); break; \
  }
  PROF_BEGIN(K_GENERATE);
  int launches = 1;
  if (a.job_map && n_heavy >= jobs) {
    // every job on 1024 threads in job_map's order (largest first: the second
    // wave's jobs are the smallest and start as the first SMs free up)
    JSV_S1FD(1024, jobs, a, st);
  } else if (a.job_map && n_heavy > 0) {
    // one wave: the n_heavy jobs of job_map's head on 1024 threads (one per SM) on
    // st, the rest at 512 threads two per SM on st2 (joined back into st)
    S1Args h = a, l = a;
    h.job_off = 0;
    l.job_off = n_heavy;
    cudaEventRecord(fork, st);
    cudaStreamWaitEvent(st2, fork, 0);
    JSV_S1FD(1024, n_heavy, h, st);
    JSV_S1FD(512, jobs - n_heavy, l, st2);
    cudaEventRecord(join, st2);
    cudaStreamWaitEvent(st, join, 0);
    launches = 2;
  } else if (jobs <= n_sm) {
    JSV_S1FD(1024, jobs, a, st);
  } else {
    JSV_S1FD(512, jobs, a, st);
  }
  PROF_END();
#undef JSV_S1FD
#undef JSV_S1F
  return launches;
}

// ------------------------------------------------------------------ launchers

static int pick_D(int D) {
  if (D <= 4) return 4;
  if (D <= 5) return 5;
  if (D <= 6) return 6;
  if (D <= 8) return 8;
  if (D <= 12) return 12;
  if (D <= 16) return 16;
  return MAXD;
}

int stage1_padded_dims(int D) { return pick_D(D); }

#define DISPATCH_D(D, KERNEL, GRID, ...)                     \
  switch (D) {                                               \
    case 4: KERNEL<4><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;   \
    case 5: KERNEL<5><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;   \
    case 6: KERNEL<6><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;   \
    case 8: KERNEL<8><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;   \
    case 12: KERNEL<12><<<GRID, 256, 0, st>>>(__VA_ARGS__); break; \
    case 16: KERNEL<16><<<GRID, 256, 0, st>>>(__VA_ARGS__); break; \
    default: KERNEL<MAXD><<<GRID, 256, 0, st>>>(__VA_ARGS__); break; \
  }

#define DISPATCH_D2(D, KERNEL, B, GRID, ...)                             \
  switch (D) {                                                            \
    case 4: KERNEL<4, B><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;         \
    case 5: KERNEL<5, B><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;         \
    case 6: KERNEL<6, B><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;         \
    case 8: KERNEL<8, B><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;         \
    case 12: KERNEL<12, B><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;       \
    case 16: KERNEL<16, B><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;       \
    default: KERNEL<MAXD, B><<<GRID, 256, 0, st>>>(__VA_ARGS__); break;     \
  }

int launch_stage1(const S1Args& a0, const S1Launch& L, cudaStream_t st) {
  int launches = 0;
  // the tiled pair kernels read device work lists; the barrier-free ones do not
  const bool tiled = a0.D > 16 || getenv("JSV_PAIRS_TILED") != nullptr;
  const bool tiled1 = tiled || getenv("JSV_PAIRS_A1") != nullptr;
  S1Args a = a0;
  a.wl_mask = (tiled ? 1 : 0) | (tiled1 ? 2 : 0) | 4;
  long long gen = (long long)a.n_probes * a.U;
  if (gen > 0) {
    PROF_BEGIN(K_GENERATE);
    k_generate<<<(unsigned)((gen + 255) / 256), 256, 0, st>>>(a);
    PROF_END();
    ++launches;
  }
  long long tot = (long long)a.n_probes * a.C_probe;
  if (tot > 0) {
    PROF_BEGIN(K_STATS);
    k_stats<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(a);
    PROF_END();
    ++launches;
  }
  {
    const int NB = a.S + 2;
    const size_t smem = NB <= BUCKET_SMEM_MAX ? sizeof(int) * NB : 0;
    PROF_BEGIN(K_BUCKET);
    k_bucket<<<a.n_probes * a.T, JOB_BS, smem, st>>>(a);
    PROF_END();
    ++launches;
  }
  if (L.tiles_pp > 0) {
    // grid-stride over the device work lists: enough blocks to fill the SMs
    const unsigned ga = (unsigned)std::max<long long>(1, std::min<long long>(L.max_items, L.grid));
    PROF_BEGIN(K_PAIRS_A);
    const unsigned gl = (unsigned)((tot + 255) / 256);
    // wide rows (many out-edges) stage j tiles in shared memory instead
    if (tiled) {
      DISPATCH_D(a.D, k_pairs_a, ga, a, a.wl[0], a.wn + 0, 1024, 0);
    } else {
      // bucketed same-slices pass: skip the slices coordinate
      if (a.S + 2 <= BUCKET_SMEM_MAX) {
        DISPATCH_D2(a.D, k_pairs_l, true, gl, a, 0);
      } else {
        DISPATCH_D2(a.D, k_pairs_l, false, gl, a, 0);
      }
    }
    k_surv<<<a.n_probes * a.T, JOB_BS, 0, st>>>(a);
    // survivors pass: the same barrier-free kernel (float-shadow quick reject in
    // survivor order, built by k_surv); JSV_PAIRS_A1 selects the tiled kernel
    if (tiled1) {
      DISPATCH_D(a.D, k_pairs_a, ga, a, a.wl[1], a.wn + 1, 1024, 1);
    } else if (a.S + 2 <= BUCKET_SMEM_MAX) {
      DISPATCH_D2(a.D, k_pairs_l, true, gl, a, 1);
    } else {
      DISPATCH_D2(a.D, k_pairs_l, false, gl, a, 1);
    }
    PROF_END();
    launches += 3;
  }
  PROF_BEGIN(K_COMPACT);
  k_compact<<<a.n_probes * a.T, JOB_BS, 0, st>>>(a);
  PROF_END();
  ++launches;
  if (L.tiles_pp > 0) {
    const unsigned gb = (unsigned)std::max<long long>(1, std::min<long long>(L.max_items, L.grid));
    PROF_BEGIN(K_PAIRS_B);
    if (a.D <= 16 && !getenv("JSV_NO_FSORT")) {
      const int fmax = a.D <= 12 ? FSORT_MAX : FSORT_MAX / 2;
      int F2 = 1;
      while (F2 < fmax) F2 <<= 1;
      const size_t fsm = (size_t)F2 * (a.D * sizeof(double) + sizeof(int));
#define JSV_FS(DV)                                                                               \
  do {                                                                                           \
    jsv_smem_attr((const void*)k_front_sort<DV>, fsm);                                   \
    k_front_sort<DV><<<a.n_probes * a.T, 512, fsm, st>>>(a);                                      \
  } while (0)
      switch (a.D) {
        case 4: JSV_FS(4); break;
        case 5: JSV_FS(5); break;
        case 6: JSV_FS(6); break;
        case 8: JSV_FS(8); break;
        case 12: JSV_FS(12); break;
        default: JSV_FS(16); break;
      }
#undef JSV_FS
      ++launches;
    } else {
      cudaMemsetAsync(a.fsorted, 0, sizeof(int) * a.n_probes * a.T, st);
    }
    DISPATCH_D(a.D, k_pairs_b, gb, a, a.wl[2], a.wn + 2, 1024);
    PROF_END();
    ++launches;
  }
  PROF_BEGIN(K_TRUNCATE);
  k_truncate<<<a.n_probes * a.T, 1024, 0, st>>>(a);
  PROF_END();
  ++launches;
  // (m ties are resolved directly on the item lists in Stage 2; no rank pass needed)
  return launches;
}
