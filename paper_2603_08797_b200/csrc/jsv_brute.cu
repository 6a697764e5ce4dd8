// jsv_brute.cu -- brute_force_plan() on sm_100a (reference planner.py:1181-1272).
//
// The reference's oracle enumerates every instance-count map over the
// request space's profile keys (sorted (task, variant, segment, batch)), each
// count in 0..min(max_count, left // cost) with left the unspent slice budget,
// depth-first (key 0 most significant, counts ascending), derives and
// validates each map and keeps the argmax of (objective, -total_slices), ties
// on the smaller canonical m.  Here the maps are a ranked set: ways[i][left] =
// number of count suffixes of keys i.. within `left` slices, so an index in
// [0, ways[0][S]) unranks to exactly the reference's i-th map.  One thread
// evaluates one map at a time (grid-stride) with the same device
// derive/validate code as every other path (bundle_stats + evaluate, the
// reference's float order); the argmax is a block tree reduction followed by
// a one-block fold over the block results.  The tie-break compares the m
// tuples the reference compares (planner.py:1241-1243) -- on count vectors:
// at the first differing key, two non-zero counts compare as counts; a zero
// count drops that key from m, so that m is larger unless it has no later
// non-zero key (then it is a strict prefix, hence smaller).
#include "jsv_internal.cuh"
#include "jsv_kernels.h"

#define BF_THREADS 256

__device__ void bf_decode(const BruteArgs& a, long long idx, uint16_t* cnt) {
  int left = a.S;
  for (int i = 0; i < a.K; ++i) {
    const int cost = a.key_cost[i];
    const int cap = min(a.maxc, left / cost);
    const long long* w = a.ways + (long long)(i + 1) * (a.S + 1);
    int c = 0;
    for (; c < cap; ++c) {
      const long long n = w[left - c * cost];
      if (idx < n) break;
      idx -= n;
    }
    cnt[i] = (uint16_t)c;
    left -= c * cost;
  }
}

// m(idx1) vs m(idx2) as Python tuples of ((key), count) pairs
__device__ int bf_cmp_m(const BruteArgs& a, long long i1, long long i2) {
  uint16_t x[BF_MAXK], y[BF_MAXK];
  bf_decode(a, i1, x);
  bf_decode(a, i2, y);
  for (int i = 0; i < a.K; ++i) {
    if (x[i] == y[i]) continue;
    if (x[i] != 0 && y[i] != 0) return x[i] < y[i] ? -1 : 1;
    const uint16_t* z = x[i] == 0 ? x : y;  // the map that skips key i
    bool later = false;
    for (int j = i + 1; j < a.K; ++j) later |= z[j] != 0;
    const int zx = later ? 1 : -1;  // sign of m(z) - m(other)
    return x[i] == 0 ? zx : -zx;
  }
  return 0;
}

__device__ __forceinline__ bool bf_better(const BruteArgs& a, const BruteBest& A, const BruteBest& B) {
  if (!A.has) return false;
  if (!B.has) return true;
  if (A.obj != B.obj) return A.obj > B.obj;
  if (A.sl != B.sl) return A.sl < B.sl;
  return bf_cmp_m(a, A.idx, B.idx) < 0;
}

__device__ void bf_eval(const BruteArgs& a, long long idx, BruteBest& best) {
  const DGraph& g = *a.g;
  uint16_t cnt[BF_MAXK];
  bf_decode(a, idx, cnt);
  double lat[MAXT], cap[MAXT], acc[MAXT], fan[MAXE];
  int sl[MAXT];
  uint32_t present = 0;
  int i = 0;
  for (int t = 0; t < g.T; ++t) {
    uint32_t items[MAXI];
    int n = 0;
    for (; i < a.K && a.key_task[i] == t; ++i)
      if (cnt[i]) items[n++] = ((uint32_t)a.key_local[i] << 16) | cnt[i];
    Stat s;
    bundle_stats(g, a.tb, t, items, n, s);
    lat[t] = s.lat; cap[t] = s.cap; acc[t] = s.acc; sl[t] = s.sl;
    const int outd = g.succ_off[t + 1] - g.succ_off[t];
    for (int j = 0; j < outd; ++j) fan[g.succ_off[t] + j] = s.fan[j];
    if (n) present |= 1u << t;
  }
  EvalOut ev;
  evaluate<false>(g, *a.rq, *a.probe, lat, cap, acc, sl, fan, present, ev, nullptr, nullptr,
                  nullptr, nullptr);
  if (!ev.feasible) return;
  BruteBest c{1, ev.total_sl, ev.objective, idx};
  if (bf_better(a, c, best)) best = c;
}

__device__ void bf_block_fold(const BruteArgs& a, BruteBest& mine, BruteBest* sh) {
  sh[threadIdx.x] = mine;
  __syncthreads();
  for (int s = blockDim.x >> 1; s > 0; s >>= 1) {
    if (threadIdx.x < s && bf_better(a, sh[threadIdx.x + s], sh[threadIdx.x]))
      sh[threadIdx.x] = sh[threadIdx.x + s];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(BF_THREADS) k_brute(const __grid_constant__ BruteArgs a) {
  __shared__ BruteBest sh[BF_THREADS];
  BruteBest best{0, 0, 0.0, 0};
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < a.total; idx += stride)
    bf_eval(a, idx, best);
  bf_block_fold(a, best, sh);
  if (threadIdx.x == 0) a.part[blockIdx.x] = sh[0];
}

// fold the block results; write the winner's per-task items for k_derive
__global__ void __launch_bounds__(BF_THREADS) k_brute_fold(const __grid_constant__ BruteArgs a, int n_part) {
  __shared__ BruteBest sh[BF_THREADS];
  BruteBest best{0, 0, 0.0, 0};
  for (int k = threadIdx.x; k < n_part; k += blockDim.x)
    if (bf_better(a, a.part[k], best)) best = a.part[k];
  bf_block_fold(a, best, sh);
  if (threadIdx.x != 0) return;
  const BruteBest w = sh[0];
  *a.found = w.has;
  *a.win = w.idx;
  uint16_t cnt[BF_MAXK];
  if (w.has) bf_decode(a, w.idx, cnt);
  int i = 0;
  for (int t = 0; t < a.g->T; ++t) {
    int n = 0;
    for (; i < a.K && a.key_task[i] == t; ++i)
      if (w.has && cnt[i]) a.items[t * MAXI + n++] = ((uint32_t)a.key_local[i] << 16) | cnt[i];
    a.n_items[t] = n;
  }
}

int launch_brute(const BruteArgs& a, int blocks, cudaStream_t st) {
  k_brute<<<blocks, BF_THREADS, 0, st>>>(a);
  k_brute_fold<<<1, BF_THREADS, 0, st>>>(a, blocks);
  return 2;
}
