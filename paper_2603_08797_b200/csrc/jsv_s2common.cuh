// jsv_s2common.cuh -- leaf helpers shared by the Stage-2 translation units
// (jsv_stage2.cu: search + finalize, jsv_exh.cu: exhaustive sweep, jsv_fo.cu: fan-out).
#pragma once
#include "jsv_internal.cuh"
#include "jsv_kernels.h"

__device__ __forceinline__ void pack16(unsigned long long* w, int k, unsigned v) {
  w[k >> 2] |= (unsigned long long)(v & 0xFFFFu) << ((3 - (k & 3)) * 16);
}


__device__ inline void leaf_key(int T, const uint16_t* ch_topo, unsigned long long* w) {
  w[0] = w[1] = w[2] = w[3] = 0ull;
  for (int k = 0; k < T; ++k) pack16(w, k, ch_topo[k] == NONE16 ? 0u : ch_topo[k]);
}

__device__ inline void load_leaf(const S2Args& a, int probe, const uint16_t* ch_topo, double* lat,
                                 double* cap, double* acc, int* sl, double* fan, uint32_t& present) {
  const DGraph& g = *a.g;
  present = 0;
  for (int u = 0; u < a.T; ++u) {
    const int c = ch_topo[g.pos_of[u]];
    const int job = probe * a.T + u;
    const int outd = g.succ_off[u + 1] - g.succ_off[u];
    if (c == NONE16) {
      lat[u] = 0.0; cap[u] = 0.0; acc[u] = 1.0; sl[u] = 0;
      for (int j = 0; j < outd; ++j) fan[g.succ_off[u] + j] = 0.0;
    } else {
      const long long q = (long long)job * a.W + c;
      lat[u] = a.p_lat[q]; cap[u] = a.p_cap[q]; acc[u] = a.p_acc[q]; sl[u] = a.p_sl[q];
      for (int j = 0; j < outd; ++j) fan[g.succ_off[u] + j] = a.p_fan[q * a.maxout + j];
      present |= 1u << u;
    }
  }
}

__device__ __forceinline__ int find_probe(const long long* off, int n, long long x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Cursor over the canonical m of one leaf: ((task, variant, segment, batch), count)
// tuples in task-id order (planner.py:262), each encoded as task << 32 | key << 16 | count.
struct MCursor {
  const S2Args* a;
  int probe;
  const uint16_t* ch;  // choices by topo position
  int u, k, n;
  long long base;
  __device__ void open_task() {
    while (u < a->T) {
      const int c = ch[a->g->pos_of[u]];
      if (c != NONE16) {
        const long long q = (long long)(probe * a->T + u) * a->W + c;
        base = (long long)probe * a->C_probe + a->task_base[u] + a->pool_cand[q];
        n = a->nitems[base];
        if (n > 0) return;
      }
      ++u;
    }
  }
  __device__ bool next(unsigned long long& e) {
    if (u >= a->T) return false;
    e = ((unsigned long long)u << 32) | a->items[base * a->maxi + k];
    if (++k >= n) {
      ++u;
      k = 0;
      open_task();
    }
    return true;
  }
};
