// jsv_place.cu -- placement of a plan's MIG instances onto physical GPUs
// (reference pkg/src/sliceserve/placement.py:150-290, called on a plan's
// instance_segments, simulator.py:271-273, by cli.py:173-174 and
// workload.py:278).
//
// Host code: a first-fit-decreasing pass over <= a few hundred instances and,
// when it strands some, a budgeted backtracking search over per-GPU occupancy
// bitmasks.  Both are sequential, branchy tree walks over a handful of machine
// words -- no data-parallel work a GPU launch would amortise -- so they run on
// the host inside libjsv (no CUDA call), next to the planner they consume.
//
// Exactness: the same instance order (max footprint desc, compute cost desc,
// profile name, index), the same start order (ascending start), the same
// first-fit rule, and the same backtracking tree (symmetry rule for identical
// consecutive profiles, "fresh GPUs tried at most once", node counter and
// budget) as the reference, so placements are identical, including which
// layout an exhausted budget falls back to.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/jsv.h"

int jsv_fail_msg(int code, const std::string& msg);  // jsv_api.cu

namespace {

struct Geo {
  int np, spg;
  std::vector<std::vector<std::pair<int, int>>> starts;  // per profile (start, width), start asc
  std::vector<int> rank;                                 // first-fit-decreasing sort rank
  std::vector<int> min_w;
};

int load_geo(const jsv_geometry* g, Geo& G) {
  if (!g || g->n_profiles <= 0 || g->slices_per_gpu <= 0 || g->slices_per_gpu > 63)
    return jsv_fail_msg(JSV_ERR_ARG, "bad geometry");
  G.np = g->n_profiles;
  G.spg = g->slices_per_gpu;
  G.starts.assign(G.np, {});
  G.rank.assign(G.np, 0);
  G.min_w.assign(G.np, 0);
  for (int p = 0; p < G.np; ++p) {
    for (int k = g->start_off[p]; k < g->start_off[p + 1]; ++k)
      G.starts[p].push_back({g->start_pos[k], g->start_width[k]});
    std::sort(G.starts[p].begin(), G.starts[p].end());
    if (G.starts[p].empty()) return jsv_fail_msg(JSV_ERR_ARG, "profile without starts");
    G.rank[p] = g->order_rank[p];
    int mw = G.starts[p][0].second;
    for (auto& s : G.starts[p]) mw = std::min(mw, s.second);
    G.min_w[p] = mw;
  }
  return JSV_OK;
}

// 64-bit occupancy masks: up to 63 slices per GPU
inline uint64_t span(int start, int width) { return ((1ull << width) - 1ull) << start; }

// _exact_pack (placement.py:219-266): (gpu, start, width) per sorted position
struct Exact {
  const Geo& G;
  const std::vector<int>& migs;  // profile per sorted position
  int gpus;
  long long budget, nodes = 0;
  bool exhausted = false;
  uint64_t full;
  std::vector<uint64_t> fr;
  std::vector<int> cg, cs, cw;
  Exact(const Geo& g, const std::vector<int>& m, int n, long long b)
      : G(g), migs(m), gpus(n), budget(b), full((1ull << g.spg) - 1ull), fr(n, (1ull << g.spg) - 1ull) {}
  bool place(size_t i, int floor_gpu, int floor_start) {
    if (i == migs.size()) return true;
    ++nodes;
    if (nodes > budget) {
      exhausted = true;
      return false;
    }
    const bool same_as_prev = i > 0 && migs[i] == migs[i - 1];
    int used_hi = -1;
    for (int g = 0; g < gpus; ++g)
      if (fr[g] != full) used_hi = g;
    for (int g = 0; g < gpus; ++g) {
      if (g > used_hi + 1) break;  // every further GPU is empty and interchangeable
      for (const auto& sw : G.starts[migs[i]]) {
        const int s = sw.first, w = sw.second;
        if (same_as_prev && (g < floor_gpu || (g == floor_gpu && s < floor_start))) continue;
        const uint64_t m = span(s, w);
        if ((fr[g] & m) == m) {
          fr[g] &= ~m;
          cg.push_back(g); cs.push_back(s); cw.push_back(w);
          if (place(i + 1, g, s)) return true;
          cg.pop_back(); cs.pop_back(); cw.pop_back();
          fr[g] |= m;
          if (exhausted) return false;
        }
      }
    }
    return false;
  }
};

// pack (placement.py:163-216); out arrays by input instance
int pack_impl(const Geo& G, const int32_t* prof, int n, int gpu_count, long long budget,
              int32_t* gpu, int32_t* start, int32_t* width, int32_t* placed) {
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int x, int y) { return G.rank[prof[x]] < G.rank[prof[y]]; });
  std::vector<uint64_t> fr(gpu_count, 0ull);  // occupied bits
  bool any_unplaced = false;
  for (int i = 0; i < n; ++i) placed[i] = 0;
  for (int idx : order) {
    const int p = prof[idx];
    bool done = false;
    for (int g = 0; g < gpu_count && !done; ++g)
      for (const auto& sw : G.starts[p]) {
        const uint64_t m = span(sw.first, sw.second);
        if (!(fr[g] & m)) {
          fr[g] |= m;
          gpu[idx] = g; start[idx] = sw.first; width[idx] = sw.second; placed[idx] = 1;
          done = true;
          break;
        }
      }
    if (!done) any_unplaced = true;
  }
  if (any_unplaced && gpu_count > 0) {
    std::vector<int> migs(n);
    for (int j = 0; j < n; ++j) migs[j] = prof[order[j]];
    Exact ex(G, migs, gpu_count, budget);
    if (ex.place(0, 0, 0)) {
      for (int j = 0; j < n; ++j) {
        const int idx = order[j];
        gpu[idx] = ex.cg[j]; start[idx] = ex.cs[j]; width[idx] = ex.cw[j]; placed[idx] = 1;
      }
    }
  }
  return JSV_OK;
}

}  // namespace

extern "C" int jsv_pack(const jsv_geometry* geometry, const int32_t* inst_profile, int32_t n,
                        int32_t gpu_count, int64_t node_budget, int32_t* gpu, int32_t* start,
                        int32_t* width, int32_t* placed) {
  if (n < 0 || (n > 0 && (!inst_profile || !gpu || !start || !width || !placed)))
    return jsv_fail_msg(JSV_ERR_ARG, "null argument");
  if (gpu_count < 0) return jsv_fail_msg(JSV_ERR_CONFIG, "gpu_count must be non-negative");
  Geo G;
  int rc = load_geo(geometry, G);
  if (rc) return rc;
  for (int i = 0; i < n; ++i)
    if (inst_profile[i] < 0 || inst_profile[i] >= G.np)
      return jsv_fail_msg(JSV_ERR_ARG, "instance profile out of range");
  return pack_impl(G, inst_profile, n, gpu_count, node_budget, gpu, start, width, placed);
}

extern "C" int jsv_min_gpus(const jsv_geometry* geometry, const int32_t* inst_profile, int32_t n,
                            int64_t node_budget, int32_t* out) {
  if (!out || n < 0 || (n > 0 && !inst_profile)) return jsv_fail_msg(JSV_ERR_ARG, "null argument");
  Geo G;
  int rc = load_geo(geometry, G);
  if (rc) return rc;
  *out = 0;
  if (n == 0) return JSV_OK;
  std::vector<int32_t> g(n), s(n), w(n), pl(n);
  // every instance must fit an empty GPU (placement.py:282-284)
  for (int i = 0; i < n; ++i) {
    if (inst_profile[i] < 0 || inst_profile[i] >= G.np)
      return jsv_fail_msg(JSV_ERR_ARG, "instance profile out of range");
    pack_impl(G, inst_profile + i, 1, 1, node_budget, g.data(), s.data(), w.data(), pl.data());
    if (!pl[0]) {
      *out = -1 - i;
      return JSV_OK;
    }
  }
  long long total = 0;
  for (int i = 0; i < n; ++i) total += G.min_w[inst_profile[i]];
  const int lo = (int)std::max<long long>(1, (total + G.spg - 1) / G.spg);
  for (int k = lo; k <= n; ++k) {
    pack_impl(G, inst_profile, n, k, node_budget, g.data(), s.data(), w.data(), pl.data());
    bool all = true;
    for (int i = 0; i < n && all; ++i) all = pl[i] != 0;
    if (all) {
      *out = k;
      return JSV_OK;
    }
  }
  *out = n;
  return JSV_OK;
}
