// Host-side subject planner (no device work): the assignment of
// plan_partitions (reference partition.py:49-98), native so the partition
// layer does not loop over subjects in Python.
//
//   hash: owner(e) = ((e * 0x9E3779B1) mod 2^32) mod m        (partition.py:80-84)
//   LPT : subjects ordered by (out-degree desc, id asc), each placed on the
//         partition with the smallest (load, index)          (partition.py:85-94)
//
// The LPT argmin is a segment tree over the m partitions (an internal node
// holds the winner of its two children, ties to the lower index), so a
// placement is one leaf update plus log2(m) re-comparisons; this yields the
// same sequence as any exact (load, index) priority order.
#include <stdint.h>

#include <algorithm>
#include <numeric>
#include <vector>

#include "../../include/th_b200.h"
#include "common.cuh"

namespace {

struct MinTree {
  int m = 0, leaves = 1;
  std::vector<int64_t> load;  // per partition
  std::vector<int32_t> win;   // node -> partition index (or -1 for padding)

  explicit MinTree(int m_) : m(m_), load(m_, 0) {
    while (leaves < m) leaves <<= 1;
    win.assign(2 * leaves, -1);
    for (int p = 0; p < m; ++p) win[leaves + p] = p;
    for (int n = leaves - 1; n >= 1; --n) win[n] = better(win[2 * n], win[2 * n + 1]);
  }
  int32_t better(int32_t a, int32_t b) const {
    if (a < 0) return b;
    if (b < 0) return a;
    if (load[a] != load[b]) return load[a] < load[b] ? a : b;
    return a < b ? a : b;
  }
  int32_t top() const { return win[1]; }
  void add(int32_t p, int64_t w) {
    load[p] += w;
    for (int n = (leaves + p) >> 1; n >= 1; n >>= 1) win[n] = better(win[2 * n], win[2 * n + 1]);
  }
};

}  // namespace

extern "C" int th_plan_subjects(const int64_t* h_degrees, int64_t n_entities, int32_t m,
                                int32_t strategy, int32_t* h_assignment, int64_t* h_loads) {
  try {
    if (n_entities < 0 || m < 1 || (n_entities > 0 && (!h_degrees || !h_assignment)) || !h_loads) {
      th::set_error("bad planner arguments");
      return TH_ERR_INVALID;
    }
    std::fill(h_loads, h_loads + m, int64_t(0));
    if (strategy == TH_PLAN_HASH) {
      for (int64_t e = 0; e < n_entities; ++e) {
        if (h_degrees[e] <= 0) {
          h_assignment[e] = -1;
          continue;
        }
        const uint32_t h = (uint32_t)((uint64_t)e * 0x9E3779B1ull);
        const int32_t p = (int32_t)(h % (uint32_t)m);
        h_assignment[e] = p;
        h_loads[p] += h_degrees[e];
      }
      return TH_OK;
    }
    if (strategy != TH_PLAN_LPT) {
      th::set_error("unknown planner strategy");
      return TH_ERR_INVALID;
    }
    std::vector<int32_t> subjects;
    subjects.reserve((size_t)n_entities);
    for (int64_t e = 0; e < n_entities; ++e) {
      h_assignment[e] = -1;
      if (h_degrees[e] > 0) subjects.push_back((int32_t)e);
    }
    // heaviest first, ties by smaller id (stable on the ascending id list)
    std::stable_sort(subjects.begin(), subjects.end(),
                     [&](int32_t a, int32_t b) { return h_degrees[a] > h_degrees[b]; });
    MinTree tree(m);
    for (const int32_t e : subjects) {
      const int32_t p = tree.top();
      h_assignment[e] = p;
      tree.add(p, h_degrees[e]);
    }
    for (int p = 0; p < m; ++p) h_loads[p] = tree.load[p];
    return TH_OK;
  } catch (const std::bad_alloc&) {
    th::set_error("host allocation failed");
    return TH_ERR_NOMEM;
  }
}
