// Batched multi-source k-hop engine (K2 push, K3 pull, K4 canonicalise).
#pragma once
#include <stdint.h>

#include <vector>

#include "../../include/th_b200.h"
#include "graph.cuh"

namespace th {

constexpr int kMaxK = 32;
constexpr int kMaxWave = 1024;  // queries per wave = bits per entity row

// device control block of one wave
struct Ctl {
  int32_t list_len[kMaxK + 2];
  int64_t list_off[kMaxK + 2];
  unsigned long long push_cost[kMaxK + 2];
  int32_t mode[kMaxK + 2];  // 0 = push, 1 = pull
  int32_t heavy_len;
  int32_t err;
  int64_t ids_used;
  int64_t act_used;
  int32_t push_hops, pull_hops;
  int64_t path_used;
  int32_t mat_rows;  // length of the compacted row list of the layer being materialised
};

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Session {
  Graph* g = nullptr;
  cudaStream_t st = nullptr;
  double pull_divisor = 8.0;
  int64_t list_min_entities = int64_t(4) << 20;  // K4 list-driven above this E
  int64_t launches = 0;
  // wave state
  DBuf X, N, V, S, Xf, Nf, Vf, lists, heavy, M, counts, totals, rowlist, rowscan;
  DBuf ctl;
  // outputs
  DBuf f_off, f_len, f_ids, a_off, a_len, a_ids, edges, p_off, p_cnt, p_trunc, p_tids, p_scratch;
  int64_t f_cap = 0, a_cap = 0, p_cap = 0;
  // last run
  th_query last{};
  bool has_run = false;
  int64_t last_f_need = 0, last_a_need = 0, last_p_need = 0;
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> pending_cat;
  std::vector<int64_t> pending_launch;
  size_t ev_used = 0;
  double prof_ms[TH_PROF_CATEGORIES] = {};
  int64_t prof_launches[TH_PROF_CATEGORIES] = {};
  int64_t wave_lists[kMaxK + 2] = {};
  int last_k = 0;
};

// RAII timing scope for one kernel group
struct ProfScope {
  Session* s;
  int cat;
  int64_t l0;
  ProfScope(Session* s_, int c);
  ~ProfScope() noexcept(false);
};

int session_profile(Session* s, double* ms, int64_t* launches, int n);
int session_wave_lists(Session* s, int64_t* lens, int n);

int session_run(Session* s, const th_query* q);
int session_finish(Session* s, th_result* out);
void session_free(Session* s);
void plan_owner_hash(const Graph* g, int32_t m, int32_t* d_owner, cudaStream_t st);

}  // namespace th
