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
  unsigned long long sent[kMaxK + 2];  // shards: records written to other ranks' inboxes per hop
  int32_t mode[kMaxK + 2];  // 0 = push, 1 = pull
  int32_t dense[kMaxK + 2]; // pull hop over a frontier that sources most in-edges
  int32_t pull_items[kMaxK + 2];  // two-phase pull: items the screen kept per hop
  int32_t heavy_len;
  int32_t err;
  int64_t ids_used;
  int64_t act_used;
  int32_t push_hops, pull_hops;
  int64_t path_used;
  int32_t mat_rows;  // length of the compacted row list of the layer being materialised
  int32_t olen;      // shards: staged remote rows this hop
  int32_t mat_rows2; // compacted row count of the second K4 slot
};

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

// shape of a run a captured CUDA graph is valid for (engine.cu run_graphed)
struct GraphKey {
  int64_t B, k, semantics, flags, mask_words, max_paths, f_cap, a_cap, p_cap, list_min, knobs;
  double pull_divisor, dense_pull;
  uint64_t epoch;
  bool operator==(const GraphKey& o) const {
    return B == o.B && k == o.k && semantics == o.semantics && flags == o.flags &&
           mask_words == o.mask_words && max_paths == o.max_paths && f_cap == o.f_cap &&
           a_cap == o.a_cap && p_cap == o.p_cap && list_min == o.list_min && knobs == o.knobs &&
           pull_divisor == o.pull_divisor && dense_pull == o.dense_pull && epoch == o.epoch;
  }
};

struct Session {
  Graph* g = nullptr;
  cudaStream_t st = nullptr;
  double pull_divisor = 8.0;
  double dense_pull = 2.0;  // pull hops gather unconditionally above 1/dense_pull active in-edges
  int64_t list_min_entities = int64_t(4) << 20;  // K4 list-driven above this E
  // shards: K4 covers rows [0, mat_rows) (owned entities) and maps rows /
  // local triples to global ids; defaults cover the whole single graph
  // K4 of hop h overlaps hop h+1's expansion on a side stream (frontier-only
  // runs; the main stream joins before it recycles the layer's rows)
  bool overlap = true;
  bool k4_cache = true;
  bool paths_k2 = true;     // k = 2 singleton capped path queries: a CTA per query (paths.cu)
  // pull items screened first: -1 by graph shape, 0 off, 1 per lane inside the
  // pull kernel, 2 a separate edge-parallel screen kernel + a compacted pull
  int pull_screen = -1;
  int k4_mode = 1;  // count pass: 0 word-per-warp, 1 row-major for list-driven layers, 2 for all (k4_rowmajor.cuh)
  // captured waves: the hop chain's kernels get the device's highest stream
  // priority and K4's side streams the lowest, so the block scheduler feeds
  // the critical path first and K4 fills the gaps
  bool priority = true;
  bool k4_bucket = true;  // list-driven layers: scatter/gather write pass (k4_rowmajor.cuh)
  bool pull_pair = true;  // two-phase pull gather: two target rows per lane group in flight
  // filtered waves' layers (no fused edge sums) cache their masks too: off --
  // their layers are sparse, and the bit-sliced count + transposing write
  // beat storing and re-reading the masks (C3 3.84 -> ~3.6 ms)
  bool k4_cache_filtered = false;
  bool list_first_hop = true;  // K4 of hop 1 follows the compacted row list  // small layers: count pass caches tile masks for the write pass
  cudaStream_t side = nullptr, side2 = nullptr;  // K4 streams (odd / even layers)
  int k4_slot = 0;                                // which K4 scratch set is in use
  cudaEvent_t ev_expand[kMaxK + 2] = {};
  cudaEvent_t ev_mat[kMaxK + 2] = {};
  cudaEvent_t ev_cnt[kMaxK + 2] = {};  // K4 of the layer no longer reads it (count pass done)
  cudaEvent_t mark_counted = nullptr;  // set by run_wave around a K4 call
  bool counted_recorded = false;
  int64_t mat_rows = -1;
  const int32_t* row_map = nullptr;
  const int32_t* tid_map = nullptr;
  int64_t launches = 0;
  // wave state
  DBuf X, N, V, S, Xf, Nf, Vf, lists, heavy, M, counts, totals, rowlist, rowscan, k4_S, k4_meta, heavy_off;
  DBuf counts2, totals2, rowlist2, rowscan2, k4_S2, k4_meta2;  // second K4 slot
  DBuf k4_P, k4_G, k4_P2, k4_G2;
  DBuf pull_items;  // two-phase pull: the screened items (v, lo, hi)  // bucketed write pass: entries, group counts (per slot)
  DBuf ctl;
  // outputs
  DBuf f_off, f_len, f_ids, a_off, a_len, a_ids, edges, p_off, p_cnt, p_trunc, p_tids, p_scratch, p_tmp;
  int64_t f_cap = 0, a_cap = 0, p_cap = 0;
  // last run
  th_query last{};
  bool has_run = false;
  int64_t last_f_need = 0, last_a_need = 0, last_p_need = 0;
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> pending_cat;
  std::vector<int> pending_tag;     // stream of each scope: 0 main, 1/2 the K4 side streams
  std::vector<int64_t> pending_launch;
  std::vector<double> prof_trace;   // last drained run: (category, stream, start ms, end ms) per scope
  size_t ev_used = 0;
  double prof_ms[TH_PROF_CATEGORIES] = {};
  int64_t prof_launches[TH_PROF_CATEGORIES] = {};
  int64_t wave_lists[kMaxK + 2] = {};
  int last_k = 0;
  // CUDA-graph replay of repeated shapes
  bool use_graphs = true;
  cudaStream_t cap = nullptr;       // capture stream
  bool capturing = false;
  DBuf in_offs, in_seeds, in_masks;
  cudaGraphExec_t gexec = nullptr;
  GraphKey gkey{};
  bool g_seen = false, g_valid = false;
  int64_t g_launches = 0;
  std::vector<int> g_pend_cat;     // profile scopes the graph records
  std::vector<int> g_pend_tag;
  std::vector<int64_t> g_pend_launch;
  size_t g_ev_used = 0;
  int g_failures = 0;               // captures that fell back to eager runs
};

// RAII timing scope for one kernel group
struct ProfScope {
  Session* s;
  int cat;
  int tag = 0;
  int64_t l0;
  ProfScope(Session* s_, int c);
  ~ProfScope() noexcept(false);
};

int session_profile(Session* s, double* ms, int64_t* launches, int n);
int64_t session_profile_trace(Session* s, double* out4, int64_t cap);
int session_wave_lists(Session* s, int64_t* lens, int n);
int session_wave_modes(Session* s, int32_t* modes, int n);

int session_run(Session* s, const th_query* q);
int session_finish(Session* s, th_result* out);
void session_free(Session* s);
void plan_owner_hash(const Graph* g, int32_t m, int32_t* d_owner, cudaStream_t st);

// ---- K6 partitioned graphs (one rank's shard; see k6_shard.cuh) ----
struct Shard;
int shard_create(Shard** out, const int32_t* d_subj, const int32_t* d_rel, const int32_t* d_obj,
                 int64_t T, int64_t E, int64_t R, const int32_t* d_lidx,
                 const int32_t* d_hub_index, const int32_t* d_hub_ids, int64_t H,
                 const int32_t* d_l2g, int64_t n_local, int32_t rank, int32_t world,
                 int64_t inbox_records, cudaStream_t st);
int64_t shard_local_triples(const Shard* sh);
int shard_region(const Shard* sh, void** base, uint64_t* bytes, int64_t* records);
int shard_ipc_handle(const Shard* sh, void* out64);
int shard_connect(Shard* sh, int32_t peer, void* base, bool ipc);
int shard_ipc_open(Shard* sh, int32_t peer, const void* handle64);
int shard_grow_inbox(Shard* sh, int64_t records);
int shard_inbox_overflowed(const Shard* sh);
void shard_set_pull_divisor(Shard* sh, double d);
int shard_begin(Shard* sh, const th_query* q);
int shard_hop(Shard* sh, int h, int phase);
int shard_can_pull(const Shard* sh);
int shard_finish(Shard* sh, th_result* out);
int shard_sent(Shard* sh, int64_t* per_hop, int n);
int shard_columns(const Shard* sh, th_shard_cols* out);
Session* shard_session(Shard* sh);
struct HubCache;
int shard_hub_cache(Shard* sh, int64_t capacity);
// an in-process world's whole wave (begin + every hop), graph-captured per shape
int shards_run_wave(Shard* const* sh, int n, const th_query* q, const int64_t* n_seeds);
HubCache* shard_hub_cache_of(Shard* sh);
void shard_free(Shard* sh);

}  // namespace th
