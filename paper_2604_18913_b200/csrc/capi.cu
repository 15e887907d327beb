// extern "C" boundary (include/th_b200.h).  No C++ exception crosses it:
// every entry point converts failures into a status code plus a
// thread-local message (th_last_error).
#include <cstdlib>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/th_b200.h"
#include "engine.cuh"
#include "graph.cuh"
#include "hubcache.cuh"
#include "idset.cuh"

struct th_graph {
  th::Graph g;
};
struct th_session {
  th::Session s;
};
struct th_shard {
  th::Shard* sh = nullptr;
};

namespace th {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace th

namespace {

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const th::CudaError& e) {
    th::set_error(std::string(e.where) + ": " + cudaGetErrorString(e.code));
    return e.code == cudaErrorMemoryAllocation ? TH_ERR_NOMEM : TH_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    th::set_error("host allocation failed");
    return TH_ERR_NOMEM;
  } catch (const std::exception& e) {
    th::set_error(e.what());
    return TH_ERR_STATE;
  }
}

}  // namespace

extern "C" {

int th_abi_version(void) { return TH_ABI_VERSION; }

const char* th_last_error(void) { return th::g_last_error.c_str(); }

int th_graph_create(const int32_t* d_subj, const int32_t* d_rel, const int32_t* d_obj,
                    int64_t n_triples, int64_t n_entities, int64_t n_relations, uint32_t flags,
                    void* stream, th_graph** out) {
  return guarded([&]() -> int {
    if (!out) {
      th::set_error("out is NULL");
      return TH_ERR_INVALID;
    }
    *out = nullptr;
    if (n_triples < 0 || n_entities < 0 || n_relations < 0) {
      th::set_error("negative size");
      return TH_ERR_INVALID;
    }
    if (n_triples >= INT32_MAX || n_entities >= INT32_MAX) {
      th::set_error("int32 id space exceeded (n_triples, n_entities < 2^31-1)");
      return TH_ERR_INVALID;
    }
    if (n_relations > 65535) {
      th::set_error("relation ids are stored as uint16 (n_relations <= 65535)");
      return TH_ERR_INVALID;
    }
    if (n_triples > 0 && (!d_subj || !d_rel || !d_obj)) {
      th::set_error("NULL triple column");
      return TH_ERR_INVALID;
    }
    auto* h = new th_graph();
    const int rc = th::graph_build(&h->g, d_subj, d_rel, d_obj, n_triples, n_entities, n_relations,
                                   !(flags & TH_GRAPH_NO_REVERSE),
                                   static_cast<cudaStream_t>(stream));
    if (rc != TH_OK) {
      th::graph_free(&h->g);
      delete h;
      return rc;
    }
    *out = h;
    return TH_OK;
  });
}

int th_graph_create_lkg(const void* d_indptr, const void* d_tids, const void* d_obj,
                        const void* d_rel, int32_t id_width, int64_t n_triples,
                        int64_t n_entities, int64_t n_relations, uint32_t flags, void* stream,
                        th_graph** out) {
  return guarded([&]() -> int {
    if (!out) {
      th::set_error("out is NULL");
      return TH_ERR_INVALID;
    }
    *out = nullptr;
    if (id_width != 4 && id_width != 8) {
      th::set_error("unsupported id width " + std::to_string(id_width));
      return TH_ERR_DATA;
    }
    if (n_triples < 0 || n_entities < 0 || n_relations < 0) {
      th::set_error("negative size");
      return TH_ERR_INVALID;
    }
    if (n_triples >= INT32_MAX || n_entities >= INT32_MAX || n_relations > 65535) {
      th::set_error("archive exceeds the device id space (int32 entities/triples, uint16 relations)");
      return TH_ERR_INVALID;
    }
    if (!d_indptr || (n_triples > 0 && (!d_tids || !d_obj || !d_rel))) {
      th::set_error("NULL payload array");
      return TH_ERR_INVALID;
    }
    auto* h = new th_graph();
    const int rc = th::graph_build_lkg(&h->g, d_indptr, d_tids, d_obj, d_rel, id_width, n_triples,
                                       n_entities, n_relations, !(flags & TH_GRAPH_NO_REVERSE),
                                       static_cast<cudaStream_t>(stream));
    if (rc != TH_OK) {
      th::graph_free(&h->g);
      delete h;
      return rc;
    }
    *out = h;
    return TH_OK;
  });
}

int th_graph_destroy(th_graph* g) {
  return guarded([&]() -> int {
    if (!g) return TH_OK;
    th::graph_free(&g->g);
    delete g;
    return TH_OK;
  });
}

int th_graph_info_get(const th_graph* gh, th_graph_info* out) {
  if (!gh || !out) {
    th::set_error("NULL handle");
    return TH_ERR_INVALID;
  }
  const th::Graph& g = gh->g;
  out->n_entities = g.E;
  out->n_triples = g.T;
  out->n_relations = g.R;
  out->indptr = g.indptr;
  out->csr_tid = g.csr_tid;
  out->csr_obj = g.csr_obj;
  out->csr_rel = g.csr_rel;
  out->subj = g.subj;
  out->obj = g.obj;
  out->rel = g.rel;
  out->rindptr = g.rindptr;
  out->rsrc = g.rsrc;
  out->rrel = g.rrel;
  out->max_out_degree = g.max_out;
  out->max_in_degree = g.max_in;
  out->n_heavy_in = g.n_split;
  out->device_bytes = g.bytes;
  return TH_OK;
}

int th_session_create(th_graph* g, void* stream, th_session** out) {
  return guarded([&]() -> int {
    if (!g || !out) {
      th::set_error("NULL handle");
      return TH_ERR_INVALID;
    }
    auto* s = new th_session();
    s->s.g = &g->g;
    s->s.st = static_cast<cudaStream_t>(stream);
    *out = s;
    return TH_OK;
  });
}

int th_session_destroy(th_session* s) {
  return guarded([&]() -> int {
    if (!s) return TH_OK;
    th::session_free(&s->s);
    delete s;
    return TH_OK;
  });
}

int th_run(th_session* s, const th_query* q) {
  return guarded([&]() -> int {
    if (!s || !q) {
      th::set_error("NULL handle");
      return TH_ERR_INVALID;
    }
    return th::session_run(&s->s, q);
  });
}

int th_finish(th_session* s, th_result* out) {
  return guarded([&]() -> int {
    if (!s || !out) {
      th::set_error("NULL handle");
      return TH_ERR_INVALID;
    }
    return th::session_finish(&s->s, out);
  });
}

int th_session_set_pull_divisor(th_session* s, double pull_divisor) {
  if (!s) {
    th::set_error("NULL handle");
    return TH_ERR_INVALID;
  }
  s->s.pull_divisor = pull_divisor;
  return TH_OK;
}

int th_session_set_dense_pull(th_session* s, double divisor) {
  if (!s) {
    th::set_error("NULL handle");
    return TH_ERR_INVALID;
  }
  s->s.dense_pull = divisor;
  return TH_OK;
}

int th_session_set_list_min_entities(th_session* s, int64_t min_entities) {
  if (!s) {
    th::set_error("NULL handle");
    return TH_ERR_INVALID;
  }
  s->s.list_min_entities = min_entities;
  return TH_OK;
}

int th_session_set_graphs(th_session* s, int on) {
  if (!s) {
    th::set_error("NULL handle");
    return TH_ERR_INVALID;
  }
  s->s.use_graphs = on != 0;
  return TH_OK;
}

int th_session_set_overlap(th_session* s, int on) {
  if (!s) {
    th::set_error("NULL handle");
    return TH_ERR_INVALID;
  }
  s->s.overlap = on != 0;
  return TH_OK;
}

int th_session_set_k4_mode(th_session* s, int mode) {
  if (!s || mode < 0 || mode > 2) {
    th::set_error(!s ? "NULL handle" : "k4 mode must be 0, 1 or 2");
    return TH_ERR_INVALID;
  }
  s->s.k4_mode = mode;
  return TH_OK;
}

int th_session_set_pull_screen(th_session* s, int mode) {
  if (!s || mode < -1 || mode > 2) {
    th::set_error(!s ? "NULL handle" : "pull screen mode must be -1, 0, 1 or 2");
    return TH_ERR_INVALID;
  }
  s->s.pull_screen = mode;
  return TH_OK;
}

int th_session_set_knob(th_session* s, const char* name, int64_t value) {
  if (!s || !name) {
    th::set_error("NULL argument");
    return TH_ERR_INVALID;
  }
  const std::string n(name);
  if (n == "paths_k2") {
    s->s.paths_k2 = value != 0;
  } else if (n == "k4_cache") {
    s->s.k4_cache = value != 0;
  } else if (n == "list_first_hop") {
    s->s.list_first_hop = value != 0;
  } else if (n == "priority") {
    s->s.priority = value != 0;
  } else if (n == "k4_bucket") {
    s->s.k4_bucket = value != 0;
  } else if (n == "pull_pair") {
    s->s.pull_pair = value != 0;
  } else if (n == "k4_cache_filtered") {
    s->s.k4_cache_filtered = value != 0;
  } else {
    th::set_error("unknown knob " + n);
    return TH_ERR_INVALID;
  }
  return TH_OK;
}

int64_t th_session_launch_count(const th_session* s) { return s ? s->s.launches : -1; }

int th_session_set_profiling(th_session* s, int on) {
  if (!s) {
    th::set_error("NULL handle");
    return TH_ERR_INVALID;
  }
  s->s.prof = on != 0;
  return TH_OK;
}

int th_session_profile(th_session* s, double* ms, int64_t* launches, int n) {
  return guarded([&]() -> int {
    if (!s) {
      th::set_error("NULL handle");
      return TH_ERR_INVALID;
    }
    return th::session_profile(&s->s, ms, launches, n);
  });
}

int64_t th_session_profile_trace(th_session* s, double* h_out4, int64_t cap) {
  if (!s) return -1;
  int64_t n = -1;
  const int rc = guarded([&]() -> int {
    n = th::session_profile_trace(&s->s, h_out4, cap);
    return TH_OK;
  });
  return rc == TH_OK ? n : -1;
}

int th_session_wave_modes(const th_session* s, int32_t* modes, int n) {
  return guarded([&]() -> int {
    if (!s || !modes) {
      th::set_error("NULL handle");
      return TH_ERR_INVALID;
    }
    return th::session_wave_modes(const_cast<th::Session*>(&s->s), modes, n);
  });
}

int th_session_wave_lists(const th_session* s, int64_t* lens, int n) {
  return guarded([&]() -> int {
    if (!s || !lens) {
      th::set_error("NULL handle");
      return TH_ERR_INVALID;
    }
    return th::session_wave_lists(const_cast<th::Session*>(&s->s), lens, n);
  });
}

int th_plan_owner_hash(const th_graph* g, int32_t m, int32_t* d_owner, void* stream) {
  return guarded([&]() -> int {
    if (!g || !d_owner || m < 1) {
      th::set_error("bad arguments");
      return TH_ERR_INVALID;
    }
    th::plan_owner_hash(&g->g, m, d_owner, static_cast<cudaStream_t>(stream));
    return TH_OK;
  });
}

// ---- partitioned graphs ----------------------------------------------------

int th_shard_create(const int32_t* d_subj, const int32_t* d_rel, const int32_t* d_obj,
                    int64_t n_triples, int64_t n_entities, int64_t n_relations,
                    const int32_t* d_lidx, const int32_t* d_hub_index, const int32_t* d_hub_ids,
                    int64_t n_hubs, const int32_t* d_l2g, int64_t n_local, int32_t rank,
                    int32_t world, int64_t inbox_records, void* stream, th_shard** out) {
  return guarded([&]() -> int {
    if (!out) {
      th::set_error("out is NULL");
      return TH_ERR_INVALID;
    }
    *out = nullptr;
    if (n_triples < 0 || n_entities < 0 || n_relations < 0 || n_hubs < 0 || n_local < 0 ||
        n_local > n_entities || n_hubs > n_entities) {
      th::set_error("bad sizes");
      return TH_ERR_INVALID;
    }
    if (n_triples >= INT32_MAX || n_entities >= INT32_MAX || n_relations > 65535) {
      th::set_error("id space exceeded (int32 entities/triples, uint16 relations)");
      return TH_ERR_INVALID;
    }
    if (world < 1 || rank < 0 || rank >= world) {
      th::set_error("rank must be in [0, world)");
      return TH_ERR_INVALID;
    }
    if ((n_triples > 0 && (!d_subj || !d_rel || !d_obj)) ||
        (n_entities > 0 && (!d_lidx || !d_hub_index)) || (n_hubs > 0 && !d_hub_ids) ||
        (n_local > 0 && !d_l2g)) {
      th::set_error("NULL input array");
      return TH_ERR_INVALID;
    }
    auto* h = new th_shard();
    th::Shard* sh = nullptr;
    int rc = TH_OK;
    try {
      rc = th::shard_create(&sh, d_subj, d_rel, d_obj, n_triples, n_entities, n_relations, d_lidx,
                            d_hub_index, d_hub_ids, n_hubs, d_l2g, n_local, rank, world,
                            inbox_records, static_cast<cudaStream_t>(stream));
    } catch (...) {
      if (sh) th::shard_free(sh);
      delete h;
      throw;
    }
    if (rc != TH_OK) {
      if (sh) th::shard_free(sh);
      delete h;
      return rc;
    }
    h->sh = sh;
    *out = h;
    return TH_OK;
  });
}

int th_shard_destroy(th_shard* s) {
  if (!s) return TH_OK;
  if (s->sh) th::shard_free(s->sh);
  delete s;
  return TH_OK;
}

int64_t th_shard_local_triples(const th_shard* s) {
  return (s && s->sh) ? th::shard_local_triples(s->sh) : -1;
}

#define TH_SHARD_GUARD(s)            \
  if (!(s) || !(s)->sh) {            \
    th::set_error("NULL handle");    \
    return TH_ERR_INVALID;           \
  }

int th_shard_begin(th_shard* s, const th_query* q) {
  return guarded([&]() -> int {
    TH_SHARD_GUARD(s);
    if (!q) {
      th::set_error("NULL query");
      return TH_ERR_INVALID;
    }
    return th::shard_begin(s->sh, q);
  });
}

int th_shard_can_pull(const th_shard* s) { return (s && s->sh) ? th::shard_can_pull(s->sh) : 0; }

int th_shard_region(const th_shard* s, void** d_base, uint64_t* bytes, int64_t* inbox_records) {
  return guarded([&]() -> int {
    if (!s || !s->sh || !d_base || !bytes) {
      th::set_error("bad arguments");
      return TH_ERR_INVALID;
    }
    return th::shard_region(s->sh, d_base, bytes, inbox_records);
  });
}

int th_shard_ipc_handle(const th_shard* s, void* h_handle64) {
  return guarded([&]() -> int {
    if (!s || !s->sh || !h_handle64) {
      th::set_error("bad arguments");
      return TH_ERR_INVALID;
    }
    return th::shard_ipc_handle(s->sh, h_handle64);
  });
}

int th_shard_connect(th_shard* s, int32_t peer, void* d_peer_base) {
  return guarded([&]() -> int {
    if (!s || !s->sh || !d_peer_base) {
      th::set_error("bad arguments");
      return TH_ERR_INVALID;
    }
    return th::shard_connect(s->sh, peer, d_peer_base, false);
  });
}

int th_shard_ipc_open(th_shard* s, int32_t peer, const void* h_handle64) {
  return guarded([&]() -> int {
    if (!s || !s->sh || !h_handle64) {
      th::set_error("bad arguments");
      return TH_ERR_INVALID;
    }
    return th::shard_ipc_open(s->sh, peer, h_handle64);
  });
}

int th_shard_grow_inbox(th_shard* s, int64_t inbox_records) {
  return guarded([&]() -> int {
    if (!s || !s->sh || inbox_records < 1) {
      th::set_error("bad arguments");
      return TH_ERR_INVALID;
    }
    return th::shard_grow_inbox(s->sh, inbox_records);
  });
}

int th_shard_sent(th_shard* s, int64_t* h_per_hop, int n) {
  return guarded([&]() -> int {
    if (!s || !s->sh || !h_per_hop || n < 0) {
      th::set_error("bad arguments");
      return TH_ERR_INVALID;
    }
    return th::shard_sent(s->sh, h_per_hop, n);
  });
}

int th_shard_columns(const th_shard* s, th_shard_cols* out) {
  return guarded([&]() -> int {
    if (!s || !s->sh || !out) {
      th::set_error("bad arguments");
      return TH_ERR_INVALID;
    }
    return th::shard_columns(s->sh, out);
  });
}

int th_shard_inbox_overflowed(const th_shard* s) {
  return (s && s->sh) ? th::shard_inbox_overflowed(s->sh) : -1;
}

int th_shard_set_pull_divisor(th_shard* s, double pull_divisor) {
  if (!s || !s->sh) {
    th::set_error("NULL handle");
    return TH_ERR_INVALID;
  }
  th::shard_set_pull_divisor(s->sh, pull_divisor);
  return TH_OK;
}

int th_shard_hop(th_shard* s, int32_t hop, int32_t phase) {
  return guarded([&]() -> int {
    if (!s || !s->sh || phase < 0 || phase > 2) {
      th::set_error("bad arguments");
      return TH_ERR_INVALID;
    }
    return th::shard_hop(s->sh, hop, phase);
  });
}

int th_shard_finish(th_shard* s, th_result* out) {
  return guarded([&]() -> int {
    TH_SHARD_GUARD(s);
    if (!out) {
      th::set_error("NULL output");
      return TH_ERR_INVALID;
    }
    return th::shard_finish(s->sh, out);
  });
}

int th_shards_run_hops(th_shard* const* shards, int32_t n, int32_t k) {
  return guarded([&]() -> int {
    if (!shards || n < 1) {
      th::set_error("bad arguments");
      return TH_ERR_INVALID;
    }
    for (int32_t i = 0; i < n; ++i) TH_SHARD_GUARD(shards[i]);
    for (int32_t h = 1; h <= k; ++h)
      for (int32_t phase = 0; phase < 3; ++phase)
        for (int32_t i = 0; i < n; ++i) {
          const int rc = th::shard_hop(shards[i]->sh, h, phase);
          if (rc != TH_OK) return rc;
        }
    return TH_OK;
  });
}

int th_shards_run_wave(th_shard* const* shards, int32_t n, const th_query* queries,
                       const int64_t* h_n_seeds) {
  return guarded([&]() -> int {
    if (!shards || n < 1 || !queries || !h_n_seeds) {
      th::set_error("bad arguments");
      return TH_ERR_INVALID;
    }
    std::vector<th::Shard*> sh(n);
    for (int32_t i = 0; i < n; ++i) {
      TH_SHARD_GUARD(shards[i]);
      sh[i] = shards[i]->sh;
    }
    return th::shards_run_wave(sh.data(), n, queries, h_n_seeds);
  });
}

int th_shard_set_profiling(th_shard* s, int on) {
  TH_SHARD_GUARD(s);
  th::shard_session(s->sh)->prof = on != 0;
  return TH_OK;
}

int64_t th_shard_profile_trace(th_shard* s, double* h_out4, int64_t cap) {
  if (!s || !s->sh) return -1;
  int64_t n = -1;
  const int rc = guarded([&]() -> int {
    n = th::session_profile_trace(th::shard_session(s->sh), h_out4, cap);
    return TH_OK;
  });
  return rc == TH_OK ? n : -1;
}

int th_shard_hub_cache(th_shard* s, int64_t capacity_pages) {
  return guarded([&]() -> int {
    TH_SHARD_GUARD(s);
    return th::shard_hub_cache(s->sh, capacity_pages);
  });
}

int th_shard_hub_cache_stats(th_shard* s, int64_t* h_out8) {
  TH_SHARD_GUARD(s);
  th::HubCache* hc = th::shard_hub_cache_of(s->sh);
  if (!hc || !h_out8) {
    th::set_error(hc ? "NULL output" : "the shard has no hub cache (th_shard_hub_cache)");
    return hc ? TH_ERR_INVALID : TH_ERR_STATE;
  }
  th::hubcache_stats(hc, h_out8);
  return TH_OK;
}

int64_t th_shard_hub_cache_trace(th_shard* s, int64_t* h_out, int64_t cap) {
  th::HubCache* hc = (s && s->sh) ? th::shard_hub_cache_of(s->sh) : nullptr;
  return hc ? th::hubcache_trace(hc, h_out, cap) : -1;
}

int64_t th_shard_hub_cache_resident(th_shard* s, int64_t* h_out, int64_t cap) {
  th::HubCache* hc = (s && s->sh) ? th::shard_hub_cache_of(s->sh) : nullptr;
  return hc ? th::hubcache_resident(hc, h_out, cap) : -1;
}

// ---- id sets (store-backed partitioned retrieval) ----

#define TH_NONNULL(p)                 \
  do {                                \
    if (!(p)) {                       \
      th::set_error("NULL argument"); \
      return TH_ERR_INVALID;          \
    }                                 \
  } while (0)

int th_ids_route_count(const int32_t* d_assign, int64_t n_entities, const int32_t* d_ids, int64_t n,
                       int32_t m, int64_t* d_counts, void* stream) {
  return guarded([&]() -> int {
    TH_NONNULL(d_assign);
    TH_NONNULL(d_counts);
    if (n > 0) TH_NONNULL(d_ids);
    const int rc = th::ids_route_count(d_assign, n_entities, d_ids, n, m, d_counts,
                                       static_cast<cudaStream_t>(stream));
    if (rc != TH_OK) th::set_error("id out of range for the partition plan");
    return rc;
  });
}

int th_ids_map_scatter(const int32_t* d_map, int64_t map_len, const int32_t* d_ids, int64_t n,
                       uint32_t* d_bits, int64_t nbits, void* stream) {
  return guarded([&]() -> int {
    TH_NONNULL(d_bits);
    if (n > 0) TH_NONNULL(d_ids);
    const int rc = th::ids_map_scatter(d_map, map_len, d_ids, n, d_bits, nbits,
                                       static_cast<cudaStream_t>(stream));
    if (rc != TH_OK) th::set_error("id out of range for the map or bitmap");
    return rc;
  });
}

int th_ids_to_local_bits(const int32_t* d_sorted_map, int64_t map_len, const int32_t* d_ids,
                         int64_t n, uint32_t* d_bits, void* stream) {
  return guarded([&]() -> int {
    TH_NONNULL(d_bits);
    if (n > 0) TH_NONNULL(d_ids);
    if (map_len > 0) TH_NONNULL(d_sorted_map);
    return th::ids_to_local_bits(d_sorted_map, map_len, d_ids, n, d_bits,
                                 static_cast<cudaStream_t>(stream));
  });
}

int th_bits_andnot_update(uint32_t* d_fresh, uint32_t* d_visited, int64_t nbits, void* stream) {
  return guarded([&]() -> int {
    TH_NONNULL(d_fresh);
    TH_NONNULL(d_visited);
    return th::bits_andnot_update(d_fresh, d_visited, nbits, static_cast<cudaStream_t>(stream));
  });
}

int th_bits_or(uint32_t* d_dst, const uint32_t* d_src, int64_t nbits, void* stream) {
  return guarded([&]() -> int {
    TH_NONNULL(d_dst);
    TH_NONNULL(d_src);
    return th::bits_or(d_dst, d_src, nbits, static_cast<cudaStream_t>(stream));
  });
}

int th_bits_compact(const uint32_t* d_bits, int64_t nbits, int32_t* d_out, int64_t cap,
                    int64_t* n_out, void* stream) {
  return guarded([&]() -> int {
    TH_NONNULL(d_bits);
    TH_NONNULL(n_out);
    if (cap > 0) TH_NONNULL(d_out);
    const int rc = th::bits_compact(d_bits, nbits, d_out, cap, n_out, static_cast<cudaStream_t>(stream));
    if (rc == TH_ERR_OVERFLOW) th::set_error("id list longer than the output capacity");
    return rc;
  });
}

int64_t th_shard_launch_count(const th_shard* s) {
  return (s && s->sh) ? th::shard_session(s->sh)->launches : -1;
}

}  // extern "C"
