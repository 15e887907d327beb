/*
 * th_b200.h -- C ABI of the B200-native k-hop retrieval engine.
 *
 * Drop-in boundary for the hot path of the reference `triplehop` package
 * (/root/reference/pkg/src/triplehop).  The reference is pure Python/numpy
 * and has no FFI of its own; these entry points are what its Python layer
 * binds (through ctypes) in place of the numpy code:
 *
 *   th_graph_create   <- build_incidence            incidence.py:154-196
 *   th_run (frontiers, activated, edge counts)
 *                     <- k_hop / run_hops / _expand incidence.py:214-221,268-330
 *                        one_hop                    incidence.py:224-232
 *   th_run (paths)    <- reconstruct_paths / assemble_paths
 *                                                   incidence.py:361-408
 *   th_plan_owner     <- plan_partitions            partition.py:49-98
 *   th_shard_*        <- materialize_subgraphs / route / _partitioned_expand /
 *                        cross_graph_k_hop          partition.py:101-181,
 *                                                   engine.py:94-154
 *                        (ranks exchange through each other's device memory)
 *
 * Conventions
 *   - plain C types only; every pointer argument documented as device (d_)
 *     or host (h_); int status return (TH_OK == 0); no exceptions cross the
 *     ABI; th_last_error() gives a thread-local message for the last failure.
 *   - every call that launches work takes the CUDA stream (cudaStream_t passed
 *     as void*) and is asynchronous unless documented otherwise.
 *   - the graph is immutable after creation and may be shared by sessions on
 *     different streams; a session owns all per-query workspace and results
 *     (results stay valid until the next th_run on that session).
 */
#ifndef TH_B200_H
#define TH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TH_ABI_VERSION 1

/* status codes (Python mapping in paper_2604_18913_b200/_lib.py) */
#define TH_OK 0
#define TH_ERR_INVALID 1  /* contract violation          -> ValueError    */
#define TH_ERR_RANGE 2    /* id out of range             -> ValueError    */
#define TH_ERR_CUDA 3     /* CUDA runtime failure        -> RuntimeError  */
#define TH_ERR_NOMEM 4    /* device allocation failed    -> MemoryError   */
#define TH_ERR_OVERFLOW 5 /* result capacity too small: call th_run again  */
#define TH_ERR_STATE 6    /* misuse of handles           -> RuntimeError  */
#define TH_ERR_DATA 7     /* malformed archive payload   -> ArchiveError  */

/* hop semantics, incidence.py:52-75 */
#define TH_EXACT 0
#define TH_FRONTIER 1
#define TH_CUMULATIVE 2

/* th_query.flags */
#define TH_WANT_FRONTIERS 0x1u /* per-query sorted frontier ids per hop      */
#define TH_WANT_ACTIVATED 0x2u /* per-query sorted activated triple ids/hop  */
#define TH_WANT_PATHS 0x4u     /* capped lexicographic walk enumeration       */
#define TH_SINGLETON_SEEDS 0x8u /* every query is one seed (retrieve(seeds)):
                                   query q = {d_seeds[q]}, d_seeds holds
                                   n_queries ids and d_seed_offsets is NOT
                                   read; paths start from the seed's CSR row */

/* th_graph_create flags */
#define TH_GRAPH_NO_REVERSE 0x1u /* skip the reverse (by-object) CSR: no pull hops */

typedef struct th_graph th_graph;
typedef struct th_session th_session;

int th_abi_version(void);
const char* th_last_error(void);

/* ---- graph ------------------------------------------------------------- */

/* Build the device incidence structure from (subject, relation, object)
 * columns in triple-id order (d_ int32, n_triples long).  Ids are range
 * checked (TH_ERR_RANGE, incidence.py:175-179).  Synchronises `stream`. */
int th_graph_create(const int32_t* d_subj, const int32_t* d_rel, const int32_t* d_obj,
                    int64_t n_triples, int64_t n_entities, int64_t n_relations,
                    uint32_t flags, void* stream, th_graph** out);
int th_graph_destroy(th_graph* g);

/* Build from the payload of an LKG1 archive (archive.py:1-24,66-133) copied
 * verbatim to the device: d_indptr = u64[E+1] row offsets, d_tids = the
 * row-ordered triple ids, d_obj / d_rel in triple-id order, each id_width
 * (4 or 8) bytes.  The header and CRC32 are the host's job.  Structural
 * errors (offsets, permutation, ranges, row order) return TH_ERR_DATA with
 * the reference's message.  Synchronises `stream`. */
int th_graph_create_lkg(const void* d_indptr, const void* d_tids, const void* d_obj,
                        const void* d_rel, int32_t id_width, int64_t n_triples,
                        int64_t n_entities, int64_t n_relations, uint32_t flags, void* stream,
                        th_graph** out);

typedef struct {
  int64_t n_entities, n_triples, n_relations;
  const int32_t* indptr;   /* [E+1] subject CSR row offsets                 */
  const int32_t* csr_tid;  /* [T] triple id per CSR slot, ascending per row */
  const int32_t* csr_obj;  /* [T] object per CSR slot                       */
  const uint16_t* csr_rel; /* [T] relation per CSR slot                     */
  const int32_t* subj;     /* [T] triple-id order                           */
  const int32_t* obj;      /* [T]                                           */
  const uint16_t* rel;     /* [T]                                           */
  const int32_t* rindptr;  /* [E+1] object CSR (NULL with NO_REVERSE)       */
  const int32_t* rsrc;     /* [T] subject of each in-edge                   */
  const uint16_t* rrel;    /* [T] relation of each in-edge                  */
  int64_t max_out_degree, max_in_degree;
  int64_t n_heavy_in;      /* in-rows split across warps in pull hops       */
  uint64_t device_bytes;
} th_graph_info;
int th_graph_info_get(const th_graph* g, th_graph_info* out);

/* ---- queries ------------------------------------------------------------ */

/* B queries; query q starts from the entity set
 * d_seeds[d_seed_offsets[q] .. d_seed_offsets[q+1]) (any order, duplicates
 * allowed).  retrieve(seeds) uses one singleton query per seed. */
typedef struct {
  int32_t n_queries;
  const int32_t* d_seed_offsets; /* [B+1] */
  const int32_t* d_seeds;
  int32_t k;          /* hops, >= 1 (incidence.py:282-283) */
  int32_t semantics;  /* TH_EXACT / TH_FRONTIER / TH_CUMULATIVE */
  const uint32_t* d_rel_masks; /* [B][mask_words] bit r = relation r allowed; NULL = all */
  int32_t mask_words;
  uint32_t flags;     /* TH_WANT_* */
  int64_t max_paths;  /* >= 0, or -1 for uncapped (max_paths=None) */
} th_query;

/* Device-resident results of the last th_run on a session.
 * Frontier of query q at hop h (1-based):
 *   frontier_ids[frontier_off[(h-1)*B+q] .. +frontier_len[(h-1)*B+q]]
 * (segments are found through the offsets only: their placement in the id
 * array may differ from run to run; their contents are deterministic)
 * Activated triples likewise with act_*.  Paths of query q:
 *   path_tids[(path_off[q] + i) * k + d], i < path_count[q], d < k. */
typedef struct {
  int32_t n_queries, k;
  const int64_t* frontier_off; const int64_t* frontier_len; const int32_t* frontier_ids;
  const int64_t* act_off;      const int64_t* act_len;      const int32_t* act_ids;
  const int64_t* edges;        /* [k][B] |T_h(q)| = edges traversed (app.py:97) */
  const int64_t* path_off;     const int64_t* path_count;   const uint8_t* path_truncated;
  const int32_t* path_tids;
  /* host-side totals, valid after th_finish */
  int64_t frontier_total, act_total, path_total;
  int32_t push_hops, pull_hops; /* direction choices taken (diagnostics) */
} th_result;

int th_session_create(th_graph* g, void* stream, th_session** out);
int th_session_destroy(th_session* s);

/* Enqueue one query batch on the session stream (asynchronous). */
int th_run(th_session* s, const th_query* q);
/* Synchronise the stream and describe the results.  Returns TH_ERR_OVERFLOW
 * when an output buffer was too small; capacities have then been grown and
 * the same th_run must be issued again.  TH_ERR_RANGE for a bad seed id. */
int th_finish(th_session* s, th_result* out);

/* Tuning knobs (diagnostics / benchmarks): pull when the frontier's
 * out-edge total exceeds n_triples / pull_divisor; 0 = never pull,
 * <0 = always pull. */
int th_session_set_pull_divisor(th_session* s, double pull_divisor);
/* K4 materialisation strategy: graphs with at least `min_entities` entities
 * first compact each layer's flag bitmap into an ascending row list (work
 * follows the reached rows); smaller graphs scan the flag bitmap directly.
 * Default 4 Mi.  0 = always list-driven. */
int th_session_set_list_min_entities(th_session* s, int64_t min_entities);
/* Overlap hop h's frontier materialisation (K4) with hop h+1's expansion
 * on an internal stream (frontier-only runs).  Default on. */
int th_session_set_overlap(th_session* s, int on);
/* K4 count pass: 0 = word-per-warp loads with bit transposes everywhere;
 * 1 = row-major (whole-row loads, carry-save bit counting) for list-driven
 * layers without fused edge counts (default); 2 = row-major for every
 * entity layer (no mask cache for small dense layers). */
int th_session_set_k4_mode(th_session* s, int mode);
/* Pull hops screen their in-row items for a frontier in-edge before lane
 * groups expand the survivors: -1 = when the graph's mean in-edges per pull
 * item is below 4 (default; as mode 2), 0 = never, 1 = one item per lane
 * inside the pull kernel, 2 = a separate edge-parallel screen kernel that
 * compacts the surviving items, then the pull over that list. */
int th_session_set_pull_screen(th_session* s, int mode);
/* Boolean strategy knobs by name (A/B and tests): "paths_k2" (k = 2
 * singleton capped path queries on a CTA each; default 1), "k4_cache"
 * (small dense layers cache their tile masks; 1), "list_first_hop" (the
 * first layer's overlapped K4 follows its row list; 1), "priority" (the
 * hop chain at the highest stream priority; 1), "k4_bucket" (list-driven
 * layers up to 20M ids take the bucketed write; 1), "pull_pair" (the
 * two-phase pull's gather keeps two target rows per lane group in flight;
 * 1), "k4_cache_filtered" (relation-filtered waves' layers cache their
 * masks too when "k4_cache" is on; 0). */
int th_session_set_knob(th_session* s, const char* name, int64_t value);
/* Pull hops whose frontier sources more than 1/divisor of all in-edges
 * (by the frontier's out-degree sum) gather every in-neighbour row instead
 * of testing frontier flags first (default 2; <= 0 never). */
int th_session_set_dense_pull(th_session* s, double divisor);
/* CUDA-graph replay (default on): a TH_SINGLETON_SEEDS query with the same
 * shape (B, k, semantics, flags, masks, max_paths, capacities, knobs) as the
 * previous run is captured once and then replayed as one graph launch.
 * Inputs are copied into session buffers first, so callers may reuse or
 * free theirs after th_run as before.  Under profiling the timing events are
 * part of the graph; a run whose previous events were not yet drained
 * (th_finish / th_session_profile) runs eagerly. */
int th_session_set_graphs(th_session* s, int on);
/* Number of kernels this session has launched since creation. */
int64_t th_session_launch_count(const th_session* s);

/* Per-category device timing (CUDA events recorded on the session stream
 * around each kernel group while profiling is on).  Categories: */
#define TH_PROF_SETUP 0      /* seed rows, masks, hop bookkeeping          */
#define TH_PROF_EDGES 1      /* per-query edge counts |T_h|                */
#define TH_PROF_ACTIVATED 2  /* activated-triple materialisation           */
#define TH_PROF_PUSH 3       /* push hop kernels                           */
#define TH_PROF_PULL 4       /* pull hop kernels                           */
#define TH_PROF_FRONTIER 5   /* frontier materialisation (K4)              */
#define TH_PROF_CLEAR 6      /* state recycling                            */
#define TH_PROF_PATHS 7      /* path enumeration (K5)                      */
#define TH_PROF_CATEGORIES 8
int th_session_set_profiling(th_session* s, int on);
/* Accumulated milliseconds and launches per category since the last call
 * (arrays of n >= TH_PROF_CATEGORIES); resets the accumulators. Syncs. */
int th_session_profile(th_session* s, double* ms, int64_t* launches, int n);
/* Timeline of the last profiled run: n scopes of 4 doubles (category, stream
 * 0 = main / 1, 2 = the K4 side streams, start ms, end ms relative to the
 * run's first scope), copied when cap >= n; returns n (-1 on error). */
int64_t th_session_profile_trace(th_session* s, double* h_out4, int64_t cap);
/* Entity-list lengths of the last wave: [0] = distinct seed entities,
 * [h] = entities newly set at hop h (rows of the hop-h layer).  n >= k+1. */
int th_session_wave_lists(const th_session* s, int64_t* lens, int n);
/* Direction of each hop of the last wave: [h] = 1 pull, 0 push ([0] = 0). */
int th_session_wave_modes(const th_session* s, int32_t* modes, int n);

/* ---- partitioning (multi-GPU ownership) -------------------------------- */

/* Subject -> owner assignment, partition.py:49-98.  strategy 0 = hash
 * ((e * 0x9E3779B1) mod 2^32) mod m (partition.py:80-84), computed on the
 * device; entities with no out-edges get -1 (UNASSIGNED, partition.py:23).
 * d_owner: int32[E].  Asynchronous. */
int th_plan_owner_hash(const th_graph* g, int32_t m, int32_t* d_owner, void* stream);

/* Host-only planner (no GPU needed): the assignment and per-partition loads
 * of plan_partitions (partition.py:49-98) from subject out-degrees
 * (h_degrees[E], 0 = not a subject -> -1 UNASSIGNED).  TH_PLAN_HASH = the
 * multiplicative hash (partition.py:80-84); TH_PLAN_LPT = heaviest subject
 * first (ties by id) onto the lightest partition (ties by index)
 * (partition.py:85-94).  h_loads[m].  Range checks on m against the subject
 * count are the caller's (they raise UsageError in the reference). */
#define TH_PLAN_HASH 0
#define TH_PLAN_LPT 1
int th_plan_subjects(const int64_t* h_degrees, int64_t n_entities, int32_t m, int32_t strategy,
                     int32_t* h_assignment, int64_t* h_loads);

/* ---- partitioned graphs (multi-GPU; one shard per rank) ---------------- */

/* Ownership: own(v) = ((v * 0x9E3779B1) mod 2^32) mod world for every
 * entity (the reference hash plan, partition.py:80-84).  own(v) stores v's
 * out-row (subject-cohesive, partition.py:125-154) and v's per-query
 * visited/next bits.  Hub entities (d_hub_index[v] >= 0) are the exception:
 * their rows are edge-split, triple t of a hub living on rank own(t), and a
 * hub in the frontier is expanded by every rank.
 *   d_subj/d_rel/d_obj  the FULL graph's columns in tid order (device int32)
 *   d_lidx[E]           row of every entity at its owner (an owner's rows
 *                       number its entities in ascending id order)
 *   d_hub_index[E]      -1 or hub number < n_hubs; d_hub_ids[n_hubs] inverse
 *   d_l2g[n_local]      this rank's owned entities, ascending
 *   inbox_records       capacity of this rank's exchange inbox (records)
 * The shard copies what it keeps; inputs may be freed afterwards. */
typedef struct th_shard th_shard;
int th_shard_create(const int32_t* d_subj, const int32_t* d_rel, const int32_t* d_obj,
                    int64_t n_triples, int64_t n_entities, int64_t n_relations,
                    const int32_t* d_lidx, const int32_t* d_hub_index, const int32_t* d_hub_ids,
                    int64_t n_hubs, const int32_t* d_l2g, int64_t n_local, int32_t rank,
                    int32_t world, int64_t inbox_records, void* stream, th_shard** out);
int th_shard_destroy(th_shard* s);
int64_t th_shard_local_triples(const th_shard* s);
int64_t th_shard_launch_count(const th_shard* s);
int th_shard_can_pull(const th_shard* s);
/* Pull hops when the ranks' summed frontier out-edges exceed
 * n_triples / pull_divisor (default 8; <= 0 = push only). */
int th_shard_set_pull_divisor(th_shard* s, double pull_divisor);

/* Exchange.  Every shard owns an exchange region in its device memory --
 * control words (inbox cursor, overflow flag, every rank's published
 * frontier cost), an inbox of (int64 key, uint32 bits) records and a hub-row
 * board -- and its peers' KERNELS WRITE INTO IT DIRECTLY (remote atomics
 * reserve inbox space; stores deliver records, costs and hub rows).  Before
 * a wave every shard must be connected to every peer's region:
 *   same process (one device, or peer access enabled between devices):
 *       th_shard_region(peer, &base, ...); th_shard_connect(self, p, base)
 *   other processes: th_shard_ipc_handle(peer) -> 64 bytes, shipped to the
 *       others, th_shard_ipc_open(self, p, bytes) (CUDA IPC mapping)
 * Nothing is read back to the host during a wave. */
int th_shard_region(const th_shard* s, void** d_base, uint64_t* bytes, int64_t* inbox_records);
int th_shard_ipc_handle(const th_shard* s, void* h_handle64);
int th_shard_connect(th_shard* s, int32_t peer, void* d_peer_base);
int th_shard_ipc_open(th_shard* s, int32_t peer, const void* h_handle64);
/* After an inbox overflow (th_shard_finish -> TH_ERR_OVERFLOW with
 * th_shard_inbox_overflowed() == 1 on some rank): every rank grows its inbox
 * (the region is reallocated), all ranks reconnect, and the wave runs again. */
int th_shard_grow_inbox(th_shard* s, int64_t inbox_records);
int th_shard_inbox_overflowed(const th_shard* s);
/* Every hop and phase of a begun wave for n shards that share one stream
 * and one process (in-process worlds: stream order is the barrier), in the
 * order th_shard_hop would take them -- one call instead of 3 k n. */
int th_shards_run_hops(th_shard* const* shards, int32_t n, int32_t k);
/* A whole wave (th_shard_begin of every shard with queries[i], then every
 * hop and phase) for such a world, replayed as one CUDA graph once a shape
 * repeats (inputs staged into session buffers; h_n_seeds[i] = length of
 * queries[i].d_seeds).  Eager for shards with a hub cache or profiling. */
int th_shards_run_wave(th_shard* const* shards, int32_t n, const th_query* queries,
                       const int64_t* h_n_seeds);
/* Per-phase kernel-group timing of the shard's waves (as th_session_*). */
int th_shard_set_profiling(th_shard* s, int on);
int64_t th_shard_profile_trace(th_shard* s, double* h_out4, int64_t cap);

/* K7 on-demand hub-adjacency cache (the reference's LRU,
 * cache.py:38-89, reached per partition from engine.py:80-81).  The shard's
 * hub-slice rows leave HBM for a pinned host store; their CSR range is
 * re-mapped page by page (CUDA virtual memory) onto `capacity_pages`
 * physical HBM pages.  Before each hop the pages of the frontier's hubs are
 * made resident, the least recently used page evicted first; a hop whose
 * hubs span more pages than the capacity fails with TH_ERR_INVALID.
 * Counters keep the reference's algebra: hits + misses = accesses, loads =
 * misses, one eviction per load at capacity.  Enable between waves, once. */
int th_shard_hub_cache(th_shard* s, int64_t capacity_pages);
/* h_out8: hits, misses, loads, evictions, resident pages, capacity, pages of
 * the hub region, edges per page. */
int th_shard_hub_cache_stats(th_shard* s, int64_t* h_out8);
/* Access log (page numbers, oldest first): returns its length n and, when
 * cap >= n, copies it to h_out and clears it; -1 without a cache. */
int64_t th_shard_hub_cache_trace(th_shard* s, int64_t* h_out, int64_t cap);
/* Resident pages, least recently used first (copied when cap >= n). */
int64_t th_shard_hub_cache_resident(th_shard* s, int64_t* h_out, int64_t cap);
/* Records this rank wrote into OTHER ranks' inboxes at hops 1..n of the
 * last wave (12 bytes each over the interconnect).  Synchronises. */
int th_shard_sent(th_shard* s, int64_t* h_per_hop, int n);

/* One wave of <= 1024 queries; every rank makes the same calls with the
 * same query arrays, and all ranks pass a barrier between consecutive calls
 * (the peers' writes of the previous step are then complete):
 *   th_shard_begin(q)          seeds (hub seeds on every rank); publishes
 *                              hop 1's frontier cost to every rank
 *   for h = 1..k, phase 0..2:  th_shard_hop(h, phase)
 *     phase 0 (send)    direction from the published costs, edge counts;
 *                       push: local test-and-set + records for remote
 *                       targets into their owners' inboxes; pull: the owned
 *                       frontier rows into every rank's inbox
 *     phase 1 (receive) apply the inbox (push) or stage the frontier and
 *                       pull over the owned in-edges (pull); owners write
 *                       their hubs' next-layer rows onto every hub board
 *     phase 2 (end)     hub frontier rows from the board, K4 over the owned
 *                       rows, publish the new layer's frontier cost
 *   th_shard_finish(&result)   like th_finish, with frontier ids = owned
 *       entities (global ids, sorted), activated = local triples (global
 *       tids, sorted), edges = this rank's share (sum over ranks = |T_h|).
 *       TH_ERR_OVERFLOW: result capacities or the inbox grew/must grow;
 *       every rank runs the wave again.  Paths are not available here. */
/* The shard's own triples (device arrays, local tid order = ascending
 * global tid): subject as a LOCAL row (rows < n_local map through l2g,
 * hub slice rows n_local + h through hub_ids), relation, object (global),
 * and the global tid of each local triple. */
typedef struct {
  int64_t n_triples, n_local, n_hubs;
  const int32_t* subj_row;
  const uint16_t* rel;
  const int32_t* obj;
  const int32_t* tid_l2g;
  const int32_t* l2g;
  const int32_t* hub_ids;
} th_shard_cols;
int th_shard_columns(const th_shard* s, th_shard_cols* out);

int th_shard_begin(th_shard* s, const th_query* q);
int th_shard_hop(th_shard* s, int32_t hop, int32_t phase);
int th_shard_finish(th_shard* s, th_result* out);

/* ---- id sets: store-backed partitioned retrieval ------------------------
 * The per-hop glue of the reference's out-of-core Algorithm 1
 * (engine.py:94-135: route the frontier, map to a partition's local ids,
 * expand, map back, union sorted) on device bitmaps of nbits bits
 * ((nbits + 31) / 32 uint32 words, caller-owned, zeroed by the caller).
 * Calls that report a count or an error synchronise `stream`. */
/* counts[p] = |{i : assign[ids[i]] == p}| (UNASSIGNED = -1 skipped);
 * replaces route's bucketing (partition.py:170-181); TH_ERR_INVALID for ids
 * outside [0, n_entities). */
int th_ids_route_count(const int32_t* d_assign, int64_t n_entities, const int32_t* d_ids, int64_t n,
                       int32_t m, int64_t* d_counts, void* stream);
/* bits[map[ids[i]]] = 1, or bits[ids[i]] = 1 with d_map NULL (local -> global
 * maps, ent_to_global / tid_to_global, partition.py:113-114). */
int th_ids_map_scatter(const int32_t* d_map, int64_t map_len, const int32_t* d_ids, int64_t n,
                       uint32_t* d_bits, int64_t nbits, void* stream);
/* bits[j] = 1 for every ids[i] == sorted_map[j] (Subgraph.entities_to_local,
 * partition.py:115-122: absent ids dropped). */
int th_ids_to_local_bits(const int32_t* d_sorted_map, int64_t map_len, const int32_t* d_ids,
                         int64_t n, uint32_t* d_bits, void* stream);
/* fresh &= ~visited; visited |= fresh (run_hops, incidence.py:301-315). */
int th_bits_andnot_update(uint32_t* d_fresh, uint32_t* d_visited, int64_t nbits, void* stream);
/* dst |= src (CUMULATIVE union of layers, incidence.py:309-312). */
int th_bits_or(uint32_t* d_dst, const uint32_t* d_src, int64_t nbits, void* stream);
/* The set bits as an ascending int32 list; *n_out = their number.
 * TH_ERR_OVERFLOW (nothing written) when it exceeds cap. */
int th_bits_compact(const uint32_t* d_bits, int64_t nbits, int32_t* d_out, int64_t cap,
                    int64_t* n_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TH_B200_H */
