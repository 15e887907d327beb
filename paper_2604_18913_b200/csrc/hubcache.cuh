// K7: on-demand hub-adjacency cache of a shard.
//
// The forward CSR rows of the hub slices -- the tail rows [row0, row0 + n)
// of a shard's graph -- move out of HBM into a pinned host store; the CSR
// arrays become a virtual address range whose hub part is backed page by
// page by a fixed pool of `capacity` physical HBM slots (CUDA virtual
// memory management).  Before each hop the pages of the frontier's hub rows
// are made resident, least recently used page out first, so the hop kernels
// read the same CSR addresses as without the cache and need no change.
//
// Counters follow the reference's LRU algebra (cache.py:38-89): an access
// hits or misses, every miss loads once, a load at capacity evicts one.  A
// hop's accesses run resident pages first (in their recency order), then
// the missing pages in ascending order, so the pages a hop needs are all
// resident together; the access trace is kept for checking against the
// independent model (tests/lru_model.py).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "graph.cuh"

namespace th {

struct HubCache;

// Takes over g's forward CSR arrays (csr_obj / csr_rel / csr_tid) with the
// rows [row0, g->E) as the cached hub region.  Shifts g->indptr so the hub
// region starts on a page boundary.  Synchronises `st`.
int hubcache_create(HubCache** out, Graph* g, int64_t row0, int64_t capacity, cudaStream_t st);
// Makes the pages of every hub row whose bit is set in the row flag words
// `d_flags` resident (the caller has synchronised `st`); H2D loads are
// queued on `st`.  TH_ERR_INVALID when the hop needs more pages than fit.
int hubcache_step(HubCache* hc, const uint32_t* d_flags, cudaStream_t st);
// hits, misses, loads, evictions, resident pages, capacity, pages, edges per page
void hubcache_stats(const HubCache* hc, int64_t out[8]);
// access log (page numbers, oldest first): copies up to cap entries and
// clears the log; returns the number of entries it held
int64_t hubcache_trace(HubCache* hc, int64_t* out, int64_t cap);
// resident pages, least recently used first; returns their number
int64_t hubcache_resident(const HubCache* hc, int64_t* out, int64_t cap);
// unmaps and releases everything; g's CSR arrays are gone afterwards
void hubcache_free(HubCache* hc, Graph* g);

}  // namespace th
