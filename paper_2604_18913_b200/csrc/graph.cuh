// Device incidence graph (K1): subject CSR + tid-ordered columns + reverse CSR.
#pragma once
#include <stdint.h>

#include "common.cuh"

namespace th {

// pull hops walk in-rows in items of at most kPullChunk in-edges; a lane
// group owns one item (see engine.cu pull_kernel)
constexpr int32_t kPullChunk = 32;

struct Graph {
  int64_t E = 0, T = 0, R = 0;
  // subject CSR (replaces IncidenceGraph.indptr/tids, incidence.py:125-126)
  int32_t* indptr = nullptr;   // [E+1]
  int32_t* csr_tid = nullptr;  // [T]
  int32_t* csr_obj = nullptr;  // [T]
  uint16_t* csr_rel = nullptr; // [T]
  // triple-id order columns (IncidenceGraph.obj/rel + the lazy subj inverse)
  int32_t* subj = nullptr;
  int32_t* obj = nullptr;
  uint16_t* rel = nullptr;
  // reverse CSR by object, for pull hops
  int32_t* rindptr = nullptr;  // [E+1]
  int32_t* rsrc = nullptr;     // [T]
  uint16_t* rrel = nullptr;    // [T]
  // target row of each in-edge (~v when the row is split over several
  // items): lets the two-phase pull's screen stream the in-edges
  int32_t* rdst = nullptr;     // [T]
  // static pull schedule: item i covers in-edges [item_lo[i], item_hi[i]) of
  // entity item_v[i] (stored as ~v when the in-row is split over several
  // items, which then merge with atomics); items ascend by entity
  int32_t* item_v = nullptr;
  int32_t* item_lo = nullptr;
  int32_t* item_hi = nullptr;
  int64_t n_items = 0;
  int64_t n_split = 0;  // entities whose in-row spans several items
  int64_t max_out = 0, max_in = 0;
  uint64_t bytes = 0;
  int64_t launches = 0;
};

// Builds everything; throws CudaError / std::invalid_argument-like status via
// the return code (TH_ERR_RANGE for out-of-range ids).
// obj_bound: object ids must be < obj_bound (default E; a shard's rows are
// local while its objects keep global ids)
int graph_build(Graph* g, const int32_t* d_subj, const int32_t* d_rel, const int32_t* d_obj,
                int64_t T, int64_t E, int64_t R, bool reverse, cudaStream_t st,
                int64_t obj_bound = -1);
void graph_free(Graph* g);

// LKG1 archive payload already on the device (archive.cu): narrow, validate
// (TH_ERR_DATA + message on a structural error), recover subjects, build.
int graph_build_lkg(Graph* g, const void* d_indptr, const void* d_tids, const void* d_obj,
                    const void* d_rel, int width, int64_t T, int64_t E, int64_t R, bool reverse,
                    cudaStream_t st);

}  // namespace th
