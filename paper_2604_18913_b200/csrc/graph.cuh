// Device incidence graph (K1): subject CSR + tid-ordered columns + reverse CSR.
#pragma once
#include <stdint.h>

#include "common.cuh"

namespace th {

// in-rows longer than this are split into chunks of kPullChunk edges and
// processed by many warps (pull hops); see engine.cu
constexpr int32_t kHeavyPull = 4096;
constexpr int32_t kPullChunk = 2048;

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
  // pull schedule for heavy in-rows: chunk c covers in-edges
  // [chunk_lo[c], chunk_hi[c]) of entity heavy_ids[chunk_hv[c]]
  int32_t* heavy_ids = nullptr;
  int64_t n_heavy = 0;
  int32_t* chunk_hv = nullptr;
  int32_t* chunk_lo = nullptr;
  int32_t* chunk_hi = nullptr;
  int64_t n_chunks = 0;
  int64_t max_out = 0, max_in = 0;
  uint64_t bytes = 0;
  int64_t launches = 0;
};

// Builds everything; throws CudaError / std::invalid_argument-like status via
// the return code (TH_ERR_RANGE for out-of-range ids).
int graph_build(Graph* g, const int32_t* d_subj, const int32_t* d_rel, const int32_t* d_obj,
                int64_t T, int64_t E, int64_t R, bool reverse, cudaStream_t st);
void graph_free(Graph* g);

}  // namespace th
