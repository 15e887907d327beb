// K5: capped lexicographic walk enumeration (reconstruct_paths).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace th {

struct PathArgs {
  const int32_t* indptr;
  const int32_t* csr_tid;
  const int32_t* csr_obj;
  const uint16_t* csr_rel;
  const int32_t* t_obj;
  const uint16_t* t_rel;
  const int32_t* qoff;
  const int32_t* seeds;
  const uint32_t* masks;
  int mask_words;
  // hop-1 activated triple lists (used for multi-seed queries)
  const int64_t* l0_off;
  const int64_t* l0_len;
  const int32_t* l0_ids;
  bool singleton;
  int32_t B, k;
  int64_t E;
  int64_t max_paths;  // -1 = uncapped
  int64_t* p_off;     // [B+1]
  int64_t* p_cnt;     // [B]
  uint8_t* p_trunc;   // [B]
  int32_t* p_tids;    // [cap][k]
  int64_t* scratch;
  int64_t cap;        // capacity in paths
  int64_t* used;      // device: total paths
  // capped queries: one DFS writes each query's paths into its own
  // max_paths-sized slot of tmp ([B][max_paths][k]), a compaction packs
  // them (instead of a counting DFS + a writing DFS); null = two passes
  int32_t* tmp = nullptr;
  bool k2_parallel = true;  // k = 2 singleton capped queries: a CTA per query
};

int64_t scan_scratch_elems_i64(int64_t n);
// returns the number of kernels launched
int launch_paths(const PathArgs& a, cudaStream_t st);

}  // namespace th
