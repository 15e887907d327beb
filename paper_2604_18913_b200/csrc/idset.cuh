// Id-set kernels (idset.cu): bitmap unions/differences and ordered
// compaction for the store-backed partitioned path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace th {

int ids_route_count(const int32_t* assign, int64_t E, const int32_t* ids, int64_t n, int32_t m,
                    int64_t* d_counts, cudaStream_t st);
int ids_map_scatter(const int32_t* map, int64_t map_n, const int32_t* ids, int64_t n,
                    uint32_t* bits, int64_t nbits, cudaStream_t st);
int ids_to_local_bits(const int32_t* sorted, int64_t m, const int32_t* ids, int64_t n,
                      uint32_t* bits, cudaStream_t st);
int bits_andnot_update(uint32_t* fresh, uint32_t* visited, int64_t nbits, cudaStream_t st);
int bits_or(uint32_t* dst, const uint32_t* src, int64_t nbits, cudaStream_t st);
int bits_compact(const uint32_t* bits, int64_t nbits, int32_t* out, int64_t cap, int64_t* n_out,
                 cudaStream_t st);

}  // namespace th
