// Device-wide primitives: exclusive scans and a stable LSD radix sort.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace th {

// Exclusive prefix sum of n elements (in may alias out).  `scratch` must
// hold scan_scratch_elems(n) elements of T.  Returns the number of kernels
// launched (for the session launch counter).
template <typename T>
int64_t scan_scratch_elems(int64_t n);
template <typename T>
int scan_exclusive(const T* in, T* out, int64_t n, T* scratch, cudaStream_t st);

// Stable LSD radix sort of (key, value) int32 pairs by the low `key_bits`
// bits of key.  Buffers ping-pong between (k0,v0) and (k1,v1); returns 0 if
// the sorted data ended in (k0,v0), 1 if in (k1,v1).  `hist` must hold
// radix_hist_elems(n) int32.
int64_t radix_hist_elems(int64_t n);
int radix_sort_pairs(int32_t* k0, int32_t* v0, int32_t* k1, int32_t* v1, int64_t n,
                     int key_bits, int32_t* hist, int32_t* scan_scratch, cudaStream_t st,
                     int64_t* launches);

}  // namespace th
