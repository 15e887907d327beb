// Device loading of LKG1 graph archives.
//
// Reference format (archive.py:1-24, graph_to_bytes :66-81): a header, then
// the payload indptr (u64 x E+1) and the row-ordered triple ids, followed
// by obj and rel in triple-id order, each u32 or u64 ("id width").  The
// host checks the header and the CRC32 (archive.py:84-105) and copies the
// raw payload to the device; here the payload is narrowed to int32 with
// range checks, validated like _validate_structure (archive.py:121-133:
// monotone offsets, triple ids a permutation, strictly ascending within a
// row, object/relation ids in range), the subject column is recovered from
// the row structure, and the usual device graph (K1) is built from it.
#include <algorithm>
#include <cstdint>
#include <string>

#include "../../include/th_b200.h"
#include "common.cuh"
#include "graph.cuh"

namespace th {
namespace {

enum : int32_t {
  kBadOffsets = 1,   // corrupt sub row offsets
  kBadRange = 2,     // object or relation id out of range
  kNotPerm = 4,      // sub columns are not a permutation of the triple ids
  kUnsorted = 8,     // sub row columns not strictly sorted
};

unsigned lkg_grid(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, kNumSMs * 16));
}

__global__ void lkg_offsets_kernel(const uint64_t* __restrict__ ip, int64_t E, int64_t T,
                                   int32_t* out, int32_t* err) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u <= E;
       u += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t v = ip[u];
    bool bad = v > (uint64_t)T;
    if (u == 0) bad |= v != 0;
    if (u == E) bad |= v != (uint64_t)T;
    if (u > 0) bad |= ip[u - 1] > v;
    if (bad) atomicOr(err, kBadOffsets);
    out[u] = (int32_t)(v > (uint64_t)T ? 0 : v);
  }
}

template <typename I>
__global__ void lkg_ids_kernel(const I* __restrict__ src, int64_t n, uint64_t bound, int32_t* dst,
                               int32_t code, int32_t* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t v = (uint64_t)src[i];
    if (v >= bound) {
      atomicOr(err, code);
      dst[i] = 0;
    } else {
      dst[i] = (int32_t)v;
    }
  }
}

// per CSR slot: its row (binary search over the offsets), the permutation
// test (bitmap test-and-set), row-local ascent, and subj[tid] = row
__global__ void lkg_rows_kernel(const int32_t* __restrict__ ip, int64_t E,
                                const int32_t* __restrict__ tids, int64_t T, int32_t* subj,
                                uint32_t* seen, int32_t* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = E;  // row = last u with ip[u] <= i
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (ip[mid] <= i) lo = mid;
      else hi = mid - 1;
    }
    const int32_t t = tids[i];
    const uint32_t b = 1u << (t & 31);
    if (atomicOr(&seen[t >> 5], b) & b) atomicOr(err, kNotPerm);
    subj[t] = (int32_t)lo;
    if (i > ip[lo] && tids[i - 1] >= t) atomicOr(err, kUnsorted);
  }
}

}  // namespace

int graph_build_lkg(Graph* g, const void* d_indptr, const void* d_tids, const void* d_obj,
                    const void* d_rel, int width, int64_t T, int64_t E, int64_t R, bool reverse,
                    cudaStream_t st) {
  int32_t *ip = nullptr, *tids = nullptr, *obj = nullptr, *rel = nullptr, *subj = nullptr,
          *err = nullptr;
  uint32_t* seen = nullptr;
  const int64_t tn = std::max<int64_t>(T, 1);
  TH_CUDA(cudaMalloc(&ip, sizeof(int32_t) * (E + 1)));
  TH_CUDA(cudaMalloc(&tids, sizeof(int32_t) * tn));
  TH_CUDA(cudaMalloc(&obj, sizeof(int32_t) * tn));
  TH_CUDA(cudaMalloc(&rel, sizeof(int32_t) * tn));
  TH_CUDA(cudaMalloc(&subj, sizeof(int32_t) * tn));
  TH_CUDA(cudaMalloc(&seen, sizeof(uint32_t) * ((tn + 31) / 32)));
  TH_CUDA(cudaMalloc(&err, sizeof(int32_t)));
  TH_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
  TH_CUDA(cudaMemsetAsync(seen, 0, sizeof(uint32_t) * ((tn + 31) / 32), st));
  lkg_offsets_kernel<<<lkg_grid(E + 1), 256, 0, st>>>(static_cast<const uint64_t*>(d_indptr), E, T,
                                                        ip, err);
  TH_LAUNCHED();
  if (T > 0) {
    if (width == 4) {
      lkg_ids_kernel<<<lkg_grid(T), 256, 0, st>>>(static_cast<const uint32_t*>(d_tids), T, T, tids,
                                                   kNotPerm, err);
      lkg_ids_kernel<<<lkg_grid(T), 256, 0, st>>>(static_cast<const uint32_t*>(d_obj), T, E, obj,
                                                   kBadRange, err);
      lkg_ids_kernel<<<lkg_grid(T), 256, 0, st>>>(static_cast<const uint32_t*>(d_rel), T, R, rel,
                                                   kBadRange, err);
    } else {
      lkg_ids_kernel<<<lkg_grid(T), 256, 0, st>>>(static_cast<const uint64_t*>(d_tids), T, T, tids,
                                                   kNotPerm, err);
      lkg_ids_kernel<<<lkg_grid(T), 256, 0, st>>>(static_cast<const uint64_t*>(d_obj), T, E, obj,
                                                   kBadRange, err);
      lkg_ids_kernel<<<lkg_grid(T), 256, 0, st>>>(static_cast<const uint64_t*>(d_rel), T, R, rel,
                                                   kBadRange, err);
    }
    TH_LAUNCHED();
  }
  int32_t h_err = 0;
  TH_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  TH_CUDA(cudaStreamSynchronize(st));
  if (!(h_err & kBadOffsets) && T > 0) {
    lkg_rows_kernel<<<lkg_grid(T), 256, 0, st>>>(ip, E, tids, T, subj, seen, err);
    TH_LAUNCHED();
    TH_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    TH_CUDA(cudaStreamSynchronize(st));
  }
  int rc = TH_OK;
  if (h_err) {
    // same precedence and wording as archive.py:121-133
    if (h_err & kBadOffsets) set_error("corrupt sub row offsets");
    else if (h_err & kNotPerm) set_error("sub columns are not a permutation of the triple ids");
    else if (h_err & kBadRange) set_error("object or relation id out of range");
    else set_error("sub row columns not strictly sorted");
    rc = TH_ERR_DATA;
  } else {
    rc = graph_build(g, subj, rel, obj, T, E, R, reverse, st);
  }
  TH_CUDA(cudaStreamSynchronize(st));
  for (void* p : {(void*)ip, (void*)tids, (void*)obj, (void*)rel, (void*)subj, (void*)seen,
                  (void*)err})
    cudaFree(p);
  return rc;
}

}  // namespace th
