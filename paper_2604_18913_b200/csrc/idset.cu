// Id-set kernels for store-backed partitioned retrieval: the per-hop glue
// of the reference's Algorithm 1 (engine.py:94-135 -- route the frontier to
// its partitions, map global ids to a partition's local ids, map results
// back, union them sorted) kept on the device as bitmaps over the id space.
//
// A sorted duplicate-free id list is the canonical EntityVector/TripleVector
// form (incidence.py:78-118); here every union/difference is a word-wise
// bitmap operation and the list is recovered by an ordered compaction
// (popcount per word -> exclusive scan of block counts -> ascending write).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/th_b200.h"
#include "common.cuh"
#include "idset.cuh"
#include "prims.cuh"

namespace th {
namespace {

constexpr int kIdThreads = 256;
constexpr int kIdWordsPerThread = 8;
constexpr int kIdWordsPerBlock = kIdThreads * kIdWordsPerThread;

unsigned id_grid(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kIdThreads - 1) / kIdThreads,
                                                           (int64_t)kNumSMs * 16));
}

__device__ __forceinline__ uint32_t word_below(const uint32_t* bits, int64_t w, int64_t nbits) {
  if (w * 32 >= nbits) return 0u;
  const uint32_t f = bits[w];
  const int64_t left = nbits - w * 32;
  return left >= 32 ? f : f & ((1u << left) - 1u);
}

__device__ __forceinline__ int block_scan_excl(int v, int* total) {
  __shared__ int ws[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(TH_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    int s = lane < nw ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(TH_FULL, s, o);
      if (lane >= o) s += y;
    }
    ws[lane] = s;
  }
  __syncthreads();
  const int before = warp ? ws[warp - 1] : 0;
  *total = ws[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before + x - v;
}

__global__ void route_count_kernel(const int32_t* __restrict__ assign, int64_t E,
                                   const int32_t* __restrict__ ids, int64_t n, int32_t m,
                                   int64_t* counts, int32_t* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = ids[i];
    if (v < 0 || v >= E) {
      atomicExch(err, 1);
      continue;
    }
    const int32_t p = assign[v];
    if (p >= 0 && p < m) atomicAdd(reinterpret_cast<unsigned long long*>(counts + p), 1ull);
  }
}

// bits[map[ids[i]]] = 1 (map == nullptr: identity); out-of-range ids flag err
__global__ void map_scatter_kernel(const int32_t* __restrict__ map, int64_t map_n,
                                   const int32_t* __restrict__ ids, int64_t n, uint32_t* bits,
                                   int64_t nbits, int32_t* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = ids[i];
    if (map) {
      if (v < 0 || v >= map_n) {
        atomicExch(err, 1);
        continue;
      }
      v = map[v];
    }
    if (v < 0 || v >= nbits) {
      atomicExch(err, 1);
      continue;
    }
    atomicOr(bits + (v >> 5), 1u << (v & 31));
  }
}

// local bitmap of the positions of ids present in the ascending map
// (Subgraph.entities_to_local, partition.py:115-122: absent ids dropped)
__global__ void to_local_kernel(const int32_t* __restrict__ sorted, int64_t m,
                                const int32_t* __restrict__ ids, int64_t n, uint32_t* bits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = ids[i];
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (sorted[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    if (lo < m && sorted[lo] == v) atomicOr(bits + (lo >> 5), 1u << (lo & 31));
  }
}

// fresh = reached & ~visited; visited |= fresh (run_hops, incidence.py:301-315)
__global__ void andnot_update_kernel(uint32_t* fresh, uint32_t* visited, int64_t nwords) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t f = fresh[w] & ~visited[w];
    fresh[w] = f;
    visited[w] |= f;
  }
}

__global__ void or_kernel(uint32_t* dst, const uint32_t* src, int64_t nwords) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x)
    dst[w] |= src[w];
}

__global__ void __launch_bounds__(kIdThreads) bits_count_kernel(const uint32_t* __restrict__ bits,
                                                                int64_t nbits, int32_t* bcount) {
  const int64_t w0 = (int64_t)blockIdx.x * kIdWordsPerBlock + threadIdx.x * kIdWordsPerThread;
  int c = 0;
#pragma unroll
  for (int i = 0; i < kIdWordsPerThread; ++i) c += __popc(word_below(bits, w0 + i, nbits));
  int total;
  block_scan_excl(c, &total);
  if (threadIdx.x == 0) bcount[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kIdThreads) bits_write_kernel(const uint32_t* __restrict__ bits,
                                                                int64_t nbits,
                                                                const int32_t* __restrict__ boff,
                                                                int32_t* out) {
  const int64_t w0 = (int64_t)blockIdx.x * kIdWordsPerBlock + threadIdx.x * kIdWordsPerThread;
  uint32_t f[kIdWordsPerThread];
  int c = 0;
#pragma unroll
  for (int i = 0; i < kIdWordsPerThread; ++i) {
    f[i] = word_below(bits, w0 + i, nbits);
    c += __popc(f[i]);
  }
  int total;
  int o = boff[blockIdx.x] + block_scan_excl(c, &total);
#pragma unroll
  for (int i = 0; i < kIdWordsPerThread; ++i) {
    uint32_t x = f[i];
    const int32_t base = (int32_t)((w0 + i) * 32);
    while (x) {
      out[o++] = base + __ffs(x) - 1;
      x &= x - 1u;
    }
  }
}

__global__ void total_kernel(const int32_t* bcount_excl, const int32_t* bcount_last, int nb,
                             int64_t* n_out) {
  *n_out = (int64_t)bcount_excl[nb - 1] + *bcount_last;
}

}  // namespace

int ids_route_count(const int32_t* assign, int64_t E, const int32_t* ids, int64_t n, int32_t m,
                    int64_t* d_counts, cudaStream_t st) {
  int32_t* err = nullptr;
  TH_CUDA(cudaMallocAsync(&err, sizeof(int32_t), st));
  TH_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
  TH_CUDA(cudaMemsetAsync(d_counts, 0, sizeof(int64_t) * std::max<int32_t>(m, 1), st));
  if (n > 0) {
    route_count_kernel<<<id_grid(n), kIdThreads, 0, st>>>(assign, E, ids, n, m, d_counts, err);
    TH_LAUNCHED();
  }
  int32_t h = 0;
  TH_CUDA(cudaMemcpyAsync(&h, err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  TH_CUDA(cudaFreeAsync(err, st));
  TH_CUDA(cudaStreamSynchronize(st));
  return h ? TH_ERR_INVALID : TH_OK;
}

int ids_map_scatter(const int32_t* map, int64_t map_n, const int32_t* ids, int64_t n,
                    uint32_t* bits, int64_t nbits, cudaStream_t st) {
  if (n <= 0) return TH_OK;
  int32_t* err = nullptr;
  TH_CUDA(cudaMallocAsync(&err, sizeof(int32_t), st));
  TH_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
  map_scatter_kernel<<<id_grid(n), kIdThreads, 0, st>>>(map, map_n, ids, n, bits, nbits, err);
  TH_LAUNCHED();
  int32_t h = 0;
  TH_CUDA(cudaMemcpyAsync(&h, err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  TH_CUDA(cudaFreeAsync(err, st));
  TH_CUDA(cudaStreamSynchronize(st));
  return h ? TH_ERR_INVALID : TH_OK;
}

int ids_to_local_bits(const int32_t* sorted, int64_t m, const int32_t* ids, int64_t n,
                      uint32_t* bits, cudaStream_t st) {
  if (n <= 0 || m <= 0) return TH_OK;
  to_local_kernel<<<id_grid(n), kIdThreads, 0, st>>>(sorted, m, ids, n, bits);
  TH_LAUNCHED();
  return TH_OK;
}

int bits_andnot_update(uint32_t* fresh, uint32_t* visited, int64_t nbits, cudaStream_t st) {
  const int64_t nw = (nbits + 31) / 32;
  if (nw <= 0) return TH_OK;
  andnot_update_kernel<<<id_grid(nw), kIdThreads, 0, st>>>(fresh, visited, nw);
  TH_LAUNCHED();
  return TH_OK;
}

int bits_or(uint32_t* dst, const uint32_t* src, int64_t nbits, cudaStream_t st) {
  const int64_t nw = (nbits + 31) / 32;
  if (nw <= 0) return TH_OK;
  or_kernel<<<id_grid(nw), kIdThreads, 0, st>>>(dst, src, nw);
  TH_LAUNCHED();
  return TH_OK;
}

int bits_compact(const uint32_t* bits, int64_t nbits, int32_t* out, int64_t cap, int64_t* n_out,
                 cudaStream_t st) {
  *n_out = 0;
  const int64_t nw = (nbits + 31) / 32;
  if (nw <= 0) return TH_OK;
  const int nb = (int)((nw + kIdWordsPerBlock - 1) / kIdWordsPerBlock);
  const int64_t scratch = scan_scratch_elems<int32_t>(nb);
  int32_t* buf = nullptr;  // [nb] counts, [1] last count, [nb] scan, scratch
  int64_t* d_n = nullptr;
  TH_CUDA(cudaMallocAsync(&buf, sizeof(int32_t) * (2 * (size_t)nb + 1 + scratch), st));
  TH_CUDA(cudaMallocAsync(&d_n, sizeof(int64_t), st));
  int32_t* cnt = buf;
  int32_t* last = buf + nb;
  int32_t* off = buf + nb + 1;
  bits_count_kernel<<<nb, kIdThreads, 0, st>>>(bits, nbits, cnt);
  TH_LAUNCHED();
  TH_CUDA(cudaMemcpyAsync(last, cnt + nb - 1, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  scan_exclusive<int32_t>(cnt, off, nb, off + nb, st);
  total_kernel<<<1, 1, 0, st>>>(off, last, nb, d_n);
  TH_LAUNCHED();
  int64_t total = 0;
  TH_CUDA(cudaMemcpyAsync(&total, d_n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TH_CUDA(cudaStreamSynchronize(st));
  if (total <= cap) {
    bits_write_kernel<<<nb, kIdThreads, 0, st>>>(bits, nbits, off, out);
    TH_LAUNCHED();
  }
  TH_CUDA(cudaFreeAsync(buf, st));
  TH_CUDA(cudaFreeAsync(d_n, st));
  *n_out = total;
  return total <= cap ? TH_OK : TH_ERR_OVERFLOW;
}

}  // namespace th
