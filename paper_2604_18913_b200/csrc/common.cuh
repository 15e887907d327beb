// Shared device helpers for the k-hop engine (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#define TH_FULL 0xffffffffu

namespace th {

// thread-local error string behind th_last_error()
void set_error(const std::string& msg);

struct CudaError {
  cudaError_t code;
  const char* where;
};

#define TH_CUDA(expr)                                                  \
  do {                                                                 \
    cudaError_t _e = (expr);                                           \
    if (_e != cudaSuccess) throw ::th::CudaError{_e, #expr};           \
  } while (0)

#define TH_LAUNCHED() TH_CUDA(cudaPeekAtLastError())

constexpr int kNumSMs = 148;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// 32x32 bit-matrix transpose across a warp: on entry lane i holds row i
// (bit j = column j); on exit lane j holds column j (bit i = row i).
__device__ __forceinline__ uint32_t transpose32(uint32_t x) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int s = 16, k = 0; s >= 1; s >>= 1, ++k) {
    const uint32_t m = s == 16 ? 0x0000ffffu : s == 8 ? 0x00ff00ffu : s == 4 ? 0x0f0f0f0fu
                     : s == 2 ? 0x33333333u : 0x55555555u;
    const uint32_t o = __shfl_xor_sync(TH_FULL, x, s);
    x = (lane & s) ? (((o >> s) & m) | (x & ~m)) : ((x & m) | ((o & m) << s));
  }
  return x;
}

// position of the r-th (0-based) set bit of x (r < popc(x)): a five-step
// popcount search, a fixed dozen instructions (__fns is a software loop)
__device__ __forceinline__ int select_bit(uint32_t x, int r) {
  int pos = 0;
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const int c = __popc(x & ((1u << w) - 1u));
    if (r >= c) {
      r -= c;
      x >>= w;
      pos += w;
    }
  }
  return pos;
}

// Warp-aggregated append of `item` from the lanes with `take` set.  Must be
// called by all 32 lanes in converged code (full-mask collectives only; no
// __activemask-based aggregation, which can deadlock under independent
// thread scheduling when lanes diverge inside the aggregated region).
// Also adds `cost` of the appending lanes (clamped to 2^26 each) to *sum.
template <typename T>
__device__ __forceinline__ void warp_append_all(bool take, T item, uint32_t cost, T* list,
                                                int32_t* counter, int64_t cap,
                                                unsigned long long* sum) {
  const unsigned m = __ballot_sync(TH_FULL, take);
  if (!m) return;
  const int leader = __ffs(m) - 1;
  int32_t base = 0;
  if ((int)lane_id() == leader) base = atomicAdd(counter, __popc(m));
  base = __shfl_sync(TH_FULL, base, leader);
  const unsigned rank = __popc(m & lanemask_lt());
  if (take && base + (int64_t)rank < cap) list[base + rank] = item;
  if (sum) {
    const unsigned c = __reduce_add_sync(TH_FULL, take ? (cost > (1u << 26) ? (1u << 26) : cost) : 0u);
    if ((int)lane_id() == leader) atomicAdd(sum, (unsigned long long)c);
  }
}

}  // namespace th
