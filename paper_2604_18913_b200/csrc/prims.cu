// Exclusive scan (3-phase) and stable LSD radix sort (8-bit digits) used by
// the device CSR build (K1, replaces the bincount/cumsum/stable-argsort of
// build_incidence, incidence.py:181-188).
#include "common.cuh"
#include "prims.cuh"

namespace th {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ T block_exclusive_scan(T v, T* warp_sums, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(TH_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    T w = lane < nw ? warp_sums[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(TH_FULL, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) warp_sums[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const T warp_off = warp ? warp_sums[warp - 1] : T(0);
  *total = warp_sums[(blockDim.x >> 5) - 1];
  return warp_off + x - v;
}

template <typename T>
__global__ void scan_reduce_kernel(const T* __restrict__ in, T* __restrict__ partial, int64_t n) {
  __shared__ T ws[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) s += in[base + i];
  T total;
  block_exclusive_scan(s, ws, &total);
  if (threadIdx.x == 0) partial[blockIdx.x] = total;
}

// single block: exclusive scan of the per-tile partials, in place
template <typename T>
__global__ void scan_partials_kernel(T* partial, int64_t nb) {
  __shared__ T ws[32];
  T carry = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += kScanThreads) {
    const int64_t i = b0 + threadIdx.x;
    const T v = i < nb ? partial[i] : T(0);
    T total;
    const T ex = block_exclusive_scan(v, ws, &total);
    if (i < nb) partial[i] = carry + ex;
    carry += total;
    __syncthreads();
  }
}

template <typename T>
__global__ void scan_apply_kernel(const T* in, T* out, const T* __restrict__ partial, int64_t n) {
  __shared__ T ws[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? in[base + i] : T(0);
    s += v[i];
  }
  T total;
  T run = block_exclusive_scan(s, ws, &total) + partial[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
}

// ---- radix sort -----------------------------------------------------------

constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixRounds = 16;  // keys per lane
constexpr int kRadixTile = kRadixThreads * kRadixRounds;  // 4096
constexpr int kWarpSpan = 32 * kRadixRounds;               // 512 keys per warp

__global__ void radix_hist_kernel(const int32_t* __restrict__ keys, int64_t n, int shift,
                                  int32_t* __restrict__ hist, int64_t ntiles) {
  __shared__ int32_t cnt[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t base = (int64_t)blockIdx.x * kRadixTile + (int64_t)warp * kWarpSpan;
  for (int r = 0; r < kRadixRounds; ++r) {
    const int64_t i = base + r * 32 + lane;
    const int d = i < n ? (int)(((uint32_t)keys[i] >> shift) & 255u) : 256;
    const unsigned peers = __match_any_sync(TH_FULL, d);
    if (d < 256 && lane == __ffs(peers) - 1) atomicAdd(&cnt[d], __popc(peers));
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[(int64_t)d * ntiles + blockIdx.x] = cnt[d];
}

__global__ void radix_scatter_kernel(const int32_t* __restrict__ kin, const int32_t* __restrict__ vin,
                                     int32_t* __restrict__ kout, int32_t* __restrict__ vout,
                                     int64_t n, int shift, const int32_t* __restrict__ hist,
                                     int64_t ntiles) {
  __shared__ int32_t wcnt[kRadixWarps][256];
  __shared__ int32_t gbase[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < 256; i += 32) wcnt[warp][i] = 0;
  for (int d = threadIdx.x; d < 256; d += blockDim.x) gbase[d] = hist[(int64_t)d * ntiles + blockIdx.x];
  __syncwarp();
  const int64_t base = (int64_t)blockIdx.x * kRadixTile + (int64_t)warp * kWarpSpan;
  int32_t key[kRadixRounds], val[kRadixRounds], local[kRadixRounds];
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    const int64_t i = base + r * 32 + lane;
    const bool ok = i < n;
    key[r] = ok ? kin[i] : 0;
    val[r] = ok ? vin[i] : 0;
    const int d = ok ? (int)(((uint32_t)key[r] >> shift) & 255u) : 256;
    const unsigned peers = __match_any_sync(TH_FULL, d);
    int32_t b = 0;
    if (ok) b = wcnt[warp][d];
    __syncwarp();
    if (ok && lane == 31 - __clz(peers)) wcnt[warp][d] = b + __popc(peers);
    __syncwarp();
    local[r] = ok ? b + __popc(peers & lt) : -1;
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x) {
    int32_t run = 0;
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
      const int32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    if (local[r] < 0) continue;
    const int d = (int)(((uint32_t)key[r] >> shift) & 255u);
    const int64_t pos = (int64_t)gbase[d] + wcnt[warp][d] + local[r];
    kout[pos] = key[r];
    vout[pos] = val[r];
  }
}

}  // namespace

template <typename T>
int64_t scan_scratch_elems(int64_t n) {
  return ceil_div(n > 0 ? n : 1, kScanTile) + 1;
}

template <typename T>
int scan_exclusive(const T* in, T* out, int64_t n, T* scratch, cudaStream_t st) {
  if (n <= 0) return 0;
  const int64_t nb = ceil_div(n, kScanTile);
  scan_reduce_kernel<T><<<(unsigned)nb, kScanThreads, 0, st>>>(in, scratch, n);
  TH_LAUNCHED();
  scan_partials_kernel<T><<<1, kScanThreads, 0, st>>>(scratch, nb);
  TH_LAUNCHED();
  scan_apply_kernel<T><<<(unsigned)nb, kScanThreads, 0, st>>>(in, out, scratch, n);
  TH_LAUNCHED();
  return 3;
}

template int64_t scan_scratch_elems<int32_t>(int64_t);
template int64_t scan_scratch_elems<int64_t>(int64_t);
template int scan_exclusive<int32_t>(const int32_t*, int32_t*, int64_t, int32_t*, cudaStream_t);
template int scan_exclusive<int64_t>(const int64_t*, int64_t*, int64_t, int64_t*, cudaStream_t);

int64_t radix_hist_elems(int64_t n) { return 256 * ceil_div(n > 0 ? n : 1, kRadixTile); }

int radix_sort_pairs(int32_t* k0, int32_t* v0, int32_t* k1, int32_t* v1, int64_t n, int key_bits,
                     int32_t* hist, int32_t* scan_scratch, cudaStream_t st, int64_t* launches) {
  if (n <= 1 || key_bits <= 0) return 0;
  const int64_t ntiles = ceil_div(n, kRadixTile);
  int cur = 0;
  for (int shift = 0; shift < key_bits; shift += 8) {
    int32_t* ki = cur ? k1 : k0;
    int32_t* vi = cur ? v1 : v0;
    int32_t* ko = cur ? k0 : k1;
    int32_t* vo = cur ? v0 : v1;
    radix_hist_kernel<<<(unsigned)ntiles, kRadixThreads, 0, st>>>(ki, n, shift, hist, ntiles);
    TH_LAUNCHED();
    *launches += 1 + scan_exclusive<int32_t>(hist, hist, 256 * ntiles, scan_scratch, st);
    radix_scatter_kernel<<<(unsigned)ntiles, kRadixThreads, 0, st>>>(ki, vi, ko, vo, n, shift, hist,
                                                                     ntiles);
    TH_LAUNCHED();
    *launches += 1;
    cur ^= 1;
  }
  return cur;
}

}  // namespace th
