// Part of engine.cu (included inside namespace th::{anonymous}); kept in its
// own file so the kernel can be revised in isolation.
#pragma once

// one lane loads the W words of row r of an entity-major matrix
template <int W>
__device__ __forceinline__ void load_row(const uint32_t* A, int64_t r, bool live, uint32_t (&w)[W]) {
  const uint32_t* p = A + (size_t)r * W;
  if constexpr (W >= 4) {
#pragma unroll
    for (int k = 0; k < W / 4; ++k) {
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (live) v = *reinterpret_cast<const uint4*>(p + 4 * k);
      w[4 * k] = v.x;
      w[4 * k + 1] = v.y;
      w[4 * k + 2] = v.z;
      w[4 * k + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < W; ++k) w[k] = live ? p[k] : 0u;
  }
}

// rows = entities; row word j = A & ~neg, restricted to live queries
template <int W>
struct DenseSrc {
  const uint32_t* A;
  const uint32_t* neg;
  const uint32_t* flags;
  int64_t nrows;
  int nq;
  // flags of rows r0..r0+31 (warp-uniform); aux unused
  __device__ __forceinline__ uint32_t prep(int64_t r0, int64_t& aux) const {
    aux = 0;
    const int64_t left = nrows - r0;
    const uint32_t tail = left >= 32 ? TH_FULL : ((1u << left) - 1u);
    return (flags ? flags[r0 >> 5] : TH_FULL) & tail;
  }
  // the W words of row r into w (zero when !live)
  __device__ __forceinline__ void row(int64_t r, int64_t, bool live, uint32_t (&w)[W]) const {
    load_row<W>(A, r, live, w);
    if (neg && live) {
      uint32_t n[W];
      load_row<W>(neg, r, true, n);
#pragma unroll
      for (int j = 0; j < W; ++j) w[j] &= ~n[j];
    }
#pragma unroll
    for (int j = 0; j < W; ++j) w[j] &= valid_word(j, nq);
  }
};

// rows = triples in tid order; row word j = X[subj[t]] & M[rel[t]]
template <int W>
struct TripleSrc {
  const uint32_t* X;
  const uint32_t* Xf;
  const uint32_t* M;
  const int32_t* subj;
  const uint16_t* rel;
  int64_t nrows;
  int nq;
  __device__ __forceinline__ uint32_t prep(int64_t r0, int64_t& aux) const {
    const int64_t t = r0 + lane_id();
    bool act = false;
    aux = 0;
    if (t < nrows) {
      const int32_t s = subj[t];
      act = (Xf[s >> 5] >> (s & 31)) & 1u;
      aux = ((int64_t)rel[t] << 32) | (uint32_t)s;
    }
    return __ballot_sync(TH_FULL, act);
  }
  __device__ __forceinline__ void row(int64_t, int64_t aux, bool live, uint32_t (&w)[W]) const {
    load_row<W>(X, (int64_t)(uint32_t)aux, live, w);
    if (M && live) {
      uint32_t m[W];
      load_row<W>(M, aux >> 32, true, m);
#pragma unroll
      for (int j = 0; j < W; ++j) w[j] &= m[j];
    }
#pragma unroll
    for (int j = 0; j < W; ++j) w[j] &= valid_word(j, nq);
  }
};

constexpr int kMatThreads = 128;
constexpr int kMatWarps = kMatThreads / 32;

// K4 materialisation: per-query sorted id lists from entity-major bit rows.
// A warp owns a block of rows and walks it 32 rows at a time: lane i loads
// row r0+i (W words, 16-byte loads), one 32x32 bit transpose per word j
// gives lane b the 32-row mask of query 32j+b.  COUNT adds popcounts;
// WRITE visits each query with ids in the tile and lets the lanes holding
// them store their row ids into consecutive slots (one coalesced store per
// query and tile, ascending row order = the canonical sorted form).
template <int W, class Src, bool WRITE>
__global__ void __launch_bounds__(kMatThreads) mat_kernel(Src src, int64_t blk_rows, int nblk,
                                                          int32_t* counts, const int64_t* base,
                                                          int32_t* out, int64_t cap) {
  __shared__ int64_t gbase_s[kMatWarps][WRITE ? 32 * W : 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int blk = gw; blk < nblk; blk += nw) {
    int32_t run[W];
#pragma unroll
    for (int j = 0; j < W; ++j) run[j] = 0;
    if (WRITE) {
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const int q = 32 * j + lane;
        gbase_s[warp][32 * j + lane] = q < src.nq ? base[q] + counts[(size_t)q * nblk + blk] : 0;
      }
      __syncwarp();
    }
    const int64_t r_begin = (int64_t)blk * blk_rows;
    const int64_t rend = src.nrows < r_begin + blk_rows ? src.nrows : r_begin + blk_rows;
    for (int64_t r0 = r_begin; r0 < rend; r0 += 32) {
      int64_t aux;
      const uint32_t fl = src.prep(r0, aux);
      if (!fl) continue;
      uint32_t w[W];
      src.row(r0 + lane, aux, (fl >> lane) & 1u, w);
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const uint32_t t = transpose32(w[j]);
        if (WRITE) {
          unsigned act = __ballot_sync(TH_FULL, t != 0u);
          while (act) {
            const int b = __ffs(act) - 1;
            act &= act - 1u;
            const uint32_t m = __shfl_sync(TH_FULL, t, b);
            const int32_t rb = __shfl_sync(TH_FULL, run[j], b);
            if ((m >> lane) & 1u) {
              const int64_t pos = gbase_s[warp][32 * j + b] + rb + __popc(m & lt);
              if (pos < cap) out[pos] = (int32_t)(r0 + lane);
            }
          }
        }
        run[j] += __popc(t);
      }
    }
    if (!WRITE) {
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const int q = 32 * j + lane;
        if (q < src.nq) counts[(size_t)q * nblk + blk] = run[j];
      }
    }
    __syncwarp();
  }
}

