// Part of engine.cu (included inside namespace th::{anonymous}); kept in its
// own file so the kernel can be revised in isolation.
//
// K4 materialisation: per-query sorted id lists (the canonical EntityVector /
// TripleVector form, incidence.py:83-91) from entity-major bit rows.
//
// Grid = (row block) x (group of up to 8 row words).  Warp w of a CTA owns
// word j = 8g + w, i.e. queries 32j..32j+31, over the block's rows; the 8
// warps read the 8 words of one 32-byte sector per row, so every row sector
// is fetched from L2 once.  Per 32-row tile a lane loads its row's word, a
// 32x32 bit transpose hands lane b the row mask of query 32j+b.
//   COUNT: per-lane popcounts -> counts[q][blk].
//   WRITE: lane b appends its query's row ids to a 64-entry shared-memory
//          ring; whenever a ring holds 32 ids the whole warp stores them as
//          one coalesced 128-byte run.  Ascending row order is preserved, so
//          every query's output is sorted and duplicate-free.
#pragma once

constexpr int kMatWordsPerCta = 8;
constexpr int kRing = 64;
constexpr int kRingStride = kRing + 1;

// rows = entities; word j of row r = A & ~neg, restricted to live queries
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
  __device__ __forceinline__ uint32_t word(int64_t r, int64_t, int j) const {
    uint32_t x = A[(size_t)r * W + j];
    if (neg) x &= ~neg[(size_t)r * W + j];
    return x & valid_word(j, nq);
  }
};

// rows = triples in tid order; word j of row t = X[subj[t]] & M[rel[t]]
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
  __device__ __forceinline__ uint32_t word(int64_t, int64_t aux, int j) const {
    uint32_t x = X[(size_t)(uint32_t)aux * W + j];
    if (M) x &= M[(size_t)(aux >> 32) * W + j];
    return x & valid_word(j, nq);
  }
};

template <int W>
constexpr int mat_warps() {
  return W < kMatWordsPerCta ? W : kMatWordsPerCta;
}

template <int W, bool WRITE>
constexpr size_t mat_smem_bytes() {
  return WRITE ? (size_t)mat_warps<W>() * 32 * kRingStride * sizeof(int32_t) : 0;
}

// EDGES (COUNT pass over an entity layer): also sum the out-degrees of each
// query's rows -- |T_{h+1}(q)| when the layer is the next hop's frontier
// (incidence.py:214-221: one activated triple per out-edge).  Degrees are
// split into bit planes, one ballot per plane, so a query's sum is
// sum_k popc(mask & plane_k) << k with no per-id work.
struct EdgeSum {
  const int32_t* indptr = nullptr;
  int nplanes = 0;
  int64_t* out = nullptr;  // [nq], accumulated with atomics
};

template <int W, class Src, bool WRITE, bool EDGES = false>
__global__ void __launch_bounds__(32 * kMatWordsPerCta) mat_kernel(Src src, int64_t blk_rows,
                                                                   int nblk, int32_t* counts,
                                                                   const int64_t* base, int32_t* out,
                                                                   int64_t cap, EdgeSum es = {}) {
  extern __shared__ int32_t ring_smem[];
  constexpr int NW = mat_warps<W>();
  constexpr int NG = W / NW;  // word groups
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int blk = blockIdx.x / NG;
  const int j = (blockIdx.x % NG) * NW + warp;
  const int q = 32 * j + lane;
  if (blk >= nblk) return;
  int32_t* ring = ring_smem + (size_t)warp * 32 * kRingStride;
  int32_t* mine = ring + lane * kRingStride;
  int64_t pos = 0;
  int head = 0, fill = 0;
  int32_t total = 0;
  unsigned long long esum = 0;
  if (WRITE && q < src.nq) pos = base[q] + counts[(size_t)q * nblk + blk];
  const int64_t r_begin = (int64_t)blk * blk_rows;
  const int64_t rend = src.nrows < r_begin + blk_rows ? src.nrows : r_begin + blk_rows;
  for (int64_t r0 = r_begin; r0 < rend; r0 += 32) {
    int64_t aux;
    const uint32_t fl = src.prep(r0, aux);
    if (!fl) continue;
    const uint32_t x = ((fl >> lane) & 1u) ? src.word(r0 + lane, aux, j) : 0u;
    if (!__any_sync(TH_FULL, x != 0u)) continue;
    uint32_t m = transpose32(x);
    total += __popc(m);
    if (EDGES) {
      const int64_t r = r0 + lane;
      const uint32_t d = ((fl >> lane) & 1u) ? (uint32_t)(es.indptr[r + 1] - es.indptr[r]) : 0u;
      const int np = 32 - __clz((int)__reduce_max_sync(TH_FULL, d));  // planes this tile needs
      for (int k = 0; k < np; ++k)
        esum += (unsigned long long)__popc(m & __ballot_sync(TH_FULL, (d >> k) & 1u)) << k;
    }
    if (!WRITE) continue;
    while (m) {
      mine[(head + fill) & (kRing - 1)] = (int32_t)(r0 + __ffs(m) - 1);
      ++fill;
      m &= m - 1u;
    }
    __syncwarp();
    unsigned full = __ballot_sync(TH_FULL, fill >= 32);
    while (full) {
      const int b = __ffs(full) - 1;
      full &= full - 1u;
      const int hb = __shfl_sync(TH_FULL, head, b);
      const int64_t pb = __shfl_sync(TH_FULL, pos, b);
      const int32_t id = ring[b * kRingStride + ((hb + lane) & (kRing - 1))];
      if (pb + lane < cap) out[pb + lane] = id;
      if (lane == b) {
        head = (head + 32) & (kRing - 1);
        fill -= 32;
        pos += 32;
      }
    }
    __syncwarp();
  }
  if (WRITE) {
    unsigned rest = __ballot_sync(TH_FULL, fill > 0);
    while (rest) {
      const int b = __ffs(rest) - 1;
      rest &= rest - 1u;
      const int hb = __shfl_sync(TH_FULL, head, b);
      const int fb = __shfl_sync(TH_FULL, fill, b);
      const int64_t pb = __shfl_sync(TH_FULL, pos, b);
      if (lane < fb && pb + lane < cap) out[pb + lane] = ring[b * kRingStride + ((hb + lane) & (kRing - 1))];
    }
  } else if (q < src.nq) {
    counts[(size_t)q * nblk + blk] = total;
    if (EDGES && esum) atomicAdd(reinterpret_cast<unsigned long long*>(es.out + q), esum);
  }
}

