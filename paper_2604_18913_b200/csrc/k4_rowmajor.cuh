// Part of engine.cu (included inside namespace th::{anonymous}).
//
// Row-major count pass of the list-driven K4 (k4_materialize.cuh).
//
// A layer of a large graph (C4, C5) holds a few bits per 1,024-bit row --
// C4's last layer averages ~36 set bits over 32 words.  The word-per-warp
// count pass read every row as 32 separate 4-byte loads (one per word-warp,
// 32 sectors per load instruction: L1-bound at 86%, 1.75 ms for 1.64 GB on
// C4 k=3).  Here a warp reads whole rows (one coalesced 128-byte load per
// row, lane j = word j = queries 32j..32j+31) and counts bits column-wise
// with a carry-save adder tree: per (query, block) totals for the write
// pass, over the SAME row blocks the write pass uses (whole 1,024-row
// chunks, blk_rows from the device-side row count, as in mat_unit).
//
// Measured and rejected (C4 k=3, 1,024 seeds): a row-major WRITE pass that
// scatters every id to its query's cursor (one 4-byte store per id into ~1M
// concurrently open per-query runs: partially written sectors thrash L2,
// 14.2 -> 21.7 ms), and one that stages a block's ids query-major in shared
// memory (per-query bookkeeping of 1,024 queries per ~7K-id block: ~4.5
// warp instructions per id, 14.2 -> 23.5 ms).  The transposing write pass
// keeps 32 queries per warp, so its per-query staging stays small.
#pragma once

constexpr int kRsWarps = 16;   // warps per CTA
constexpr int kRsUnroll = 8;   // rows in flight per warp (the adder tree sums 8)

template <int W>
struct RowMajorSrc {
  const uint32_t* A;
  const uint32_t* neg;
  const int32_t* rows;     // ascending row list (nullptr: every row, filtered by `flags`)
  const int32_t* n_dev;    // its length (device; nullptr: n_host)
  int nq;
  const uint32_t* flags = nullptr;  // dense sources: "row is nonzero" bits
  int64_t n_host = 0;
  __device__ __forceinline__ int64_t count() const { return n_dev ? (int64_t)*n_dev : n_host; }
};

// kRsUnroll rows starting at list position i (< end): row numbers and this
// lane's words (lane j = word j)
template <int W>
__device__ __forceinline__ void rs_load(const RowMajorSrc<W>& src, int64_t i, int64_t end,
                                        int32_t (&v)[kRsUnroll], uint32_t (&x)[kRsUnroll],
                                        uint32_t valid) {
  const unsigned lane = lane_id();
  int32_t mine = -1;
  if ((int64_t)lane < kRsUnroll && i + lane < end) {
    if (src.rows) {
      mine = __ldg(src.rows + i + lane);
    } else {
      const int64_t r = i + lane;
      mine = (!src.flags || ((__ldg(src.flags + (r >> 5)) >> (r & 31)) & 1u)) ? (int32_t)r : -1;
    }
  }
#pragma unroll
  for (int u = 0; u < kRsUnroll; ++u) v[u] = __shfl_sync(TH_FULL, mine, u);
#pragma unroll
  for (int u = 0; u < kRsUnroll; ++u) {
    uint32_t w = 0u;
    if (v[u] >= 0 && lane < (unsigned)W) {
      const size_t at = (size_t)v[u] * W + lane;
      w = __ldcg(src.A + at);
      if (src.neg) w &= ~__ldcg(src.neg + at);
    }
    x[u] = w & valid;
  }
}

// full adder on bit planes (two LOP3s)
__device__ __forceinline__ void fa(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& cy) {
  s = a ^ b ^ c;
  cy = (a & b) | (c & (a ^ b));
}

// adds plane k's bits into cnt[b * 32 + lane] with weight 2^k
template <typename C>
__device__ __forceinline__ void rs_flush_plane(uint32_t p, int k, C* cnt) {
  const unsigned lane = lane_id();
  while (p) {
    const int b = __ffs(p) - 1;
    p &= p - 1u;
    cnt[b * 32 + lane] += (C)(1u << k);
  }
}

// Per-query bit counts of list rows [lo, hi) added to cnt[b*32 + lane]
// (query 32 lane + b) without per-bit work: eight rows at a time are summed
// column-wise by a carry-save adder tree into a 4-bit bit-sliced count,
// added into six running planes (counts up to 63) that are flushed to the
// shared counters every 56 rows.
template <int W, typename C>
__device__ __forceinline__ uint32_t rs_count_sliced(const RowMajorSrc<W>& src, int64_t lo, int64_t hi,
                                                    C* cnt, uint32_t valid) {
  static_assert(kRsUnroll == 8, "the adder tree sums 8 rows");
  uint32_t c0 = 0u, c1 = 0u, c2 = 0u, c3 = 0u, c4 = 0u, c5 = 0u;
  uint32_t word_bits = 0u;  // this lane's word over the slice (the bucket pass's group count)
  int acc = 0;
  for (int64_t i = lo; i < hi; i += kRsUnroll) {
    int32_t v[kRsUnroll];
    uint32_t x[kRsUnroll];
    rs_load<W>(src, i, hi, v, x, valid);
#pragma unroll
    for (int u = 0; u < kRsUnroll; ++u) word_bits += __popc(x[u]);
    uint32_t a1, b1, a2, b2, p0, b4, q1, k1;
    fa(x[0], x[1], x[2], a1, b1);
    fa(x[3], x[4], x[5], a2, b2);
    const uint32_t a3 = x[6] ^ x[7], b3 = x[6] & x[7];
    fa(a1, a2, a3, p0, b4);
    fa(b1, b2, b3, q1, k1);
    const uint32_t p1 = q1 ^ b4, k2 = q1 & b4;
    const uint32_t p2 = k1 ^ k2, p3 = k1 & k2;
    // running planes += (p3 p2 p1 p0)
    uint32_t cy, t;
    t = c0 ^ p0; cy = c0 & p0; c0 = t;
    fa(c1, p1, cy, t, cy); c1 = t;
    fa(c2, p2, cy, t, cy); c2 = t;
    fa(c3, p3, cy, t, cy); c3 = t;
    t = c4 ^ cy; cy = c4 & cy; c4 = t;
    c5 ^= cy;
    acc += kRsUnroll;
    if (acc >= 56) {
      rs_flush_plane(c0, 0, cnt); rs_flush_plane(c1, 1, cnt); rs_flush_plane(c2, 2, cnt);
      rs_flush_plane(c3, 3, cnt); rs_flush_plane(c4, 4, cnt); rs_flush_plane(c5, 5, cnt);
      c0 = c1 = c2 = c3 = c4 = c5 = 0u;
      acc = 0;
    }
  }
  rs_flush_plane(c0, 0, cnt); rs_flush_plane(c1, 1, cnt); rs_flush_plane(c2, 2, cnt);
  rs_flush_plane(c3, 3, cnt); rs_flush_plane(c4, 4, cnt); rs_flush_plane(c5, 5, cnt);
  return word_bits;
}

// EDGES variant: per-bit counting plus each row's out-degree per query
// (|T_{h+1}(q)|; the layers that need it are the small early ones)
template <int W>
__device__ __forceinline__ void rs_count_edges(const RowMajorSrc<W>& src, int64_t lo, int64_t hi,
                                               uint32_t* cnt, uint32_t* esum, const EdgeSum& es,
                                               uint32_t valid) {
  const unsigned lane = lane_id();
  for (int64_t i = lo; i < hi; i += kRsUnroll) {
    int32_t v[kRsUnroll];
    uint32_t x[kRsUnroll];
    rs_load<W>(src, i, hi, v, x, valid);
#pragma unroll
    for (int u = 0; u < kRsUnroll; ++u) {
      uint32_t m = x[u];
      // (the degree of the layer's own row: es.indptr is that graph's)
      const uint32_t d = m ? degree(es, v[u]) : 0u;
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1u;
        cnt[b * 32 + lane] += 1u;
        esum[b * 32 + lane] += d;
      }
    }
  }
}

// per-(warp, query) counters: 32-bit with degree sums, else 16-bit (a warp
// slice holds < 2^16 rows for any layer below 2^31 rows), so the plain count
// pass fits four 16-warp CTAs per SM
template <bool EDGES>
using RsCnt = std::conditional_t<EDGES, uint32_t, uint16_t>;

template <bool EDGES>
constexpr size_t rs_count_smem() {
  return (size_t)(EDGES ? 2 : 1) * kRsWarps * 1024 * sizeof(RsCnt<EDGES>);
}

// counts[q * nblk + blk] = bits of query q in row block blk of the list (or
// of the entity range, dense sources) -- the write pass's partition: whole
// kChunkRows chunks, blk_rows from the row count.  One CTA per block; its
// warps take contiguous slices.
// (gcount, when given: [nblk * kRsWarps + 1][32] bits of word j in each
// warp's slice -- the bucket write pass's partition, see below)
template <int W, bool EDGES>
__global__ void __launch_bounds__(32 * kRsWarps, 4) rs_count_kernel(RowMajorSrc<W> src, int nblk,
                                                                 int32_t* counts, EdgeSum es,
                                                                 uint32_t* gcount = nullptr) {
  // dynamic: [kRsWarps][1024] counters (+ [kRsWarps][1024] degree sums; a
  // warp's degree sum per query covers distinct rows: <= T < 2^32)
  extern __shared__ uint32_t rs_smem_words[];
  using C = RsCnt<EDGES>;
  C* rs_smem = reinterpret_cast<C*>(rs_smem_words);
  const int warp = threadIdx.x >> 5;
  const unsigned lane = lane_id();
  const int blk = blockIdx.x;
  if (blk >= nblk) return;
  C* cnt = rs_smem + warp * 1024;
  uint32_t* esum = rs_smem_words + (kRsWarps + warp) * 1024;  // (EDGES: C is 32-bit)
  const int64_t nrows = src.count();
  int64_t blk_rows = (nrows + nblk - 1) / nblk;
  blk_rows = blk_rows < kChunkRows ? kChunkRows : (blk_rows + kChunkRows - 1) / kChunkRows * kChunkRows;
  const int64_t r0 = (int64_t)blk * blk_rows;
  const int64_t r1 = nrows < r0 + blk_rows ? nrows : r0 + blk_rows;
  if (r0 >= r1) {
    // (blocks past the layer's rows: zero counts, no shared-memory work)
    for (int q = threadIdx.x; q < src.nq; q += blockDim.x) counts[(size_t)q * nblk + blk] = 0;
    if (gcount) gcount[(size_t)(blk * kRsWarps + warp) * 32 + lane] = 0u;
    return;
  }
  const int64_t per = r1 > r0 ? ((r1 - r0 + kRsWarps - 1) / kRsWarps + kRsUnroll - 1) / kRsUnroll * kRsUnroll
                              : 0;
  const int64_t lo = r0 + warp * per < r1 ? r0 + warp * per : r1;
  const int64_t hi = lo + per < r1 ? lo + per : r1;
  const uint32_t valid = lane < (unsigned)W ? valid_word((int)lane, src.nq) : 0u;
#pragma unroll 8
  for (int b = 0; b < 32; ++b) {
    cnt[b * 32 + lane] = 0;
    if (EDGES) esum[b * 32 + lane] = 0u;
  }
  if constexpr (EDGES) {
    rs_count_edges<W>(src, lo, hi, cnt, esum, es, valid);
  } else {
    const uint32_t wb = rs_count_sliced<W>(src, lo, hi, cnt, valid);
    if (gcount) gcount[(size_t)(blk * kRsWarps + warp) * 32 + lane] = wb;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < src.nq; q += blockDim.x) {
    const int at = (q & 31) * 32 + (q >> 5);
    uint32_t t = 0u;
    unsigned long long e = 0ull;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
      t += rs_smem[w * 1024 + at];
      if (EDGES) e += rs_smem_words[(kRsWarps + w) * 1024 + at];
    }
    counts[(size_t)q * nblk + blk] = (int32_t)t;
    if (EDGES && e) atomicAdd(reinterpret_cast<unsigned long long*>(es.out + q), e);
  }
}

// ---------------------------------------------------------------------------
// Bucketed write pass for list-driven layers (C4 / C5 last layers: a few
// bits per 1,024-bit row, ~450M ids per wave).  Two streaming passes over
// the row partition of rs_count instead of the transposing write pass
// (which spends ~3.8 warp instructions per id on per-tile transposes,
// atomics and ring flushes when a tile holds about one bit per word):
//
//   scatter  a warp reads its slice's rows whole (lane j = word j) and
//            appends (row - block start) << 5 | bit for every set bit of its
//            word to group j's run -- groups are the 32-query words, laid
//            out at the output offsets of their queries (off[32 j]), each
//            (block, warp) slice at its prefix of gcount.  Rows ascend in a
//            run, so a group's entries are in row order.
//   gather   a warp takes one (block, group) run and moves every entry to
//            its query's output (off[q] + the query's count in earlier
//            blocks + its rank): 32 entries per step, ranks within the step
//            from __match_any_sync, ids resolved through the row list.
//
// Each pass keeps 32 write runs open per warp, whose partially written
// sectors merge in L2 while the entry buffer is L2-sized: the passes win
// below kBucketMaxIds ids per layer (C4 k=2's 14M-id last layer: wave 1.39
// -> 1.18 ms) and lose badly above (C4 k=3's 457M ids: the scatter issues
// one L2 sector write per id, 10.5 -> 20.8 ms), where the transposing write
// pass runs instead -- chosen on the device from the layer's total.

// exclusive scan of gcount[e][j] over e for one group j per CTA (in place;
// entry n_slices holds the group total)
__global__ void bucket_scan_kernel(uint32_t* gcount, int n_slices, const int64_t* layer_total) {
  if (*layer_total > kBucketMaxIds) return;
  __shared__ uint32_t ws[32];
  const int j = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t carry = 0u;
  for (int e0 = 0; e0 < n_slices; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    const uint32_t v = e < n_slices ? gcount[(size_t)e * 32 + j] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(TH_FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(TH_FULL, w, o);
        if (lane >= o) w += y;
      }
      ws[lane] = w;
    }
    __syncthreads();
    if (e < n_slices) gcount[(size_t)e * 32 + j] = carry + (warp ? ws[warp - 1] : 0u) + x - v;
    carry += ws[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) gcount[(size_t)n_slices * 32 + j] = carry;
}

// the row block of rs_count: list rows [r0, r1)
__device__ __forceinline__ void rs_block(int64_t nrows, int nblk, int blk, int64_t& r0, int64_t& r1) {
  int64_t blk_rows = (nrows + nblk - 1) / nblk;
  blk_rows = blk_rows < kChunkRows ? kChunkRows : (blk_rows + kChunkRows - 1) / kChunkRows * kChunkRows;
  r0 = (int64_t)blk * blk_rows;
  r1 = nrows < r0 + blk_rows ? nrows : r0 + blk_rows;
}

template <int W>
__global__ void __launch_bounds__(32 * kRsWarps) bucket_scatter_kernel(RowMajorSrc<W> src, int nblk,
                                                                       const uint32_t* __restrict__ gpre,
                                                                       const int64_t* __restrict__ off,
                                                                       uint32_t* P,
                                                                       const int64_t* layer_total) {
  if (*layer_total > kBucketMaxIds) return;
  const int warp = threadIdx.x >> 5;
  const unsigned lane = lane_id();
  const int blk = blockIdx.x;
  int64_t r0, r1;
  rs_block(src.count(), nblk, blk, r0, r1);
  if (blk >= nblk || r0 >= r1) return;
  // (the slices of rs_count_kernel)
  const int64_t per = ((r1 - r0 + kRsWarps - 1) / kRsWarps + kRsUnroll - 1) / kRsUnroll * kRsUnroll;
  const int64_t lo = r0 + warp * per < r1 ? r0 + warp * per : r1;
  const int64_t hi = lo + per < r1 ? lo + per : r1;
  const uint32_t valid = lane < (unsigned)W ? valid_word((int)lane, src.nq) : 0u;
  // (entry positions relative to the layer's first output: the buffer holds
  // kBucketMaxIds entries whatever the result capacity)
  int64_t pos = 0;
  if (valid) pos = off[32 * lane] - off[0] + gpre[(size_t)(blk * kRsWarps + warp) * 32 + lane];
  for (int64_t i = lo; i < hi; i += kRsUnroll) {
    int32_t v[kRsUnroll];
    uint32_t x[kRsUnroll];
    rs_load<W>(src, i, hi, v, x, valid);
#pragma unroll
    for (int u = 0; u < kRsUnroll; ++u) {
      uint32_t m = x[u];
      const uint32_t rel = (uint32_t)(i + u - r0) << 5;
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1u;
        if (pos < kBucketMaxIds) P[pos] = rel | (uint32_t)b;
        ++pos;
      }
    }
  }
}

template <int W>
__global__ void __launch_bounds__(kThreads) bucket_gather_kernel(
    const int32_t* __restrict__ rows, const int32_t* __restrict__ map, const int32_t* n_dev, int nq,
    int nblk, const uint32_t* __restrict__ gpre, const int32_t* __restrict__ counts,
    const int64_t* __restrict__ off, const uint32_t* __restrict__ P, int32_t* out, int64_t cap,
    const int64_t* layer_total) {
  if (*layer_total > kBucketMaxIds) return;
  __shared__ uint32_t inc_s[kThreads / 32][32];
  uint32_t* inc = inc_s[threadIdx.x >> 5];
  const unsigned lane = lane_id();
  const int64_t nrows = *n_dev;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  inc[lane] = 0u;
  __syncwarp();
  for (int64_t unit = gw; unit < (int64_t)nblk * W; unit += nw) {
    const int blk = (int)(unit / W), j = (int)(unit % W);
    if (32 * j >= nq) continue;
    int64_t r0, r1;
    rs_block(nrows, nblk, blk, r0, r1);
    const int64_t g0 = off[32 * j] - off[0];
    const int64_t start = g0 + gpre[(size_t)(blk * kRsWarps) * 32 + j];
    const int64_t end = g0 + gpre[(size_t)((blk + 1) * kRsWarps) * 32 + j];
    const int q = 32 * j + (int)lane;
    int64_t cur = q < nq ? off[q] + counts[(size_t)q * nblk + blk] : 0;
    for (int64_t i0 = start; i0 < end; i0 += 32) {
      const int64_t i = i0 + lane;
      const bool ok = i < end;
      uint32_t e = 0u;
      int32_t id = 0;
      if (ok) {
        e = i < kBucketMaxIds ? __ldcs(P + i) : 0u;
        const int32_t v = __ldg(rows + r0 + (e >> 5));
        id = map ? __ldg(map + v) : v;
      }
      const int b = (int)(e & 31u);
      const unsigned grp = __match_any_sync(TH_FULL, ok ? b : 32 + (int)lane);
      const int rank = __popc(grp & lanemask_lt());
      const int64_t at = __shfl_sync(TH_FULL, cur, b) + rank;
      if (ok && at < cap) out[at] = id;
      if (ok && rank == 0) inc[b] = (uint32_t)__popc(grp);
      __syncwarp();
      cur += inc[lane];
      inc[lane] = 0u;
      __syncwarp();
    }
  }
}
