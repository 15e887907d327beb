// Part of engine.cu (included inside namespace th::{anonymous}); kept in its
// own file so the kernel can be revised in isolation.
//
// K4 materialisation: per-query sorted id lists (the canonical EntityVector /
// TripleVector form, incidence.py:83-91) from entity-major bit rows.
//
// Grid = (row block) x (group of NW row words).  Warp w of a CTA owns word
// j = NW*g + w, i.e. queries 32j..32j+31, and walks its block's rows in
// chunks of 32 tiles x 32 rows:
//   A. per tile, lane i loads row (r0+i)'s word j and a 32x32 bit transpose
//      hands lane b the tile mask of query 32j+b; the 32 masks of the chunk
//      go to shared memory as S[b][t] (lane b: its query's tile masks).
//   COUNT: per-lane popcounts -> counts[q][blk]  (+ optional degree sums).
//   WRITE: query by query, the warp takes S[b][0..31] (lane t = tile t),
//          scans the popcounts for offsets, extracts the row ids of its tile
//          into a shared staging run (ascending by construction), then
//          stores the whole run coalesced at the query's cursor.
// Ascending row order is preserved, so every query's output is sorted and
// duplicate-free.  Per output id this costs about one extraction step on
// one lane plus 1/32 of a coalesced store, instead of a per-lane serial
// append with ring flushes.
#pragma once

constexpr int kMatWordsPerCta = 8;          // warps per CTA (one row word each)
// list layers with at most this many ids take the bucketed write passes
// (k4_rowmajor.cuh): their 4-byte entry buffer stays L2-sized
constexpr int64_t kBucketMaxIds = int64_t(20) << 20;
constexpr int kChunkRows = 1024;            // 32 tiles of 32 rows
constexpr int kSStride = 33;                // S[b][t] row stride (bank-conflict free)

// rows = entities; word j of row r = A & ~neg, restricted to live queries
template <int W>
struct DenseSrc {
  const uint32_t* A;
  const uint32_t* neg;
  const uint32_t* flags;
  int64_t nrows;
  int nq;
  const int32_t* map = nullptr;  // optional row -> output id (ascending), e.g. shard local -> global
  static constexpr bool kDense = true;
  static constexpr bool kRing = false;
  // lane t: flags of rows [r0+32t, r0+32t+32) below `rend` (r0 % 32 == 0)
  __device__ __forceinline__ uint32_t chunk_flags(int64_t r0, int64_t rend) const {
    const int64_t t0 = r0 + 32 * (int64_t)lane_id();
    if (t0 >= rend) return 0u;
    const int64_t left = rend - t0;
    const uint32_t tail = left >= 32 ? TH_FULL : ((1u << left) - 1u);
    return (flags ? flags[t0 >> 5] : TH_FULL) & tail;
  }
  __device__ __forceinline__ bool chunk_any(int64_t r0, int64_t rend) const {
    return __any_sync(TH_FULL, chunk_flags(r0, rend) != 0u);
  }
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
  __device__ __forceinline__ int64_t rows_dev() const { return nrows; }
  __device__ __forceinline__ int32_t id(int64_t r) const { return map ? map[r] : (int32_t)r; }
  // the graph row of list position r (unmapped: out-degrees are the row's)
  __device__ __forceinline__ int32_t row(int64_t r) const { return (int32_t)r; }
};

// rows = the ascending list of nonzero entity rows of a layer (compacted
// from its flag bitmap), so the work is proportional to the rows a layer
// actually reached rather than to E; the list length lives on the device
template <int W>
struct ListSrc {
  const uint32_t* A;
  const uint32_t* neg;
  const int32_t* rows;
  const int32_t* n_dev;
  int64_t nrows;  // capacity (host-side grid sizing)
  int nq;
  const int32_t* map = nullptr;
  static constexpr bool kDense = true;
  static constexpr bool kRing = true;
  __device__ __forceinline__ uint32_t chunk_flags(int64_t r0, int64_t rend) const {
    const int64_t t0 = r0 + 32 * (int64_t)lane_id();
    if (t0 >= rend) return 0u;
    const int64_t left = rend - t0;
    return left >= 32 ? TH_FULL : ((1u << left) - 1u);
  }
  __device__ __forceinline__ bool chunk_any(int64_t r0, int64_t rend) const { return r0 < rend; }
  __device__ __forceinline__ uint32_t word(int64_t r, int64_t, int j) const {
    const size_t v = (size_t)rows[r];
    uint32_t x = A[v * W + j];
    if (neg) x &= ~neg[v * W + j];
    return x & valid_word(j, nq);
  }
  __device__ __forceinline__ int64_t rows_dev() const { return *n_dev; }
  __device__ __forceinline__ int32_t id(int64_t r) const {
    const int32_t v = __ldg(rows + r);
    return map ? __ldg(map + v) : v;
  }
  __device__ __forceinline__ int32_t row(int64_t r) const { return __ldg(rows + r); }
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
  const int32_t* map = nullptr;  // local triple -> global tid (shards)
  static constexpr bool kDense = false;
  static constexpr bool kRing = false;
  __device__ __forceinline__ bool chunk_any(int64_t, int64_t) const { return true; }
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
  __device__ __forceinline__ int64_t rows_dev() const { return nrows; }
  __device__ __forceinline__ int32_t id(int64_t r) const { return map ? map[r] : (int32_t)r; }
  __device__ __forceinline__ int32_t row(int64_t r) const { return (int32_t)r; }
};

template <int W>
constexpr int mat_warps() {
  return W < kMatWordsPerCta ? W : kMatWordsPerCta;
}

constexpr unsigned kSparseBits = 5;       // tiles with <= this many bits per lane skip the transpose
constexpr unsigned kCoopIdsPerQuery = 48;  // chunk ids per touched query for the cooperative write

// per-warp shared words: WRITE = S (32 x kSStride) + the staging run (a
// whole chunk's ids of one query: final int32 ids for entity layers of small
// graphs, 16-bit chunk positions for list-driven layers, which resolve them
// through the row list on the way out -- 6.1 KB per warp, four 8-warp CTAs
// per SM instead of three); COUNT = per-query counters + degree sums.
// (Round 2: list-driven layers dropped their per-lane rings for sparse
// chunks -- every chunk is written query by query -- C4 k=3 9.28 -> 9.19 ms;
// capping the run at 256 / 512 ids to fit five / four CTAs per SM, with
// longer runs stored lane by lane, lost: 11.5 / 10.5 ms.)
template <bool WRITE, bool RING = false>
constexpr size_t mat_warp_words() {
  return WRITE ? (size_t)(32 * kSStride + (RING ? kChunkRows / 2 : kChunkRows)) : 64;
}

// per-warp words of a write pass that loads cached masks: the staging run
template <bool RING>
constexpr size_t mat_load_words() {
  return RING ? kChunkRows / 2 : kChunkRows;
}

// CTA-shared words of an EDGES count pass (degree planes, see mat_unit)
constexpr size_t kEdgeWords = 32 * 8 + 64;

template <int W, bool WRITE, bool RING = false>
constexpr size_t mat_smem_bytes() {
  return ((size_t)mat_warps<W>() * mat_warp_words<WRITE, RING>() + (WRITE ? 0 : kEdgeWords)) *
         sizeof(uint32_t);
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

__device__ __forceinline__ uint32_t degree(const EdgeSum& es, int32_t v) {
  return (uint32_t)(es.indptr[v + 1] - es.indptr[v]);
}

__device__ __forceinline__ int warp_incl_scan(int v) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(TH_FULL, v, o);
    if (lane >= (unsigned)o) v += y;
  }
  return v;
}

// Cached tile masks (small graphs): the count pass also stores each chunk's
// transposed masks S and its (touched queries, ids) summary to global
// memory, and the write pass starts from them instead of redoing the
// loads and transposes.  Layout: Sg[((chunk * W + j) * 32 + b) * 32 + t].
struct SCache {
  uint32_t* S = nullptr;
  uint2* meta = nullptr;
  unsigned* work = nullptr;  // unit counter of the write pass (zeroed by the count pass)
};

// one (row block, word) unit of a pass: warp `warp` of its CTA, word j
template <int W, class Src, bool WRITE, bool EDGES, int CACHE>
__device__ __forceinline__ void mat_unit(const Src& src, int nblk, int32_t* counts,
                                         const int64_t* base, int32_t* out, int64_t cap,
                                         const EdgeSum& es, const SCache& sc, int blk, int j,
                                         int warp, int lane) {
  // CACHE 1 = count pass that stores S, CACHE 2 = write pass that loads it
  constexpr bool BUILD_S = WRITE ? CACHE != 2 : CACHE == 1;
  constexpr bool LOAD_S = WRITE && CACHE == 2;
  extern __shared__ uint32_t mat_smem[];
  constexpr int NW = mat_warps<W>();
  const int q = 32 * j + lane;
  if (blk >= nblk) return;
  // WRITE: S[32][kSStride] + staging run; COUNT: per-query counters
  constexpr bool RING = Src::kRing;
  // count pass that builds S: S + per-query counters only (no staging run)
  constexpr size_t kWarpWords = BUILD_S && !WRITE ? (size_t)(32 * kSStride + 64)
                                                  : mat_warp_words<WRITE, RING>();
  uint32_t* S = LOAD_S ? nullptr : mat_smem + (size_t)warp * kWarpWords;
  using StgT = std::conditional_t<RING, uint16_t, int32_t>;
  StgT* stg = LOAD_S ? reinterpret_cast<StgT*>(mat_smem + (size_t)warp * mat_load_words<RING>())
                     : reinterpret_cast<StgT*>(S + 32 * kSStride);
  // COUNT: [32] ids + [32] degree sums per query (sparse tiles), after S
  // when the pass also builds S
  uint32_t* cnt = BUILD_S && !WRITE ? S + 32 * kSStride : S;  // (unused when LOAD_S)
  uint32_t* ecnt = cnt + 32;
  // EDGES: CTA-shared degree planes [32 tiles][8], plane counts [32], big-row masks [32]
  uint32_t* eplanes = mat_smem + (size_t)NW * kWarpWords;
  uint32_t eplane_cnt[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
  if (!WRITE) {
    cnt[lane] = 0u;
    ecnt[lane] = 0u;
    __syncwarp();
  }
  int64_t pos = 0;
  int32_t total = 0;
  unsigned long long esum = 0;
  if (WRITE && q < src.nq) pos = base[q] + counts[(size_t)q * nblk + blk];
  // rows per block from the device-side row count (whole 1024-row chunks)
  const int64_t nrows = src.rows_dev();
  int64_t blk_rows = (nrows + nblk - 1) / nblk;
  blk_rows = blk_rows < kChunkRows ? kChunkRows : (blk_rows + kChunkRows - 1) / kChunkRows * kChunkRows;
  const int64_t r_begin = (int64_t)blk * blk_rows;
  const int64_t rend = nrows < r_begin + blk_rows ? nrows : r_begin + blk_rows;
  for (int64_t c0 = r_begin; c0 < rend; c0 += kChunkRows) {
    // (the cached write pass never reads the layer or its flags -- callers
    // recycle both once the count pass is done -- so the count pass
    // records empty chunks in the meta instead)
    if (!LOAD_S && !src.chunk_any(c0, rend)) {
      if (BUILD_S && !WRITE && lane == 0)
        sc.meta[(size_t)(c0 / kChunkRows) * W + j] = make_uint2(0u, 0u);
      continue;
    }
    // keep the CTA's warps (words of the same rows) on the same chunk so
    // each row sector they share is fetched once and hit in L1 by the
    // others (the write phase drifts them apart; so does the count pass
    // over a list of scattered rows: C4's last layer read 5.65 GB from
    // DRAM in the count pass against 1.93 GB in the synchronised write
    // pass; EDGES passes synchronise for their degree planes anyway)
    if ((WRITE ? !LOAD_S : !EDGES) && NW > 1) __syncthreads();
    if constexpr (!WRITE && !BUILD_S && !EDGES) {
      // plain count pass: a bit-sliced vertical popcount -- every lane adds
      // its row words of the chunk's 32 tiles into six counter planes
      // (ripple carry, 12 ops per word, no divergence), and one transpose
      // per plane at the end gives each query's count: 6 transposes per
      // chunk instead of one per dense tile plus per-bit atomics on sparse
      // ones
      uint32_t c[6] = {0u, 0u, 0u, 0u, 0u, 0u};
      uint32_t cfl = 0u;
      if constexpr (Src::kDense) cfl = src.chunk_flags(c0, rend);
#pragma unroll 1
      for (int t0 = 0; t0 < 32; t0 += 8) {
        uint32_t x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t r0 = c0 + 32 * (t0 + u);
          int64_t aux = 0;
          uint32_t fl;
          if constexpr (Src::kDense) fl = __shfl_sync(TH_FULL, cfl, t0 + u);
          else fl = r0 < rend ? src.prep(r0, aux) : 0u;
          x[u] = ((fl >> lane) & 1u) ? src.word(r0 + lane, aux, j) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint32_t cy = x[u];
#pragma unroll
          for (int i = 0; i < 6; ++i) {
            const uint32_t t = c[i] & cy;
            c[i] ^= cy;
            cy = t;
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 6; ++i)
        if (__any_sync(TH_FULL, c[i] != 0u)) total += __popc(transpose32(c[i])) << i;
      continue;
    }
    const size_t sbase = ((size_t)(c0 / kChunkRows) * W + j) * 1024;
    // ---- A: tile masks of this chunk, S[b][t] = rows of tile t in query b.
    // Loads of 8 tiles are issued before their transposes (memory-level
    // parallelism); dense sources get all 32 tile flags from one load.
    // Dense tiles go through the 32x32 butterfly transpose; sparse tiles
    // (at most kSparseBits bits on any lane) scatter their few bits with
    // shared-memory atomics instead, so a tile costs O(set bits) there.
    uint32_t touched = 0u;  // WRITE: queries with ids in this chunk
    uint32_t nbits = 0u;    // WRITE: set bits seen by this lane (its rows)
    uint32_t cflags = 0u;   // lane t: flags of tile t (dense sources)
    if constexpr (LOAD_S) {
      const uint2 mt = sc.meta[(size_t)(c0 / kChunkRows) * W + j];
      touched = mt.x;
      nbits = lane == 0 ? mt.y : 0u;  // the warp sum below restores the chunk's ids
    }
    if constexpr (Src::kDense && !LOAD_S) cflags = src.chunk_flags(c0, rend);
    if constexpr (EDGES) {
      // degree bit planes of the chunk's rows, once per CTA (they depend on
      // the rows only; every word-warp of the CTA reads them)
      __syncthreads();  // the previous chunk's readers are done
      for (int t = warp; t < 32; t += NW) {
        const uint32_t ft = __shfl_sync(TH_FULL, cflags, t);
        const uint32_t d = ((ft >> lane) & 1u) ? degree(es, src.row(c0 + 32 * t + lane)) : 0u;
        const uint32_t lo = d & 0xffu;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t pk = __ballot_sync(TH_FULL, (lo >> k) & 1u);
          if (lane == 0) eplanes[t * 8 + k] = pk;
        }
        const uint32_t big = __ballot_sync(TH_FULL, d > 0xffu);
        const unsigned mx = __reduce_max_sync(TH_FULL, lo);
        if (lane == 0) {
          eplanes[256 + t] = 32 - __clz((int)mx);
          eplanes[288 + t] = big;
        }
      }
      __syncthreads();
    }
#pragma unroll 1
    for (int t0 = 0; t0 < (LOAD_S ? 0 : 32); t0 += 8) {
      uint32_t x[8], fl[8];
      int64_t aux[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t r0 = c0 + 32 * (t0 + u);
        if constexpr (Src::kDense) {
          fl[u] = __shfl_sync(TH_FULL, cflags, t0 + u);
          aux[u] = 0;
        } else {
          fl[u] = r0 < rend ? src.prep(r0, aux[u]) : 0u;
        }
        x[u] = ((fl[u] >> lane) & 1u) ? src.word(r0 + lane, aux[u], j) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + u;
        const int64_t r = c0 + 32 * t + lane;
        const uint32_t xu = x[u];
        if (WRITE || BUILD_S) nbits += __popc(xu);
        const bool anyx = __any_sync(TH_FULL, xu != 0u);
        const unsigned mx = anyx ? __reduce_max_sync(TH_FULL, (unsigned)__popc(xu)) : 0u;
        if (mx > kSparseBits) {
          const uint32_t m = transpose32(xu);
          if (EDGES) {
            // low 8 bits by the shared bit planes; the rare rows of degree
            // >= 256 add their high part row by row
            // (planes read as two broadcast 16-byte loads; the upper four
            // only when a row of the tile has degree >= 16)
            const int np = (int)eplanes[256 + t];
            const uint4* pp = reinterpret_cast<const uint4*>(eplanes + t * 8);
            const uint4 p0 = pp[0];
            eplane_cnt[0] += __popc(m & p0.x);
            eplane_cnt[1] += __popc(m & p0.y);
            eplane_cnt[2] += __popc(m & p0.z);
            eplane_cnt[3] += __popc(m & p0.w);
            if (np > 4) {
              const uint4 p1 = pp[1];
              eplane_cnt[4] += __popc(m & p1.x);
              eplane_cnt[5] += __popc(m & p1.y);
              eplane_cnt[6] += __popc(m & p1.z);
              eplane_cnt[7] += __popc(m & p1.w);
            }
            uint32_t bg = eplanes[288 + t] & m;
            while (bg) {
              const int i = __ffs(bg) - 1;
              bg &= bg - 1u;
              esum += (unsigned long long)(degree(es, src.row(c0 + 32 * t + i)) >> 8) << 8;
            }
          }
          if (BUILD_S) {
            S[lane * kSStride + t] = m;
            touched |= __ballot_sync(TH_FULL, m != 0u);
          }
          if (!WRITE) total += __popc(m);
        } else {
          if (BUILD_S) S[lane * kSStride + t] = 0u;
          if (anyx) {
            uint32_t d = 0u;
            if (EDGES && xu) d = degree(es, src.row(r));
            if (BUILD_S) {
              __syncwarp();
              touched |= __reduce_or_sync(TH_FULL, xu);
            }
            uint32_t y = xu;
            while (y) {
              const int b = 31 - __clz((int)y);
              if (BUILD_S) atomicOr(&S[b * kSStride + t], 1u << lane);
              if (!WRITE) {
                atomicAdd(&cnt[b], 1u);
                if (EDGES) atomicAdd(&ecnt[b], d);
              }
              y ^= 1u << b;
            }
          }
        }
      }
    }
    if (!WRITE) {
      if constexpr (BUILD_S) {
        // publish the chunk's masks (one coalesced 128-byte row per query)
        __syncwarp();
        for (int b = 0; b < 32; ++b) sc.S[sbase + b * 32 + lane] = S[b * kSStride + lane];
        const unsigned ids = __reduce_add_sync(TH_FULL, nbits);
        if (lane == 0) sc.meta[(size_t)(c0 / kChunkRows) * W + j] = make_uint2(touched, ids);
        __syncwarp();
      }
      continue;
    }
    __syncwarp();
    // ---- WRITE.  Query by query, lane t extracts tile t's rows into a
    // staging run stored coalesced.  Sparse chunks of small graphs (a few
    // ids per query): every lane writes its own query's ids directly.
    const unsigned ids = __reduce_add_sync(TH_FULL, nbits);
    if (!RING && ids < kCoopIdsPerQuery * (unsigned)__popc(touched)) {
      if (q < src.nq) {
        for (int t = 0; t < 32; ++t) {
          uint32_t m = LOAD_S ? sc.S[sbase + lane * 32 + t] : S[lane * kSStride + t];
          const int64_t rb = c0 + 32 * t;
          while (m) {
            if (pos < cap) out[pos] = src.id(rb + __ffs(m) - 1);
            ++pos;
            m &= m - 1u;
          }
        }
      }
      __syncwarp();
      continue;
    }
    // entity layers without a row map stage final ids (the copy-out is then
    // a plain move); otherwise chunk-relative positions resolved on the way out
    const bool direct = !Src::kRing && Src::kDense && src.map == nullptr;
    const int32_t rbase = direct ? (int32_t)(c0 + 32 * lane) : 32 * lane;
    unsigned todo = touched;
    // the next query's masks are loaded while the current one is written
    int nb_ = todo ? __ffs(todo) - 1 : 0;
    uint32_t m_next = 0u;
    if (todo) m_next = LOAD_S ? sc.S[sbase + nb_ * 32 + lane] : S[nb_ * kSStride + lane];
    while (todo) {
      const int b = nb_;
      uint32_t m = m_next;
      todo &= todo - 1u;
      if (todo) {
        nb_ = __ffs(todo) - 1;
        m_next = LOAD_S ? sc.S[sbase + nb_ * 32 + lane] : S[nb_ * kSStride + lane];
      }
      const int c = __popc(m);
      const int incl = warp_incl_scan(c);
      const int n = __shfl_sync(TH_FULL, incl, 31);
      // highest set bit first, filling the lane's run from its end (FLO
      // gives the top bit directly; no bit reversal per id)
      StgT* dst = stg + incl - 1;
      while (m) {
        const int bit = 31 - __clz((int)m);
        *dst-- = (StgT)(rbase + bit);
        m ^= 1u << bit;
      }
      __syncwarp();
      const int64_t pb = __shfl_sync(TH_FULL, pos, b);
      if (direct && pb + n <= cap) {
        int32_t* o = out + pb + lane;
        const StgT* sp = stg + lane;
        int i = lane;
        for (; i + 96 < n; i += 128, o += 128, sp += 128) {
          const int32_t v0 = sp[0], v1 = sp[32], v2 = sp[64], v3 = sp[96];
          o[0] = v0;
          o[32] = v1;
          o[64] = v2;
          o[96] = v3;
        }
        for (; i < n; i += 32, o += 32, sp += 32) *o = *sp;
      } else if (direct) {
        for (int i = lane; i < n; i += 32)
          if (pb + i < cap) out[pb + i] = stg[i];
      } else if (pb + n <= cap) {
        // ids resolve through the row list / map: four independent
        // lookups in flight per lane before their stores
        int32_t* o = out + pb + lane;
        const StgT* sp = stg + lane;
        int i = lane;
        for (; i + 96 < n; i += 128, o += 128, sp += 128) {
          const int32_t v0 = src.id(c0 + sp[0]), v1 = src.id(c0 + sp[32]);
          const int32_t v2 = src.id(c0 + sp[64]), v3 = src.id(c0 + sp[96]);
          o[0] = v0;
          o[32] = v1;
          o[64] = v2;
          o[96] = v3;
        }
        for (; i < n; i += 32, o += 32, sp += 32) *o = src.id(c0 + *sp);
      } else {
        for (int i = lane; i < n; i += 32)
          if (pb + i < cap) out[pb + i] = src.id(c0 + stg[i]);
      }
      if (lane == b) pos += n;
      __syncwarp();
    }
  }
  if (!WRITE) {
    __syncwarp();
    total += (int32_t)cnt[lane];
    if (EDGES) {
      esum += ecnt[lane];
#pragma unroll
      for (int k = 0; k < 8; ++k) esum += (unsigned long long)eplane_cnt[k] << k;
    }
    if (q < src.nq) {
      counts[(size_t)q * nblk + blk] = total;
      if (EDGES && esum) atomicAdd(reinterpret_cast<unsigned long long*>(es.out + q), esum);
    }
  }
}

template <int W, class Src, bool WRITE, bool EDGES = false, int CACHE = 0>
__global__ void __launch_bounds__(32 * kMatWordsPerCta) mat_kernel(Src src, int nblk,
                                                                   int32_t* counts,
                                                                   const int64_t* base, int32_t* out,
                                                                   int64_t cap, EdgeSum es = {},
                                                                   SCache sc = {},
                                                                   const int64_t* bucket_total = nullptr) {
  // (a list layer small enough for the bucketed passes is written by them)
  if (bucket_total && *bucket_total <= kBucketMaxIds) return;
  constexpr int NW = mat_warps<W>();
  constexpr int NG = W / NW;  // word groups
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if constexpr (WRITE && CACHE == 2) {
    // cached write pass: warps are independent (no shared row sectors), so
    // each takes (block, word) units from a counter until none are left --
    // no wave-quantisation tail, dense and sparse units balance out
    const int units = nblk * W;
    for (;;) {
      int u = 0;
      if (lane == 0) u = (int)atomicAdd(sc.work, 1u);
      u = __shfl_sync(TH_FULL, u, 0);
      if (u >= units) return;
      mat_unit<W, Src, WRITE, EDGES, CACHE>(src, nblk, counts, base, out, cap, es, sc, u / W, u % W,
                                            warp, lane);
      __syncwarp();
    }
  } else {
    if (CACHE == 1 && blockIdx.x == 0 && threadIdx.x == 0) *sc.work = 0u;  // for the write pass
    mat_unit<W, Src, WRITE, EDGES, CACHE>(src, nblk, counts, base, out, cap, es, sc,
                                          (int)blockIdx.x / NG, ((int)blockIdx.x % NG) * NW + warp,
                                          warp, lane);
  }
}
