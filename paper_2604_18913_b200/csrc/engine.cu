// Batched multi-source k-hop engine for sm_100a.
//
// Reference semantics (incidence.py:214-221 _expand, :268-316 run_hops) are
// evaluated for up to 1024 independent queries at once: every entity row of
// the state matrices holds one bit per query (W = words per row).
//
//   X  frontier being expanded   (X_{h-1} of SURVEY 8a)
//   N  next layer                (R_h for exact walks, F_h = R_h \ V_{h-1} otherwise)
//   V  visited                   (per-query `visited`, incidence.py:301-308)
//   S  seed rows (cumulative semantics reports V_h \ S, incidence.py:309-312)
//   M  relation mask matrix, row r = queries allowing relation r
//
// A hop either PUSHES from the compacted frontier list (warp-cooperative CSR
// row gathers, atomicOr test-and-set into V / N, warp-aggregated compaction of
// newly reached entities), or PULLS over the reverse CSR for every entity
// (OR of in-neighbour frontier rows, early exit once all queries have visited
// the entity).  The direction is chosen on the device from the frontier's
// out-edge total, the role played by _DENSE_FRACTION in the reference
// (incidence.py:29-31,45).  Results are turned into per-query sorted id lists
// by a bit-transpose materialisation (K4), giving exactly the canonical
// sorted/unique EntityVector / TripleVector form (incidence.py:83-91).
#include <algorithm>
#include <atomic>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "engine.cuh"
#include "hubcache.cuh"
#include "paths.cuh"

namespace th {

namespace {

// NVTX range over a host scope (a wave, a hop, a shard phase): profilers
// (nsys, ncu --nvtx) attribute the kernels launched inside it
struct NvtxRange {
  explicit NvtxRange(const char* fmt, int a = 0, int b = 0) {
    char name[64];
    std::snprintf(name, sizeof(name), fmt, a, b);
    nvtxRangePushA(name);
  }
  ~NvtxRange() { nvtxRangePop(); }
};

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int32_t kHeavyPush = 64;   // rows longer than this are split across warps
constexpr int32_t kPushChunk = 64;
constexpr int kMatBlocks = 4096;      // target materialisation blocks

__device__ __forceinline__ uint32_t valid_word(int j, int nq) {
  const int lo = 32 * j;
  if (lo + 32 <= nq) return TH_FULL;
  if (lo >= nq) return 0u;
  return (1u << (nq - lo)) - 1u;
}

struct WaveArgs {
  const int32_t* indptr;
  const int32_t* csr_obj;
  const uint16_t* csr_rel;
  const int32_t* rindptr;
  const int32_t* rsrc;
  const uint16_t* rrel;
  const int32_t* rdst;  // target row of each in-edge (~v: split row)
  const int32_t* item_v;
  const int32_t* item_lo;
  const int32_t* item_hi;
  int64_t n_items;
  const int32_t* n_items_dev;  // device item count (nullptr: n_items)
  int pull_only_dense;         // pull_kernel beside the two-phase pull: dense hops only
  int64_t E, T;
  uint32_t *X, *N, *V, *S, *Xf, *Nf, *Vf;
  const uint32_t* M;
  int32_t* lists;
  int32_t* heavy;
  int64_t* heavy_off;  // [heavy_len + 1] exclusive chunk prefix of the heavy rows
  Ctl* ctl;
  int nq, sem, h;
  int last_frontier;  // FRONTIER's last hop: nothing reads V afterwards
  int last_hop;       // no hop follows: the new layer's out-degree total (push cost) is unused
};

template <int W>
struct Grp {
  static __device__ __forceinline__ unsigned shift() { return (lane_id() / W) * W; }
  static __device__ __forceinline__ unsigned mask() {
    return W == 32 ? TH_FULL : (((1u << W) - 1u) << shift());
  }
  static __device__ __forceinline__ unsigned j() { return lane_id() % W; }
  static __device__ __forceinline__ uint32_t ballot(bool p) {
    const uint32_t b = __ballot_sync(mask(), p);
    return W == 32 ? b : (b >> shift()) & ((1u << W) - 1u);
  }
};

// ---------------------------------------------------------------- seeds

template <int W>
// (e_out: unfiltered |T_1(q)| = out-degree sum of q's distinct seeds,
// written per query, so hop 1 needs no edge-count pass)
__global__ void seed_init_kernel(WaveArgs a, const int32_t* __restrict__ qoff,
                                 const int32_t* __restrict__ seeds, int q0, int64_t* e_out) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int q = gw; q < a.nq; q += nw) {
    // (qoff == nullptr: singleton queries, query q is {seeds[q0 + q]})
    const int32_t lo = qoff ? qoff[q0 + q] : q0 + q, hi = qoff ? qoff[q0 + q + 1] : q0 + q + 1;
    const uint32_t qb = 1u << (q & 31);
    const int qw = q >> 5;
    unsigned long long dsum = 0ull;
    for (int32_t i0 = lo; i0 < hi; i0 += 32) {
      const int32_t i = i0 + lane;
      int32_t e = -1;
      bool fresh = false;
      if (i < hi) {
        e = seeds[i];
        if (e < 0 || e >= a.E) {
          a.ctl->err = 1;
          e = -1;
        }
      }
      if (e >= 0) {
        const size_t r = (size_t)e * W + qw;
        const uint32_t old = atomicOr(&a.X[r], qb);
        if (e_out && !(old & qb)) dsum += (unsigned long long)(a.indptr[e + 1] - a.indptr[e]);
        if (a.sem != TH_EXACT) atomicOr(&a.V[r], qb);
        if (a.sem == TH_CUMULATIVE) atomicOr(&a.S[r], qb);
        const uint32_t fb = 1u << (e & 31);
        fresh = !(atomicOr(&a.Xf[e >> 5], fb) & fb);
        if (fresh && a.sem != TH_EXACT) atomicOr(&a.Vf[e >> 5], fb);
      }
      const uint32_t d = fresh ? (uint32_t)(a.indptr[e + 1] - a.indptr[e]) : 0u;
      warp_append_all(fresh, e, d, a.lists, &a.ctl->list_len[0], a.E, &a.ctl->push_cost[0]);
    }
    if (e_out) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) dsum += __shfl_xor_sync(TH_FULL, dsum, o);
      if (lane == 0) e_out[q] = (int64_t)dsum;
    }
  }
}

// begin hop h: place list segment h, choose the direction
// pull hops skip the per-edge frontier test when over 1/dense_div of the
// in-edges come from the frontier (dense_div <= 0: never)
__global__ void begin_hop_kernel(Ctl* ctl, int h, int64_t T, double pull_divisor, int has_reverse,
                                 double dense_div = 0.0) {
  const int32_t prev = ctl->list_len[h - 1];
  ctl->list_off[h] = ctl->list_off[h - 1] + prev;
  ctl->list_len[h] = 0;
  ctl->push_cost[h] = 0;
  ctl->heavy_len = 0;
  int pull = 0;
  if (has_reverse) {
    if (pull_divisor < 0) pull = 1;
    else if (pull_divisor > 0) pull = (double)ctl->push_cost[h - 1] * pull_divisor > (double)T;
  }
  ctl->mode[h] = pull;
  // the frontier's out-degree sum is the number of in-edges it sources
  ctl->dense[h] = pull && dense_div > 0 && (double)ctl->push_cost[h - 1] * dense_div > (double)T;
  if (pull) ctl->pull_hops++;
  else ctl->push_hops++;
}

// ------------------------------------------------------ mark new entity

// test-and-set the next-layer flag of v; true when this lane set it first
__device__ __forceinline__ bool flag_next(const WaveArgs& a, int32_t v) {
  const uint32_t fb = 1u << (v & 31);
  const bool fresh = !(atomicOr(&a.Nf[v >> 5], fb) & fb);
  if (fresh && a.sem != TH_EXACT) atomicOr(&a.Vf[v >> 5], fb);
  return fresh;
}

// converged (all 32 lanes): append the lanes' freshly flagged entities to
// the hop's list segment and add their out-degrees to the push cost
__device__ __forceinline__ void append_next(const WaveArgs& a, bool fresh, int32_t v) {
  const uint32_t d = fresh ? (uint32_t)(a.indptr[v + 1] - a.indptr[v]) : 0u;
  warp_append_all(fresh, v, d, a.lists + a.ctl->list_off[a.h], &a.ctl->list_len[a.h], a.E,
                  &a.ctl->push_cost[a.h]);
}

// Buffered form of append_next for the hop kernels: a warp collects its
// newly reached entities in shared memory and stores them with one global
// atomic per >= kAppendRun entities; the push-cost sum stays in registers
// until the kernel ends.  At low degree (C4: 1.6 edges per entity) nearly
// every warp step reaches an entity, and two same-address atomics per step
// serialised in L2; runs of 32 still left the two-phase pull waiting on the
// list counter (13% of its stalls at C4 hop 3): runs of 128 took C4 k=2
// 1.17 -> 1.10 ms, k=3 9.3 -> 9.05 ms (512: no further gain).  All calls
// converged (all 32 lanes).
constexpr int kAppendRun = 128;

struct WarpAppender {
  int32_t* wbuf;  // [kAppendRun + 32] shared, this warp's
  int fill = 0;
  unsigned long long cost = 0ull;

  __device__ __forceinline__ void flush(const WaveArgs& a) {
    __syncwarp();
    int32_t base = 0;
    if (lane_id() == 0) base = atomicAdd(&a.ctl->list_len[a.h], fill);
    base = __shfl_sync(TH_FULL, base, 0);
    int32_t* list = a.lists + a.ctl->list_off[a.h];
    for (int i = (int)lane_id(); i < fill; i += 32)
      if (base + (int64_t)i < a.E) list[base + i] = wbuf[i];
    fill = 0;
    __syncwarp();
  }
  __device__ __forceinline__ void add(const WaveArgs& a, bool fresh, int32_t v) {
    const unsigned fm = __ballot_sync(TH_FULL, fresh);
    if (!fm) return;
    if (fresh) {
      wbuf[fill + __popc(fm & lanemask_lt())] = v;
      if (!a.last_hop) {  // (the next hop's direction reads it; the last has none)
        const uint32_t d = (uint32_t)(a.indptr[v + 1] - a.indptr[v]);
        cost += d > (1u << 26) ? (1u << 26) : d;
      }
    }
    fill += __popc(fm);
    if (fill >= kAppendRun) flush(a);
  }
  __device__ __forceinline__ void finish(const WaveArgs& a) {
    if (fill) flush(a);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) cost += __shfl_xor_sync(TH_FULL, cost, o);
    if (lane_id() == 0 && cost) atomicAdd(&a.ctl->push_cost[a.h], cost);
  }
};

// ------------------------------------------------------------ push hop

// visit the (edge, nonzero frontier word) pairs of CSR slots [lo, hi) of u
template <int W, bool FILTER, class Op>
__device__ __forceinline__ void row_pairs(const WaveArgs& a, int32_t u, int32_t lo, int32_t hi,
                                          Op& op) {
  const unsigned lane = lane_id();
  const uint32_t xw = lane < (unsigned)W ? a.X[(size_t)u * W + lane] : 0u;
  const unsigned nz = __ballot_sync(TH_FULL, xw != 0u);
  if (!nz || hi <= lo) return;
  const int nzw = __popc(nz);
  const int pairs = (hi - lo) * nzw;
  const int j1 = __ffs(nz) - 1;
  for (int p0 = 0; p0 < pairs; p0 += 32) {
    const int p = p0 + (int)lane;
    int e, j;
    if (nzw == 1) {
      e = p;
      j = j1;
    } else {
      e = p / nzw;
      j = select_bit(nz, p - e * nzw);
    }
    const uint32_t x = __shfl_sync(TH_FULL, xw, j & 31);
    bool fresh = false;
    int32_t v = 0;
    if (p < pairs) {
      const int32_t pos = lo + e;
      uint32_t w = x;
      if (FILTER) w &= a.M[(size_t)a.csr_rel[pos] * W + j];
      if (w) {
        v = a.csr_obj[pos];
        fresh = op(v, j, w);
      }
    }
    if constexpr (Op::kAppends) op.app.add(a, fresh, v);
  }
}

template <int W, int SEM>
struct PushOp {
  static constexpr bool kAppends = true;
  static constexpr bool kRowWise = false;
  const WaveArgs& a;
  WarpAppender app;
  // returns true when v entered the next layer's list through this lane
  __device__ __forceinline__ bool operator()(int32_t v, int j, uint32_t w) const {
    const size_t r = (size_t)v * W + j;
    if (SEM == TH_EXACT) {
      if (!(w & ~__ldcg(&a.N[r]))) return false;
      const uint32_t old = atomicOr(&a.N[r], w);
      return old == 0u && flag_next(a, v);
    }
    const uint32_t seen = __ldcg(&a.V[r]);
    if (!(w & ~seen)) return false;
    if (a.last_frontier) {
      // FRONTIER's last hop: V is not read afterwards, so dedupe on N and
      // leave V untouched (its rows of this layer then need no clearing)
      const uint32_t nb = w & ~seen;
      const uint32_t old = atomicOr(&a.N[r], nb);
      return old == 0u && flag_next(a, v);
    }
    const uint32_t old = atomicOr(&a.V[r], w);
    const uint32_t nb = w & ~old;
    if (!nb) return false;
    atomicOr(&a.N[r], nb);
    return flag_next(a, v);
  }
};

template <int W>
struct CountOp {
  static constexpr bool kAppends = false;
  static constexpr bool kRowWise = true;
  uint32_t* sc;
  // Filtered |T_h(q)| over CSR slots [lo, hi) of frontier row u: per nonzero
  // frontier word j, 32 edges at a time, lane i holds the passing queries of
  // edge i (x_j & M[rel_i]); a 32x32 bit transpose hands lane b the edges
  // query 32j+b keeps, so one popcount + one shared atomic per lane per 32
  // edges replaces one atomic per (query, edge).
  template <int W_>
  __device__ __forceinline__ void row(const WaveArgs& a, int32_t u, int32_t lo, int32_t hi) const {
    const unsigned lane = lane_id();
    const uint32_t xw = lane < (unsigned)W_ ? a.X[(size_t)u * W_ + lane] : 0u;
    unsigned nz = __ballot_sync(TH_FULL, xw != 0u);
    while (nz) {
      const int j = __ffs(nz) - 1;
      nz &= nz - 1u;
      const uint32_t x = __shfl_sync(TH_FULL, xw, j);
      if (__popc(x) <= 4) {
        // few queries in this word (seed rows, sparse frontiers): one
        // ballot per query bit instead of a 32x32 transpose per 32 edges
        uint32_t c0 = 0u, c1 = 0u, c2 = 0u, c3 = 0u;
        const int b0 = __ffs(x) - 1;
        const uint32_t x1 = x & (x - 1u);
        const int b1 = __ffs(x1) - 1;
        const uint32_t x2 = x1 & (x1 - 1u);
        const int b2 = __ffs(x2) - 1;
        const uint32_t x3 = x2 & (x2 - 1u);
        const int b3 = __ffs(x3) - 1;
        for (int32_t e0 = lo; e0 < hi; e0 += 32) {
          const int32_t e = e0 + (int32_t)lane;
          const uint32_t w = e < hi ? x & a.M[(size_t)a.csr_rel[e] * W_ + j] : 0u;
          c0 += __popc(__ballot_sync(TH_FULL, (w >> (b0 & 31)) & 1u));
          if (b1 >= 0) c1 += __popc(__ballot_sync(TH_FULL, (w >> b1) & 1u));
          if (b2 >= 0) c2 += __popc(__ballot_sync(TH_FULL, (w >> b2) & 1u));
          if (b3 >= 0) c3 += __popc(__ballot_sync(TH_FULL, (w >> b3) & 1u));
        }
        if (lane == 0) {
          if (c0) atomicAdd(&sc[32 * j + b0], c0);
          if (c1) atomicAdd(&sc[32 * j + b1], c1);
          if (c2) atomicAdd(&sc[32 * j + b2], c2);
          if (c3) atomicAdd(&sc[32 * j + b3], c3);
        }
        continue;
      }
      for (int32_t e0 = lo; e0 < hi; e0 += 32) {
        const int32_t e = e0 + (int32_t)lane;
        const uint32_t w = e < hi ? x & a.M[(size_t)a.csr_rel[e] * W_ + j] : 0u;
        if (!__any_sync(TH_FULL, w != 0u)) continue;
        const int c = __popc(transpose32(w));
        if (c) atomicAdd(&sc[32 * j + lane], (uint32_t)c);
      }
    }
  }
};

// warp per frontier entity; rows above kHeavyPush go to the heavy list
template <int W, bool FILTER, class Op>
__device__ void drive_light(const WaveArgs& a, int seg, Op& op, bool build_heavy) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int32_t n = a.ctl->list_len[seg];
  const int32_t* list = a.lists + a.ctl->list_off[seg];
  for (int32_t i = gw; i < n; i += nw) {
    const int32_t u = list[i];
    const int32_t lo = a.indptr[u], hi = a.indptr[u + 1];
    if (hi - lo > kHeavyPush) {
      if (build_heavy && lane_id() == 0) a.heavy[atomicAdd(&a.ctl->heavy_len, 1)] = u;
      continue;
    }
    if constexpr (Op::kRowWise) op.template row<W>(a, u, lo, hi);
    else row_pairs<W, FILTER>(a, u, lo, hi, op);
  }
}

constexpr int32_t kSmallHeavy = 64;  // every warp walks a list this short (O(list) per warp)

// walk a short heavy list: every warp visits every row, taking the chunks
// of a global round-robin numbering
template <int W, bool FILTER, class Op>
__device__ void drive_heavy_short(const WaveArgs& a, Op& op, int32_t nh, int gw, int nw) {
  int64_t base = 0;
  for (int32_t i = 0; i < nh; ++i) {
    const int32_t u = a.heavy[i];
    const int32_t lo = a.indptr[u], hi = a.indptr[u + 1];
    const int32_t nc = (hi - lo + kPushChunk - 1) / kPushChunk;
    for (int64_t c = ((gw - base) % nw + nw) % nw; c < nc; c += nw) {
      const int32_t clo = lo + (int32_t)c * kPushChunk;
      if constexpr (Op::kRowWise) op.template row<W>(a, u, clo, min(hi, clo + kPushChunk));
      else row_pairs<W, FILTER>(a, u, clo, min(hi, clo + kPushChunk), op);
    }
    base += nc;
  }
}

// single block: exclusive prefix of the heavy rows' chunk counts, so the
// heavy kernels can map a global chunk index to its row by binary search
// (push_hop >= 0: skipped when that hop pulls)
__global__ void heavy_scan_kernel(const int32_t* __restrict__ indptr, const int32_t* __restrict__ heavy,
                                  const Ctl* ctl, int64_t* off, int push_hop) {
  __shared__ int64_t ws[32];
  if (push_hop >= 0 && ctl->mode[push_hop] != 0) return;
  if (ctl->heavy_len <= kSmallHeavy) return;  // drive_heavy walks short lists directly
  const int32_t nh = ctl->heavy_len;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  int64_t carry = 0;
  for (int32_t i0 = 0; i0 < nh; i0 += blockDim.x) {
    const int32_t i = i0 + threadIdx.x;
    int64_t v = 0;
    if (i < nh) {
      const int32_t u = heavy[i];
      v = (indptr[u + 1] - indptr[u] + kPushChunk - 1) / kPushChunk;
    }
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(TH_FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int64_t w = lane < nwarp ? ws[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(TH_FULL, w, o);
        if (lane >= o) w += y;
      }
      ws[lane] = w;
    }
    __syncthreads();
    if (i < nh) off[i] = carry + (warp ? ws[warp - 1] : 0) + x - v;
    carry += ws[nwarp - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) off[nh] = carry;
}

// all warps split the heavy rows into kPushChunk-slot chunks: a global chunk
// index maps to (row, chunk) through the prefix (binary search), so each
// warp only visits its own chunks
template <int W, bool FILTER, class Op>
__device__ void drive_heavy(const WaveArgs& a, Op& op) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int32_t nh = a.ctl->heavy_len;
  if (nh == 0) return;
  if (nh <= kSmallHeavy) {
    drive_heavy_short<W, FILTER>(a, op, nh, gw, nw);
    return;
  }
  const int64_t total = a.heavy_off[nh];
  for (int64_t g = gw; g < total; g += nw) {
    int32_t lo_i = 0, hi_i = nh - 1;  // last i with heavy_off[i] <= g
    while (lo_i < hi_i) {
      const int32_t mid = (lo_i + hi_i + 1) >> 1;
      if (a.heavy_off[mid] <= g) lo_i = mid;
      else hi_i = mid - 1;
    }
    const int32_t u = a.heavy[lo_i];
    const int32_t lo = a.indptr[u], hi = a.indptr[u + 1];
    const int32_t clo = lo + (int32_t)(g - a.heavy_off[lo_i]) * kPushChunk;
    if constexpr (Op::kRowWise) op.template row<W>(a, u, clo, min(hi, clo + kPushChunk));
    else row_pairs<W, FILTER>(a, u, clo, min(hi, clo + kPushChunk), op);
  }
}

template <int W, int SEM, bool FILTER>
__global__ void __launch_bounds__(kThreads) push_light_kernel(WaveArgs a) {
  if (a.ctl->mode[a.h] != 0) return;
  __shared__ int32_t abuf[kThreads / 32][kAppendRun + 32];
  PushOp<W, SEM> op{a, WarpAppender{abuf[threadIdx.x >> 5]}};
  // with a relation filter the edge-count pass already built the heavy list
  drive_light<W, FILTER>(a, a.h - 1, op, !FILTER);
  op.app.finish(a);
}

template <int W, int SEM, bool FILTER>
__global__ void __launch_bounds__(kThreads) push_heavy_kernel(WaveArgs a) {
  if (a.ctl->mode[a.h] != 0) return;
  __shared__ int32_t abuf[kThreads / 32][kAppendRun + 32];
  PushOp<W, SEM> op{a, WarpAppender{abuf[threadIdx.x >> 5]}};
  drive_heavy<W, FILTER>(a, op);
  op.app.finish(a);
}

// --------------------------------------------------------- edge counts

// |T_h(q)| = sum of out-degrees of X_{h-1}(q) (no relation filter)
template <int W>
__global__ void __launch_bounds__(kThreads) edge_count_kernel(WaveArgs a, int64_t* out) {
  __shared__ unsigned long long sc[32 * W];
  for (int t = threadIdx.x; t < 32 * W; t += blockDim.x) sc[t] = 0;
  __syncthreads();
  const int32_t n = a.ctl->list_len[a.h - 1];
  const int32_t* list = a.lists + a.ctl->list_off[a.h - 1];
  const int groups_per_warp = 32 / W;
  const int g = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * groups_per_warp + lane_id() / W;
  const int ng = ((gridDim.x * blockDim.x) >> 5) * groups_per_warp;
  const int j = lane_id() % W;
  for (int32_t i = g; i < n; i += ng) {
    const int32_t u = list[i];
    const unsigned long long d = (unsigned long long)(a.indptr[u + 1] - a.indptr[u]);
    if (!d) continue;
    uint32_t x = a.X[(size_t)u * W + j];
    while (x) {
      atomicAdd(&sc[32 * j + __ffs(x) - 1], d);
      x &= x - 1u;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 32 * W && t < a.nq; t += blockDim.x)
    if (sc[t]) atomicAdd((unsigned long long*)&out[t], sc[t]);
}

// filtered: one count per (query, passing edge)
template <int W>
__global__ void __launch_bounds__(kThreads) edge_count_filtered_kernel(WaveArgs a, int64_t* out,
                                                                       int heavy_pass) {
  __shared__ uint32_t sc[32 * W];
  for (int t = threadIdx.x; t < 32 * W; t += blockDim.x) sc[t] = 0;
  __syncthreads();
  CountOp<W> op{sc};
  if (heavy_pass) drive_heavy<W, true>(a, op);
  else drive_light<W, true>(a, a.h - 1, op, true);
  __syncthreads();
  for (int t = threadIdx.x; t < 32 * W && t < a.nq; t += blockDim.x)
    if (sc[t]) atomicAdd((unsigned long long*)&out[t], (unsigned long long)sc[t]);
}

#include "k3_pull.cuh"

// ------------------------------------------------------------- clearing

// zero rows listed in list segments [s0, s1] of matrix A (nrows rows); when
// the segments cover more than half of the rows, one streaming memset of the
// whole matrix is cheaper than the row gathers
template <int W>
__global__ void clear_rows_kernel(uint32_t* A, const int32_t* lists, const Ctl* ctl, int s0, int s1,
                                  int64_t nrows) {
  const int64_t lo = ctl->list_off[s0];
  const int64_t hi = ctl->list_off[s1] + ctl->list_len[s1];
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if ((hi - lo) * 2 > nrows) {
    if constexpr (W % 4 == 0) {
      uint4* p = reinterpret_cast<uint4*>(A);
      const int64_t n = nrows * (W / 4);
      for (int64_t i = t0; i < n; i += stride) p[i] = make_uint4(0u, 0u, 0u, 0u);
    } else {
      const int64_t n = nrows * W;
      for (int64_t i = t0; i < n; i += stride) A[i] = 0u;
    }
    return;
  }
  if constexpr (W % 4 == 0) {
    constexpr int Q = W / 4;  // 16-byte stores per row
    const int64_t n = (hi - lo) * Q;
    for (int64_t i = t0; i < n; i += stride) {
      const int32_t u = lists[lo + i / Q];
      reinterpret_cast<uint4*>(A + (size_t)u * W)[i % Q] = make_uint4(0u, 0u, 0u, 0u);
    }
  } else {
    const int64_t n = (hi - lo) * W;
    for (int64_t i = t0; i < n; i += stride) {
      const int32_t u = lists[lo + i / W];
      A[(size_t)u * W + (i % W)] = 0u;
    }
  }
}

// M[r][j] bit b = query 32j+b allows relation r
template <int W>
__global__ void build_mask_kernel(const uint32_t* __restrict__ masks, int mask_words, int q0,
                                  int nq, int64_t R, uint32_t* M) {
  const int64_t n = R * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / W;
    const int j = (int)(i % W);
    uint32_t word = 0;
    for (int b = 0; b < 32; ++b) {
      const int q = 32 * j + b;
      if (q >= nq) break;
      word |= ((masks[(size_t)(q0 + q) * mask_words + (r >> 5)] >> (r & 31)) & 1u) << b;
    }
    M[i] = word;
  }
}

// ------------------------------------------------------ materialisation

#include "k4_materialize.cuh"
#include "k4_rowmajor.cuh"

// one block per query: exclusive scan over its block counts; totals[q]
__global__ void mat_scan_rows_kernel(int32_t* counts, int nblk, int64_t* totals) {
  __shared__ int32_t ws[32];
  int32_t* c = counts + (size_t)blockIdx.x * nblk;
  int32_t carry = 0;
  for (int b0 = 0; b0 < nblk; b0 += blockDim.x) {
    const int i = b0 + threadIdx.x;
    const int32_t v = i < nblk ? c[i] : 0;
    int32_t x = v;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(TH_FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int32_t w = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(TH_FULL, w, o);
        if (lane >= o) w += y;
      }
      ws[lane] = w;
    }
    __syncthreads();
    const int32_t ex = carry + (warp ? ws[warp - 1] : 0) + x - v;
    if (i < nblk) c[i] = ex;
    carry += ws[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

// single block: per-query output offsets from the running cursor
__global__ void mat_scan_queries_kernel(const int64_t* totals, int nq, int64_t* off, int64_t* len,
                                        int64_t* cursor, int64_t* layer_total = nullptr) {
  __shared__ int64_t ws[32];
  const int q = threadIdx.x;
  const int64_t v = q < nq ? totals[q] : 0;
  int64_t x = v;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(TH_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(TH_FULL, w, o);
      if (lane >= o) w += y;
    }
    ws[lane] = w;
  }
  __syncthreads();
  // reserve this layer's output range atomically: consecutive layers' K4s
  // run on two streams and take their ranges from the same cursor
  __shared__ int64_t base_s;
  if (q == 0) {
    base_s = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(cursor),
                                (unsigned long long)ws[(blockDim.x >> 5) - 1]);
    if (layer_total) *layer_total = ws[(blockDim.x >> 5) - 1];
  }
  __syncthreads();
  const int64_t base = base_s;
  const int64_t ex = (warp ? ws[warp - 1] : 0) + x - v;
  if (q < nq) {
    off[q] = base + ex;
    len[q] = v;
  }
}

// ---------------------------------------------- flag bitmap -> row list

// Ascending list of the set bits of a flag bitmap (rows reached by a layer):
// per-block popcounts, one exclusive scan, then an ordered write.  Feeds K4's
// ListSrc so materialisation work follows the reached rows, not E.
constexpr int kCompactThreads = 256;
constexpr int kCompactPerThread = 8;
constexpr int kCompactWords = kCompactThreads * kCompactPerThread;

__device__ __forceinline__ int block_excl_scan(int v, int* ws, int* total) {
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
    int w = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(TH_FULL, w, o);
      if (lane >= o) w += y;
    }
    ws[lane] = w;
  }
  __syncthreads();
  const int ex = (warp ? ws[warp - 1] : 0) + x - v;
  *total = ws[(blockDim.x >> 5) - 1];
  __syncthreads();
  return ex;
}

// flag word w restricted to bits below nbits
__device__ __forceinline__ uint32_t flag_word(const uint32_t* flags, int64_t w, int64_t nbits) {
  if (w * 32 >= nbits) return 0u;
  const uint32_t f = flags[w];
  const int64_t left = nbits - w * 32;
  return left >= 32 ? f : f & ((1u << left) - 1u);
}

__global__ void __launch_bounds__(kCompactThreads) flag_count_kernel(const uint32_t* __restrict__ flags,
                                                                      int64_t nbits, int32_t* bcount) {
  __shared__ int ws[32];
  const int64_t w0 = (int64_t)blockIdx.x * kCompactWords + threadIdx.x * kCompactPerThread;
  int c = 0;
#pragma unroll
  for (int i = 0; i < kCompactPerThread; ++i) c += __popc(flag_word(flags, w0 + i, nbits));
  int total;
  block_excl_scan(c, ws, &total);
  if (threadIdx.x == 0) bcount[blockIdx.x] = total;
}

// single block: exclusive scan of the block counts in place; total -> *n_out
__global__ void flag_scan_kernel(int32_t* bcount, int nb, int32_t* n_out) {
  __shared__ int ws[32];
  int carry = 0;
  for (int b0 = 0; b0 < nb; b0 += blockDim.x) {
    const int i = b0 + threadIdx.x;
    const int v = i < nb ? bcount[i] : 0;
    int total;
    const int ex = block_excl_scan(v, ws, &total);
    if (i < nb) bcount[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) *n_out = carry;
}

__global__ void __launch_bounds__(kCompactThreads) flag_write_kernel(const uint32_t* __restrict__ flags,
                                                                      int64_t nbits,
                                                                      const int32_t* __restrict__ boff,
                                                                      int32_t* rows) {
  __shared__ int ws[32];
  const int64_t w0 = (int64_t)blockIdx.x * kCompactWords + threadIdx.x * kCompactPerThread;
  uint32_t f[kCompactPerThread];
  int c = 0;
#pragma unroll
  for (int i = 0; i < kCompactPerThread; ++i) {
    f[i] = flag_word(flags, w0 + i, nbits);
    c += __popc(f[i]);
  }
  int total;
  int o = boff[blockIdx.x] + block_excl_scan(c, ws, &total);
#pragma unroll
  for (int i = 0; i < kCompactPerThread; ++i) {
    uint32_t m = f[i];
    const int32_t base = (int32_t)((w0 + i) * 32);
    while (m) {
      rows[o++] = base + __ffs(m) - 1;
      m &= m - 1u;
    }
  }
}

// ---------------------------------------------------------------- host

template <typename T>
T* ensure(DBuf& b, int64_t n, cudaStream_t st) {
  const size_t need = (size_t)std::max<int64_t>(n, 1) * sizeof(T);
  if (b.bytes < need) {
    if (b.p) TH_CUDA(cudaFreeAsync(b.p, st));
    b.p = nullptr;
    TH_CUDA(cudaMallocAsync(&b.p, need, st));
    b.bytes = need;
  }
  return static_cast<T*>(b.p);
}

// Every device buffer a session's captured graph can reference; a change of
// any of their addresses or sizes invalidates that session's graph (and
// only that session's: other sessions' growth does not touch it).
template <class F>
void for_each_session_buf(Session* s, F&& f) {
  for (DBuf* d : {&s->X, &s->N, &s->V, &s->S, &s->Xf, &s->Nf, &s->Vf, &s->lists, &s->heavy,
                  &s->M, &s->counts, &s->totals, &s->ctl, &s->f_off, &s->f_len, &s->f_ids, &s->a_off,
                  &s->a_len, &s->a_ids, &s->edges, &s->p_off, &s->p_cnt, &s->p_trunc, &s->p_tids,
                  &s->p_scratch, &s->p_tmp, &s->rowlist, &s->rowscan, &s->k4_S, &s->k4_meta, &s->counts2,
                  &s->totals2, &s->rowlist2, &s->rowscan2, &s->k4_S2, &s->k4_meta2,
                  &s->k4_P, &s->k4_G, &s->k4_P2, &s->k4_G2, &s->heavy_off, &s->in_offs, &s->in_seeds, &s->in_masks,
                  &s->pull_items})
    f(d);
}

uint64_t session_alloc_sig(Session* s) {
  uint64_t h = 1469598103934665603ull;  // FNV-1a over (address, size) pairs
  for_each_session_buf(s, [&](DBuf* d) {
    for (uint64_t v : {(uint64_t)(uintptr_t)d->p, (uint64_t)d->bytes}) {
      h ^= v;
      h *= 1099511628211ull;
    }
  });
  return h;
}

unsigned persistent_grid() { return kNumSMs * 8; }

unsigned grid_for(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kThreads), kNumSMs * 16));
}

int pick_words(int nq) {
  int w = 1;
  while (32 * w < nq) w <<= 1;
  return w;
}

struct WaveBufs {
  int W;
  uint32_t *X, *N, *V, *S, *Xf, *Nf, *Vf, *M;
  int32_t *lists, *heavy, *counts, *counts2;
  int64_t *totals, *totals2;
  Ctl* ctl;
};

// count -> per-query scan -> offsets -> write, for any row source
template <int W, class Src>
void materialize(Session* s, WaveBufs& b, const Src& src, int nq, int64_t* off, int64_t* len,
                 int32_t* out, int64_t cap, int64_t* cursor, EdgeSum es = {}) {
  const int64_t rows = src.nrows;
  // scratch of the K4 slot in use (consecutive layers' K4s may run at once)
  int32_t* const counts = s->k4_slot ? b.counts2 : b.counts;
  int64_t* const totals = s->k4_slot ? b.totals2 : b.totals;
  DBuf& kS = s->k4_slot ? s->k4_S2 : s->k4_S;
  DBuf& kMeta = s->k4_slot ? s->k4_meta2 : s->k4_meta;
  if (rows == 0) {
    TH_CUDA(cudaMemsetAsync(len, 0, sizeof(int64_t) * nq, s->st));
    TH_CUDA(cudaMemsetAsync(off, 0, sizeof(int64_t) * nq, s->st));
    return;
  }
  constexpr int NW = mat_warps<W>();
  constexpr int NG = W / NW;
  constexpr size_t smem_w = mat_smem_bytes<W, true, Src::kRing>();
  // the attribute is per device: remember which devices have it (one mask
  // per template instantiation; an idempotent race at worst)
  static std::atomic<uint64_t> attr_devices{0};
  int dev = 0;
  TH_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(attr_devices.load(std::memory_order_relaxed) & bit)) {
    TH_CUDA(cudaFuncSetAttribute(mat_kernel<W, Src, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_w));
    attr_devices.fetch_or(bit, std::memory_order_relaxed);
  }
  // about twelve CTAs per SM in total (two waves of the write pass, six
  // resident CTAs per SM); blocks are whole 1024-row chunks
  const int64_t target = std::max<int64_t>(1, (int64_t)kNumSMs * 12 / NG);
  const int64_t blk_rows =
      std::max<int64_t>(kChunkRows, ceil_div(ceil_div(rows, target), kChunkRows) * kChunkRows);
  const int nblk = (int)ceil_div(rows, blk_rows);
  const unsigned grid = (unsigned)(nblk * NG);
  // small dense layers: the count pass caches the chunks' tile masks (one
  // layer-sized buffer, L2-resident at these sizes) for the write pass
  // (list-driven large layers re-read the layer instead: caching S there
  // streams a layer-sized buffer through HBM twice, C4 k=3 18.5 -> 20.9 ms)
  if constexpr (Src::kDense && !Src::kRing) {
    const int64_t nchunks = ceil_div(rows, kChunkRows);
    if (s->k4_cache && (es.out || !s->last.d_rel_masks || s->k4_cache_filtered) && s->k4_mode < 2 &&
        nchunks * W * 1024 * 4 <= (int64_t(256) << 20)) {
      SCache sc;
      sc.S = ensure<uint32_t>(kS, nchunks * W * 1024, s->st);
      sc.meta = ensure<uint2>(kMeta, nchunks * W + 1, s->st);
      sc.work = reinterpret_cast<unsigned*>(sc.meta + nchunks * W);
      constexpr size_t smem_cc = ((size_t)NW * (32 * kSStride + 64) + kEdgeWords) * sizeof(uint32_t);
      constexpr size_t smem_wc = (size_t)NW * mat_load_words<Src::kRing>() * sizeof(uint32_t);
      static std::atomic<uint64_t> attr_c{0};
      if (!(attr_c.load(std::memory_order_relaxed) & bit)) {
        TH_CUDA(cudaFuncSetAttribute(mat_kernel<W, Src, false, false, 1>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cc));
        TH_CUDA(cudaFuncSetAttribute(mat_kernel<W, Src, false, true, 1>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cc));
        TH_CUDA(cudaFuncSetAttribute(mat_kernel<W, Src, true, false, 2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_wc));
        attr_c.fetch_or(bit, std::memory_order_relaxed);
      }
      if (es.out)
        mat_kernel<W, Src, false, true, 1><<<grid, 32 * NW, smem_cc, s->st>>>(
            src, nblk, counts, nullptr, nullptr, 0, es, sc);
      else
        mat_kernel<W, Src, false, false, 1><<<grid, 32 * NW, smem_cc, s->st>>>(
            src, nblk, counts, nullptr, nullptr, 0, EdgeSum{}, sc);
      TH_LAUNCHED();
      // the write pass reads only the cached masks: the layer itself is free
      // (callers may clear it) once the count pass is done
      if (s->mark_counted) {
        TH_CUDA(cudaEventRecord(s->mark_counted, s->st));
        s->counted_recorded = true;
      }
      mat_scan_rows_kernel<<<nq, 256, 0, s->st>>>(counts, nblk, totals);
      TH_LAUNCHED();
      mat_scan_queries_kernel<<<1, kMaxWave, 0, s->st>>>(totals, nq, off, len, cursor);
      TH_LAUNCHED();
      // (warps pull units from a counter: at most one resident wave of CTAs)
      const unsigned wgrid = std::min<unsigned>(grid, kNumSMs * (2048 / (32 * NW)));
      mat_kernel<W, Src, true, false, 2><<<wgrid, 32 * NW, smem_wc, s->st>>>(
          src, nblk, counts, off, out, cap, EdgeSum{}, sc);
      TH_LAUNCHED();
      s->launches += 4;
      return;
    }
  }
  constexpr size_t smem_c = mat_smem_bytes<W, false>();
  bool counted = false;
  uint32_t* gcount = nullptr;  // bucketed write pass: per-slice group counts
  RowMajorSrc<W> rsrc{};
  if constexpr (Src::kDense) {
    // (k4_mode 1: list-driven layers without edge counts -- those keep the
    // word-per-warp form: its shared degree planes beat per-bit degree sums,
    // C4 hop 2 0.47 vs 1.03 ms; k4_mode 2: every entity layer)
    if ((s->k4_mode == 1 && Src::kRing && !es.out) || s->k4_mode == 2) {
      // list-driven layers: whole-row loads, carry-save counting (k4_rowmajor.cuh)
      static std::atomic<uint64_t> attr_r{0};
      if (!(attr_r.load(std::memory_order_relaxed) & bit)) {
        TH_CUDA(cudaFuncSetAttribute(rs_count_kernel<W, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)rs_count_smem<true>()));
        TH_CUDA(cudaFuncSetAttribute(rs_count_kernel<W, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)rs_count_smem<false>()));
        attr_r.fetch_or(bit, std::memory_order_relaxed);
      }
      rsrc.A = src.A;
      rsrc.neg = src.neg;
      rsrc.nq = src.nq;
      if constexpr (Src::kRing) {
        rsrc.rows = src.rows;
        rsrc.n_dev = src.n_dev;
        if (s->k4_bucket && !es.out)
          gcount = ensure<uint32_t>(s->k4_slot ? s->k4_G2 : s->k4_G, ((int64_t)nblk * kRsWarps + 1) * 32,
                                    s->st);
      } else {
        rsrc.flags = src.flags;
        rsrc.n_host = src.nrows;
      }
      if (es.out)
        rs_count_kernel<W, true><<<nblk, 32 * kRsWarps, rs_count_smem<true>(), s->st>>>(rsrc, nblk,
                                                                                       counts, es);
      else
        rs_count_kernel<W, false><<<nblk, 32 * kRsWarps, rs_count_smem<false>(), s->st>>>(
            rsrc, nblk, counts, es, gcount);
      TH_LAUNCHED();
      counted = true;
    }
  }
  if (!counted) {
    if (es.out)
      mat_kernel<W, Src, false, true><<<grid, 32 * NW, smem_c, s->st>>>(src, nblk, counts,
                                                                        nullptr, nullptr, 0, es);
    else
      mat_kernel<W, Src, false><<<grid, 32 * NW, smem_c, s->st>>>(src, nblk, counts, nullptr,
                                                                  nullptr, 0);
    TH_LAUNCHED();
  }
  mat_scan_rows_kernel<<<nq, 256, 0, s->st>>>(counts, nblk, totals);
  TH_LAUNCHED();
  mat_scan_queries_kernel<<<1, kMaxWave, 0, s->st>>>(totals, nq, off, len, cursor,
                                                    gcount ? totals + kMaxWave : nullptr);
  TH_LAUNCHED();
  if constexpr (Src::kRing) {
    if (gcount) {
      // (the layer's id total picks the pass on the device: the bucketed
      // passes below when their entry buffer stays L2-sized, else the
      // transposing write pass; the other side's kernels exit at once)
      const int64_t* ltot = totals + kMaxWave;
      // bucketed write: (row, bit) entries scattered into 32-query groups,
      // then gathered into each query's output (k4_rowmajor.cuh)
      uint32_t* P = ensure<uint32_t>(s->k4_slot ? s->k4_P2 : s->k4_P, kBucketMaxIds, s->st);
      bucket_scan_kernel<<<W, 1024, 0, s->st>>>(gcount, nblk * kRsWarps, ltot);
      TH_LAUNCHED();
      bucket_scatter_kernel<W><<<nblk, 32 * kRsWarps, 0, s->st>>>(rsrc, nblk, gcount, off, P, ltot);
      TH_LAUNCHED();
      // (the layer is free only after the write pass below, which re-reads
      // it when the bucketed passes stood aside)
      const int64_t units = (int64_t)nblk * W;
      bucket_gather_kernel<W><<<(unsigned)ceil_div(units, kThreads / 32), kThreads, 0, s->st>>>(
          src.rows, src.map, src.n_dev, nq, nblk, gcount, counts, off, P, out, cap, ltot);
      TH_LAUNCHED();
      mat_kernel<W, Src, true><<<grid, 32 * NW, smem_w, s->st>>>(src, nblk, counts, off, out, cap,
                                                                 EdgeSum{}, SCache{}, ltot);
      TH_LAUNCHED();
      s->launches += 7;
      return;
    }
  }
  mat_kernel<W, Src, true><<<grid, 32 * NW, smem_w, s->st>>>(src, nblk, counts, off, out,
                                                             cap);
  TH_LAUNCHED();
  s->launches += 4;
}

template <int W>
void materialize_dense(Session* s, WaveBufs& b, const uint32_t* A, const uint32_t* neg,
                       const uint32_t* flags, int nq, int64_t* off, int64_t* len, int32_t* out,
                       int64_t cap, int64_t* cursor, EdgeSum es = {}, bool prefer_list = false) {
  const int64_t E = s->mat_rows >= 0 ? s->mat_rows : s->g->E;
  if ((!prefer_list && E < s->list_min_entities) || E == 0) {
    DenseSrc<W> src{A, neg, flags, E, nq, s->row_map};
    materialize<W>(s, b, src, nq, off, len, out, cap, cursor, es);
    return;
  }
  const int64_t nwords = ceil_div(E, 32);
  const int nb = (int)ceil_div(nwords, kCompactWords);
  int32_t* rows = ensure<int32_t>(s->k4_slot ? s->rowlist2 : s->rowlist, E, s->st);
  int32_t* bsum = ensure<int32_t>(s->k4_slot ? s->rowscan2 : s->rowscan, nb, s->st);
  int32_t* n_dev = s->k4_slot ? &b.ctl->mat_rows2 : &b.ctl->mat_rows;
  flag_count_kernel<<<nb, kCompactThreads, 0, s->st>>>(flags, E, bsum);
  TH_LAUNCHED();
  flag_scan_kernel<<<1, 1024, 0, s->st>>>(bsum, nb, n_dev);
  TH_LAUNCHED();
  flag_write_kernel<<<nb, kCompactThreads, 0, s->st>>>(flags, E, bsum, rows);
  TH_LAUNCHED();
  s->launches += 3;
  ListSrc<W> src{A, neg, rows, n_dev, E, nq, s->row_map};
  materialize<W>(s, b, src, nq, off, len, out, cap, cursor, es);
}

template <int W>
void materialize_triples(Session* s, WaveBufs& b, int nq, int64_t* off, int64_t* len, int32_t* out,
                         int64_t cap, int64_t* cursor) {
  const Graph* g = s->g;
  TripleSrc<W> src{b.X, b.Xf, s->last.d_rel_masks ? b.M : nullptr, g->subj, g->rel, g->T, nq,
                   s->tid_map};
  materialize<W>(s, b, src, nq, off, len, out, cap, cursor);
}

// pull hops screen items per lane first on graphs of low mean in-degree
// per pull item (k3_pull.cuh; C4: ~2.3 in-edges per item, C2: ~10)
// (0 none, 1 per lane inside the pull kernel, 2 the two-phase screen +
// compacted pull)
int pull_screen_mode(const Graph* g, int knob = -1) {
  return knob >= 0 ? knob : (g->n_items > 0 && g->T < 4 * g->n_items) ? 2 : 0;
}

// one pull hop over graph g's items (the session's graph, or a shard's
// in-edge graph) with the session's screening mode
template <int W, int SEM, bool FILTER>
void launch_pull(Session* s, const Graph* g, const WaveArgs& a, cudaStream_t st) {
  const unsigned pg = persistent_grid();
  const int mode = pull_screen_mode(g, s->pull_screen);
  if (mode == 2) {
    // (frontier in-edges of a non-dense hop, <= T entries)
    const int64_t n = std::max<int64_t>(g->T, 1);
    int32_t* c = ensure<int32_t>(s->pull_items, (FILTER ? 3 : 2) * n, st);
    int32_t* cr = FILTER ? c + 2 * n : nullptr;
    WaveArgs ea = a;
    ea.rdst = g->rdst;
    ea.T = g->T;  // (a shard's in-edge graph: its own edge count)
    pull_screen_edges_kernel<FILTER><<<pg, kThreads, 0, st>>>(ea, c, c + n, cr);
    TH_LAUNCHED();
    if (s->pull_pair) pull_edges_kernel<W, SEM, FILTER, 2><<<pg, kThreads, 0, st>>>(a, c, c + n, cr);
    else pull_edges_kernel<W, SEM, FILTER, 1><<<pg, kThreads, 0, st>>>(a, c, c + n, cr);
    TH_LAUNCHED();
    WaveArgs pa = a;
    pa.pull_only_dense = 1;
    pull_kernel<W, SEM, FILTER, false><<<pg, kThreads, 0, st>>>(pa);  // dense hops
    TH_LAUNCHED();
    s->launches += 3;
    return;
  }
  if (mode == 1) pull_kernel<W, SEM, FILTER, true><<<pg, kThreads, 0, st>>>(a);
  else pull_kernel<W, SEM, FILTER, false><<<pg, kThreads, 0, st>>>(a);
  TH_LAUNCHED();
  s->launches += 1;
}

template <int W, int SEM, bool FILTER>
void expand_hop(Session* s, const WaveArgs& a) {
  const unsigned pg = persistent_grid();
  {
    ProfScope ps(s, TH_PROF_PUSH);
    push_light_kernel<W, SEM, FILTER><<<pg, kThreads, 0, s->st>>>(a);
    TH_LAUNCHED();
    heavy_scan_kernel<<<1, 1024, 0, s->st>>>(a.indptr, a.heavy, a.ctl, a.heavy_off, a.h);
    TH_LAUNCHED();
    push_heavy_kernel<W, SEM, FILTER><<<pg, kThreads, 0, s->st>>>(a);
    TH_LAUNCHED();
    s->launches += 3;
  }
  if (s->g->rindptr) {
    ProfScope ps(s, TH_PROF_PULL);
    launch_pull<W, SEM, FILTER>(s, s->g, a, s->st);
  }
}

// route a scope's launches to another stream of the session
struct StreamScope {
  Session* s;
  cudaStream_t saved;
  StreamScope(Session* s_, cudaStream_t to) : s(s_), saved(s_->st) { s->st = to; }
  ~StreamScope() { s->st = saved; }
};

void ensure_side_stream(Session* s) {
  if (s->side) return;
  int least = 0, greatest = 0;
  TH_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  TH_CUDA(cudaStreamCreateWithPriority(&s->side, cudaStreamNonBlocking, least));
  TH_CUDA(cudaStreamCreateWithPriority(&s->side2, cudaStreamNonBlocking, least));
  for (int i = 0; i < kMaxK + 2; ++i) {
    TH_CUDA(cudaEventCreateWithFlags(&s->ev_expand[i], cudaEventDisableTiming));
    TH_CUDA(cudaEventCreateWithFlags(&s->ev_mat[i], cudaEventDisableTiming));
    TH_CUDA(cudaEventCreateWithFlags(&s->ev_cnt[i], cudaEventDisableTiming));
  }
}

template <int W>
void run_wave(Session* s, const th_query* q, int q0, int nq) {
  const Graph* g = s->g;
  cudaStream_t st = s->st;
  const int64_t E = g->E, k = q->k, B = q->n_queries;
  const int64_t rows = std::max<int64_t>(E, 1) * W;
  const int64_t fwords = ceil_div(std::max<int64_t>(E, 1), 32) + 1;
  const bool filter = q->d_rel_masks != nullptr;
  const int sem = q->semantics;
  WaveBufs b{};
  b.W = W;
  b.X = ensure<uint32_t>(s->X, rows, st);
  b.N = ensure<uint32_t>(s->N, rows, st);
  b.V = ensure<uint32_t>(s->V, rows, st);
  b.S = sem == TH_CUMULATIVE ? ensure<uint32_t>(s->S, rows, st) : nullptr;
  b.Xf = ensure<uint32_t>(s->Xf, fwords, st);
  b.Nf = ensure<uint32_t>(s->Nf, fwords, st);
  b.Vf = ensure<uint32_t>(s->Vf, fwords, st);
  b.lists = ensure<int32_t>(s->lists, (k + 1) * std::max<int64_t>(E, 1), st);
  b.heavy = ensure<int32_t>(s->heavy, std::max<int64_t>(E, 1), st);
  b.M = filter ? ensure<uint32_t>(s->M, std::max<int64_t>(g->R, 1) * W, st) : nullptr;
  b.counts = ensure<int32_t>(s->counts, (int64_t)kMaxWave * (kMatBlocks + 64), st);
  b.totals = ensure<int64_t>(s->totals, kMaxWave + 1, st);  // (+ the layer total)
  b.counts2 = ensure<int32_t>(s->counts2, (int64_t)kMaxWave * (kMatBlocks + 64), st);
  b.totals2 = ensure<int64_t>(s->totals2, kMaxWave + 1, st);
  b.ctl = static_cast<Ctl*>(s->ctl.p);
  TH_CUDA(cudaMemsetAsync(b.ctl, 0, offsetof(Ctl, err), st));
  TH_CUDA(cudaMemsetAsync(b.Xf, 0, fwords * 4, st));
  TH_CUDA(cudaMemsetAsync(b.Nf, 0, fwords * 4, st));
  TH_CUDA(cudaMemsetAsync(b.Vf, 0, fwords * 4, st));

  WaveArgs a{};
  a.indptr = g->indptr;
  a.csr_obj = g->csr_obj;
  a.csr_rel = g->csr_rel;
  a.rindptr = g->rindptr;
  a.rsrc = g->rsrc;
  a.rrel = g->rrel;
  a.item_v = g->item_v;
  a.item_lo = g->item_lo;
  a.item_hi = g->item_hi;
  a.n_items = g->n_items;
  a.E = E;
  a.T = g->T;
  a.X = b.X;
  a.N = b.N;
  a.V = b.V;
  a.S = b.S;
  a.Xf = b.Xf;
  a.Nf = b.Nf;
  a.Vf = b.Vf;
  a.M = b.M;
  a.lists = b.lists;
  a.heavy = b.heavy;
  a.heavy_off = ensure<int64_t>(s->heavy_off, std::max<int64_t>(E, 1) + 1, st);
  a.ctl = b.ctl;
  a.nq = nq;
  a.sem = sem;
  a.h = 0;

  {
    ProfScope ps(s, TH_PROF_SETUP);
    if (filter) {
      build_mask_kernel<W><<<grid_for(g->R * W), kThreads, 0, st>>>(q->d_rel_masks, q->mask_words,
                                                                     q0, nq, g->R, b.M);
      TH_LAUNCHED();
      s->launches += 1;
    }
    seed_init_kernel<W><<<grid_for((int64_t)nq * 32), kThreads, 0, st>>>(
        a, (q->flags & TH_SINGLETON_SEEDS) ? nullptr : q->d_seed_offsets,
                                                                         q->d_seeds, q0,
        filter ? nullptr : static_cast<int64_t*>(s->edges.p) + q0);
    TH_LAUNCHED();
    s->launches += 1;
  }

  int64_t* f_off = static_cast<int64_t*>(s->f_off.p);
  int64_t* f_len = static_cast<int64_t*>(s->f_len.p);
  int64_t* a_off = static_cast<int64_t*>(s->a_off.p);
  int64_t* a_len = static_cast<int64_t*>(s->a_len.p);
  int64_t* edges = static_cast<int64_t*>(s->edges.p);
  const bool want_f = q->flags & TH_WANT_FRONTIERS;
  const bool want_a = q->flags & TH_WANT_ACTIVATED;
  const bool paths_need_l0 = (q->flags & TH_WANT_PATHS) && !(q->flags & TH_SINGLETON_SEEDS);
  const unsigned pg = persistent_grid();
  const bool overlap = s->overlap && want_f && !want_a && !(q->flags & TH_WANT_PATHS) &&
                       sem != TH_CUMULATIVE;
  if (overlap) ensure_side_stream(s);

  int nplanes = 0;
  while (nplanes < 31 && (int64_t(1) << nplanes) <= g->max_out) ++nplanes;
  bool next_edges_done = !filter;  // hop 1's counts come from seed_init
  for (int h = 1; h <= k; ++h) {
    NvtxRange nvtx_hop("th hop %d (wave of %d)", h, nq);
    a.h = h;
    a.last_frontier = h == k && sem == TH_FRONTIER;
    a.last_hop = h == k;
    const bool edges_done = next_edges_done;
    next_edges_done = false;
    {
      ProfScope ps(s, TH_PROF_SETUP);
      begin_hop_kernel<<<1, 1, 0, st>>>(b.ctl, h, g->T, s->pull_divisor, g->rindptr != nullptr,
                                        s->dense_pull);
      TH_LAUNCHED();
      s->launches += 1;
    }
    if (!edges_done) {
      ProfScope ps(s, TH_PROF_EDGES);
      int64_t* e_out = edges + (h - 1) * B + q0;
      if (filter) {
        edge_count_filtered_kernel<W><<<pg, kThreads, 0, st>>>(a, e_out, 0);
        TH_LAUNCHED();
        heavy_scan_kernel<<<1, 1024, 0, st>>>(a.indptr, a.heavy, a.ctl, a.heavy_off, -1);
        TH_LAUNCHED();
        edge_count_filtered_kernel<W><<<pg, kThreads, 0, st>>>(a, e_out, 1);
        TH_LAUNCHED();
        s->launches += 3;
      } else {
        edge_count_kernel<W><<<pg, kThreads, 0, st>>>(a, e_out);
        TH_LAUNCHED();
        s->launches += 1;
      }
    }
    if (want_a || (paths_need_l0 && h == 1)) {
      ProfScope ps(s, TH_PROF_ACTIVATED);
      materialize_triples<W>(s, b, nq, a_off + (h - 1) * B + q0, a_len + (h - 1) * B + q0,
                             static_cast<int32_t*>(s->a_ids.p), s->a_cap, &b.ctl->act_used);
    }
    if (filter) {
      if (sem == TH_EXACT) expand_hop<W, TH_EXACT, true>(s, a);
      else expand_hop<W, TH_FRONTIER, true>(s, a);
    } else {
      if (sem == TH_EXACT) expand_hop<W, TH_EXACT, false>(s, a);
      else expand_hop<W, TH_FRONTIER, false>(s, a);
    }
    if (want_f) {
      // consecutive layers alternate between two side streams with their
      // own K4 scratch, so layer h+1's K4 starts as soon as its expansion
      // ends instead of queueing behind layer h's
      const int slot = overlap ? (int)(h & 1) : 0;
      cudaStream_t kst = slot ? s->side2 : s->side;
      if (overlap) {
        TH_CUDA(cudaEventRecord(s->ev_expand[h], st));
        TH_CUDA(cudaStreamWaitEvent(kst, s->ev_expand[h], 0));
      }
      StreamScope sc(s, overlap ? kst : st);
      s->k4_slot = slot;
      s->mark_counted = overlap ? s->ev_cnt[h] : nullptr;
      s->counted_recorded = false;
      {
      // (the scope's end event must precede the join event below)
      ProfScope ps(s, TH_PROF_FRONTIER);
      if (sem == TH_CUMULATIVE)
        materialize_dense<W>(s, b, b.V, b.S, b.Vf, nq, f_off + (h - 1) * B + q0,
                             f_len + (h - 1) * B + q0, static_cast<int32_t*>(s->f_ids.p), s->f_cap,
                             &b.ctl->ids_used);
      else {
        // the layer just materialised is X_h, so its count pass also yields
        // |T_{h+1}| = sum of its out-degrees (unfiltered exact/frontier)
        EdgeSum es{};
        if (!filter && h < k) {
          es.indptr = g->indptr;
          es.nplanes = nplanes;
          es.out = edges + h * B + q0;
        }
        // the first layer is bounded by the seeds' out-degrees: when its K4
        // runs beside hop 2's expansion, follow its compacted row list (a
        // few busy CTAs) rather than scanning every chunk of E with a full
        // grid that takes SM slots from the expansion (C2 k=3 -5%; alone,
        // at k=1, the two cost the same)
        materialize_dense<W>(s, b, b.N, nullptr, b.Nf, nq, f_off + (h - 1) * B + q0,
                             f_len + (h - 1) * B + q0, static_cast<int32_t*>(s->f_ids.p), s->f_cap,
                             &b.ctl->ids_used, es, h == 1 && k > 1 && overlap && s->list_first_hop);
        next_edges_done = es.out != nullptr;
      }
      }
      if (overlap) {
        TH_CUDA(cudaEventRecord(s->ev_mat[h], kst));
        if (!s->counted_recorded) TH_CUDA(cudaEventRecord(s->ev_cnt[h], kst));
      }
      s->mark_counted = nullptr;
      s->k4_slot = 0;
    }
    {
      // retire X (rows of list segment h-1) and swap roles; with overlap the
      // layer's K4 (side stream) must be done reading it first
      if (overlap && h > 1) TH_CUDA(cudaStreamWaitEvent(st, s->ev_cnt[h - 1], 0));
      ProfScope ps(s, TH_PROF_CLEAR);
      clear_rows_kernel<W><<<grid_for(E * W), kThreads, 0, st>>>(b.X, b.lists, b.ctl, h - 1, h - 1, E);
      TH_LAUNCHED();
      TH_CUDA(cudaMemsetAsync(b.Xf, 0, fwords * 4, st));
      s->launches += 1;
    }
    std::swap(b.X, b.N);
    std::swap(b.Xf, b.Nf);
    std::swap(a.X, a.N);
    std::swap(a.Xf, a.Nf);
  }
  // leave every matrix zero for the next wave (V is not read by the
  // frontier K4, so its clear overlaps the last layer's materialisation)
  if (sem != TH_EXACT) {
    ProfScope ps(s, TH_PROF_CLEAR);
    // (FRONTIER's last hop never writes V: its layer's rows are clean)
    clear_rows_kernel<W><<<grid_for(E * W), kThreads, 0, st>>>(
        b.V, b.lists, b.ctl, 0, sem == TH_FRONTIER ? (int)k - 1 : (int)k, E);
    TH_LAUNCHED();
    s->launches += 1;
  }
  if (overlap) TH_CUDA(cudaStreamWaitEvent(st, s->ev_cnt[k], 0));
  {
    // (outside the scope above: the wait is not clearing time)
    ProfScope ps(s, TH_PROF_CLEAR);
    clear_rows_kernel<W><<<grid_for(E * W), kThreads, 0, st>>>(b.X, b.lists, b.ctl, (int)k, (int)k, E);
    TH_LAUNCHED();
    s->launches += 1;
  }
  if (overlap) {
    TH_CUDA(cudaStreamWaitEvent(st, s->ev_mat[k], 0));
    if (k > 1) TH_CUDA(cudaStreamWaitEvent(st, s->ev_mat[k - 1], 0));
  }
  ProfScope ps(s, TH_PROF_CLEAR);
  if (sem == TH_CUMULATIVE) {
    clear_rows_kernel<W><<<grid_for(E * W), kThreads, 0, st>>>(b.S, b.lists, b.ctl, 0, 0, E);
    TH_LAUNCHED();
    s->launches += 1;
  }
}


#include "k6_shard.cuh"

}  // namespace

ProfScope::ProfScope(Session* s_, int c) : s(s_), cat(c), l0(s_->launches) {
  if (!s->prof) return;
  tag = (s->side && s->st == s->side) ? 1 : (s->side2 && s->st == s->side2) ? 2 : 0;
  if (s->ev_used + 2 > s->ev_pool.size()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      TH_CUDA(cudaEventCreate(&e));
      s->ev_pool.push_back(e);
    }
  }
  // external: a captured record becomes a real event node of the graph
  TH_CUDA(cudaEventRecordWithFlags(s->ev_pool[s->ev_used], s->st,
                                   s->capturing ? cudaEventRecordExternal : cudaEventRecordDefault));
}

ProfScope::~ProfScope() noexcept(false) {
  static const bool debug_sync = std::getenv("TH_DEBUG_SYNC") != nullptr;
  if (debug_sync) {
    // diagnostics: serialise and name every kernel group as it completes
    static const char* names[] = {"setup", "edges", "activated", "push", "pull", "frontier",
                                  "clear", "paths"};
    std::fprintf(stderr, "[th] wait %s\n", names[cat]);
    TH_CUDA(cudaStreamSynchronize(s->st));
    std::fprintf(stderr, "[th] done %s\n", names[cat]);
  }
  if (!s->prof) return;
  TH_CUDA(cudaEventRecordWithFlags(s->ev_pool[s->ev_used + 1], s->st,
                                   s->capturing ? cudaEventRecordExternal : cudaEventRecordDefault));
  s->ev_used += 2;
  s->pending_cat.push_back(cat);
  s->pending_tag.push_back(tag);
  s->pending_launch.push_back(s->launches - l0);
}

static void drain_profile(Session* s) {
  if (!s->pending_cat.empty()) s->prof_trace.clear();
  for (size_t i = 0; i < s->pending_cat.size(); ++i) {
    float ms = 0.f, t0 = 0.f, t1 = 0.f;
    TH_CUDA(cudaEventElapsedTime(&ms, s->ev_pool[2 * i], s->ev_pool[2 * i + 1]));
    s->prof_ms[s->pending_cat[i]] += ms;
    s->prof_launches[s->pending_cat[i]] += s->pending_launch[i];
    // timeline relative to the run's first scope
    TH_CUDA(cudaEventElapsedTime(&t0, s->ev_pool[0], s->ev_pool[2 * i]));
    TH_CUDA(cudaEventElapsedTime(&t1, s->ev_pool[0], s->ev_pool[2 * i + 1]));
    const int tag = i < s->pending_tag.size() ? s->pending_tag[i] : 0;
    s->prof_trace.insert(s->prof_trace.end(), {(double)s->pending_cat[i], (double)tag, (double)t0, (double)t1});
  }
  s->pending_cat.clear();
  s->pending_tag.clear();
  s->pending_launch.clear();
  s->ev_used = 0;
}

int session_profile(Session* s, double* ms, int64_t* launches, int n) {
  TH_CUDA(cudaStreamSynchronize(s->st));
  drain_profile(s);
  for (int i = 0; i < n && i < TH_PROF_CATEGORIES; ++i) {
    if (ms) ms[i] = s->prof_ms[i];
    if (launches) launches[i] = s->prof_launches[i];
    s->prof_ms[i] = 0;
    s->prof_launches[i] = 0;
  }
  return TH_OK;
}

int64_t session_profile_trace(Session* s, double* out4, int64_t cap) {
  TH_CUDA(cudaStreamSynchronize(s->st));
  drain_profile(s);
  const int64_t n = (int64_t)s->prof_trace.size() / 4;
  if (out4 && cap >= n) std::copy(s->prof_trace.begin(), s->prof_trace.end(), out4);
  return n;
}

int session_wave_modes(Session* s, int32_t* modes, int n) {
  if (!s->ctl.p) return TH_ERR_STATE;
  TH_CUDA(cudaStreamSynchronize(s->st));
  Ctl c;
  TH_CUDA(cudaMemcpy(&c, s->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost));
  for (int i = 0; i < n && i < kMaxK + 2; ++i) modes[i] = i >= 1 && i <= s->last.k ? c.mode[i] : 0;
  return TH_OK;
}

int session_wave_lists(Session* s, int64_t* lens, int n) {
  if (!s->ctl.p) return TH_ERR_STATE;
  TH_CUDA(cudaStreamSynchronize(s->st));
  Ctl c;
  TH_CUDA(cudaMemcpy(&c, s->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost));
  for (int i = 0; i < n && i < kMaxK + 2; ++i) lens[i] = i <= s->last.k ? c.list_len[i] : 0;
  return TH_OK;
}

static int run_body(Session* s, const th_query* q);

// ---- CUDA-graph replay of repeated batch shapes ----
// A wave is ~30 short launches whose grids and arguments depend only on the
// query shape, the session buffers and the knobs (all control flow past the
// seeds lives on the device in Ctl).  A query repeating the previous run's
// key is captured once into a graph and replayed with one cudaGraphLaunch;
// its inputs are first copied into session-owned staging buffers so the
// graph's pointers stay valid.  Any (re)allocation of one of the session's
// buffers changes session_alloc_sig and invalidates its graph.
static bool graph_eligible(const Session* s, const th_query* q) {
  static const bool debug_sync = std::getenv("TH_DEBUG_SYNC") != nullptr;
  // profiling: event records are captured too, so a replay needs the
  // previous run's events drained (th_finish / th_session_profile)
  return s->use_graphs && !debug_sync && q->n_queries > 0 &&
         (q->flags & TH_SINGLETON_SEEDS) && s->mat_rows < 0 &&
         (!s->prof || (s->ev_used == 0 && s->pending_cat.empty()));
}

static GraphKey graph_key(Session* s, const th_query* q) {
  GraphKey k{};
  k.B = q->n_queries;
  k.k = q->k;
  k.semantics = q->semantics;
  k.flags = q->flags;
  k.mask_words = q->d_rel_masks ? q->mask_words : -1;
  k.max_paths = q->max_paths;
  k.f_cap = std::max<int64_t>({s->f_cap, s->last_f_need, 1 << 16});
  k.a_cap = std::max<int64_t>({s->a_cap, s->last_a_need, 1 << 16});
  k.p_cap = std::max<int64_t>({s->p_cap, s->last_p_need, 1 << 12});
  k.pull_divisor = s->pull_divisor;
  k.dense_pull = s->dense_pull;
  k.list_min = s->list_min_entities;
  k.knobs = (s->overlap ? 1 : 0) | (s->k4_cache ? 2 : 0) | (s->prof ? 4 : 0) | (s->k4_mode << 10) |
            ((s->pull_screen + 1) << 4) | (s->paths_k2 ? 64 : 0) | (s->priority ? 128 : 0) |
            (s->k4_bucket ? 256 : 0) | (s->pull_pair ? 512 : 0) |
            (s->k4_cache_filtered ? 1 << 20 : 0);
  k.epoch = session_alloc_sig(s);
  return k;
}

template <typename T>
static const T* stage(DBuf& b, const T* src, int64_t n, cudaStream_t st) {
  T* p = ensure<T>(b, n, st);
  if (n > 0) TH_CUDA(cudaMemcpyAsync(p, src, sizeof(T) * n, cudaMemcpyDeviceToDevice, st));
  return p;
}

static void drop_graph(Session* s) {
  if (s->gexec) cudaGraphExecDestroy(s->gexec);
  s->gexec = nullptr;
  s->g_valid = false;
}

static int run_graphed(Session* s, const th_query* q) {
  cudaStream_t st = s->st;
  const int64_t B = q->n_queries;
  th_query qs = *q;
  // stage inputs (seeds: one per query under TH_SINGLETON_SEEDS)
  qs.d_seed_offsets = stage(s->in_offs, q->d_seed_offsets, B + 1, st);
  qs.d_seeds = stage(s->in_seeds, q->d_seeds, B, st);
  if (q->d_rel_masks)
    qs.d_rel_masks = stage(s->in_masks, q->d_rel_masks, B * (int64_t)q->mask_words, st);
  const GraphKey key = graph_key(s, &qs);
  if (s->gexec && s->g_valid && key == s->gkey) {
    TH_CUDA(cudaGraphLaunch(s->gexec, st));
    s->launches += s->g_launches;
    if (s->prof) {
      s->pending_cat = s->g_pend_cat;
      s->pending_tag = s->g_pend_tag;
      s->pending_launch = s->g_pend_launch;
      s->ev_used = s->g_ev_used;
    }
    s->last = qs;
    s->has_run = true;
    return TH_OK;
  }
  if (!(s->g_seen && key == s->gkey)) {
    // first run of this shape: run eagerly (sizes every buffer), remember it
    drop_graph(s);
    const int rc = run_body(s, &qs);
    s->gkey = graph_key(s, &qs);
    s->g_seen = rc == TH_OK;
    return rc;
  }
  // second run of the same shape: capture, instantiate, launch
  drop_graph(s);
  const int64_t l0 = s->launches;
  cudaGraph_t graph = nullptr;
  // capture on a session-owned stream (the caller's may be the legacy
  // default stream, which cannot capture); nothing runs during capture, and
  // the graph is launched on the caller's stream
  if (!s->cap) {
    int least = 0, greatest = 0;
    TH_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    TH_CUDA(cudaStreamCreateWithPriority(&s->cap, cudaStreamNonBlocking, greatest));
  }
  TH_CUDA(cudaStreamBeginCapture(s->cap, cudaStreamCaptureModeThreadLocal));
  int rc = TH_OK;
  const char* fail = nullptr;
  cudaError_t fail_code = cudaSuccess;
  s->st = s->cap;
  s->capturing = true;
  try {
    rc = run_body(s, &qs);
  } catch (const CudaError& e) {
    fail = e.where;
    fail_code = e.code;
  }
  s->capturing = false;
  s->st = st;
  cudaError_t ce = cudaStreamEndCapture(s->cap, &graph);
  if (fail || rc != TH_OK || ce != cudaSuccess) {
    // capture is a pure optimisation: drop it and run this query eagerly
    if (graph) cudaGraphDestroy(graph);
    (void)cudaGetLastError();
    static const bool dbg = std::getenv("TH_GRAPH_DEBUG") != nullptr;
    if (dbg)
      std::fprintf(stderr, "[th] graph capture failed: %s: %s (end: %s)\n", fail ? fail : "rc",
                   cudaGetErrorString(fail_code), cudaGetErrorString(ce));
    s->g_seen = false;
    s->launches = l0;
    s->pending_cat.clear();
    s->pending_launch.clear();
    s->ev_used = 0;
    if (rc != TH_OK && !fail) return rc;
    s->g_failures += 1;
    if (s->g_failures >= 3) s->use_graphs = false;
    return run_body(s, &qs);
  }
  const uint64_t epoch = session_alloc_sig(s);
  cudaGraphExec_t exec = nullptr;
  // (node priorities: captured kernels carry their stream's priority)
  const cudaError_t ie =
      cudaGraphInstantiate(&exec, graph, s->priority ? cudaGraphInstantiateFlagUseNodePriority : 0);
  cudaGraphDestroy(graph);
  TH_CUDA(ie);
  s->gexec = exec;
  s->g_launches = s->launches - l0;
  s->g_pend_cat = s->pending_cat;
  s->g_pend_tag = s->pending_tag;
  s->g_pend_launch = s->pending_launch;
  s->g_ev_used = s->ev_used;
  s->launches = l0 + s->g_launches;
  s->gkey = key;
  // an allocation inside the capture would leave the graph pointing at
  // freed memory: never replay such a graph (sizes are stable on a repeat,
  // so this is a guard, not a path)
  s->g_valid = epoch == key.epoch;
  if (!s->g_valid) {
    drop_graph(s);
    s->g_seen = false;
    return run_body(s, &qs);
  }
  TH_CUDA(cudaGraphLaunch(s->gexec, st));
  return TH_OK;
}

int session_run(Session* s, const th_query* q) {
  const Graph* g = s->g;
  if (q->k < 1) {
    set_error("hop count must be >= 1");
    return TH_ERR_INVALID;
  }
  if (q->k > kMaxK) {
    set_error("hop count above the engine limit of " + std::to_string(kMaxK));
    return TH_ERR_INVALID;
  }
  if (q->semantics < TH_EXACT || q->semantics > TH_CUMULATIVE) {
    set_error("unknown hop semantics");
    return TH_ERR_INVALID;
  }
  if (q->n_queries < 0 || (q->n_queries > 0 && (!q->d_seed_offsets || !q->d_seeds))) {
    set_error("bad query arrays");
    return TH_ERR_INVALID;
  }
  if (q->d_rel_masks && q->mask_words < ceil_div(g->R, 32)) {
    set_error("mask_words too small for the relation count");
    return TH_ERR_INVALID;
  }
  if ((q->flags & TH_WANT_PATHS) && q->max_paths < -1) {
    set_error("max_paths must be >= 0");
    return TH_ERR_INVALID;
  }
  if (graph_eligible(s, q)) return run_graphed(s, q);
  return run_body(s, q);
}

static int run_body(Session* s, const th_query* q) {
  const Graph* g = s->g;
  cudaStream_t st = s->st;
  const int64_t B = q->n_queries, k = q->k;
  const int64_t kb = std::max<int64_t>(k * B, 1);
  ensure<Ctl>(s->ctl, 1, st);
  ensure<int64_t>(s->f_off, kb, st);
  ensure<int64_t>(s->f_len, kb, st);
  ensure<int64_t>(s->a_off, kb, st);
  ensure<int64_t>(s->a_len, kb, st);
  ensure<int64_t>(s->edges, kb, st);
  // output capacities grow to the last observed need (th_finish)
  s->f_cap = std::max<int64_t>({s->f_cap, s->last_f_need, 1 << 16});
  s->a_cap = std::max<int64_t>({s->a_cap, s->last_a_need, 1 << 16});
  ensure<int32_t>(s->f_ids, s->f_cap, st);
  ensure<int32_t>(s->a_ids, s->a_cap, st);
  TH_CUDA(cudaMemsetAsync(s->ctl.p, 0, sizeof(Ctl), st));
  TH_CUDA(cudaMemsetAsync(s->edges.p, 0, sizeof(int64_t) * kb, st));
  TH_CUDA(cudaMemsetAsync(s->f_len.p, 0, sizeof(int64_t) * kb, st));
  TH_CUDA(cudaMemsetAsync(s->f_off.p, 0, sizeof(int64_t) * kb, st));
  TH_CUDA(cudaMemsetAsync(s->a_len.p, 0, sizeof(int64_t) * kb, st));
  TH_CUDA(cudaMemsetAsync(s->a_off.p, 0, sizeof(int64_t) * kb, st));
  s->last = *q;
  s->has_run = true;

  const int wave = std::min<int64_t>(std::max<int64_t>(B, 1), kMaxWave);
  const int W = pick_words(wave);
  // matrices must start zero: (re)allocation leaves garbage, so clear on growth
  const int64_t rows = std::max<int64_t>(g->E, 1) * W;
  const size_t need = (size_t)rows * 4;
  for (DBuf* d : {&s->X, &s->N, &s->V, &s->S}) {
    if (d == &s->S && q->semantics != TH_CUMULATIVE) continue;
    if (d->bytes < need) {
      ensure<uint32_t>(*d, rows, st);
      TH_CUDA(cudaMemsetAsync(d->p, 0, d->bytes, st));
    }
  }
  for (int64_t q0 = 0; q0 < B; q0 += wave) {
    const int nq = (int)std::min<int64_t>(wave, B - q0);
    switch (W) {
      case 1: run_wave<1>(s, q, (int)q0, nq); break;
      case 2: run_wave<2>(s, q, (int)q0, nq); break;
      case 4: run_wave<4>(s, q, (int)q0, nq); break;
      case 8: run_wave<8>(s, q, (int)q0, nq); break;
      case 16: run_wave<16>(s, q, (int)q0, nq); break;
      default: run_wave<32>(s, q, (int)q0, nq); break;
    }
  }
  if (q->flags & TH_WANT_PATHS) {
    const Ctl* ctl = static_cast<const Ctl*>(s->ctl.p);
    PathArgs pa{};
    pa.indptr = g->indptr;
    pa.csr_tid = g->csr_tid;
    pa.csr_obj = g->csr_obj;
    pa.csr_rel = g->csr_rel;
    pa.t_obj = g->obj;
    pa.t_rel = g->rel;
    pa.qoff = q->d_seed_offsets;
    pa.seeds = q->d_seeds;
    pa.masks = q->d_rel_masks;
    pa.mask_words = q->mask_words;
    pa.l0_off = static_cast<const int64_t*>(s->a_off.p);
    pa.l0_len = static_cast<const int64_t*>(s->a_len.p);
    pa.l0_ids = static_cast<const int32_t*>(s->a_ids.p);
    pa.singleton = (q->flags & TH_SINGLETON_SEEDS) != 0;
    pa.B = (int32_t)B;
    pa.k = (int32_t)k;
    pa.E = g->E;
    pa.max_paths = q->max_paths;
    s->p_cap = std::max<int64_t>({s->p_cap, s->last_p_need, 1 << 12});
    pa.p_off = ensure<int64_t>(s->p_off, B + 1, st);
    pa.p_cnt = ensure<int64_t>(s->p_cnt, std::max<int64_t>(B, 1), st);
    pa.p_trunc = ensure<uint8_t>(s->p_trunc, std::max<int64_t>(B, 1), st);
    pa.p_tids = ensure<int32_t>(s->p_tids, s->p_cap * k, st);
    pa.scratch = ensure<int64_t>(s->p_scratch, scan_scratch_elems_i64(B + 1), st);
    pa.cap = s->p_cap;
    pa.used = const_cast<int64_t*>(&ctl->path_used);
    // capped queries whose slots fit 2 GiB take the single-DFS form
    if (q->max_paths > 0 && (int64_t)B * q->max_paths * k * 4 <= (int64_t(2) << 30))
      pa.tmp = ensure<int32_t>(s->p_tmp, (int64_t)B * q->max_paths * k, st);
    pa.k2_parallel = s->paths_k2;
    ProfScope ps(s, TH_PROF_PATHS);
    NvtxRange nvtx_paths("th paths (k=%d)", (int)k);
    s->launches += launch_paths(pa, st);
  }
  return TH_OK;
}

int session_finish(Session* s, th_result* out) {
  if (!s->has_run) {
    set_error("th_finish before th_run");
    return TH_ERR_STATE;
  }
  TH_CUDA(cudaStreamSynchronize(s->st));
  if (s->prof) drain_profile(s);
  Ctl c;
  TH_CUDA(cudaMemcpy(&c, s->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost));
  const th_query& q = s->last;
  std::memset(out, 0, sizeof(*out));
  out->n_queries = q.n_queries;
  out->k = q.k;
  out->frontier_off = static_cast<const int64_t*>(s->f_off.p);
  out->frontier_len = static_cast<const int64_t*>(s->f_len.p);
  out->frontier_ids = static_cast<const int32_t*>(s->f_ids.p);
  out->act_off = static_cast<const int64_t*>(s->a_off.p);
  out->act_len = static_cast<const int64_t*>(s->a_len.p);
  out->act_ids = static_cast<const int32_t*>(s->a_ids.p);
  out->edges = static_cast<const int64_t*>(s->edges.p);
  out->frontier_total = c.ids_used;
  out->act_total = c.act_used;
  out->push_hops = c.push_hops;
  out->pull_hops = c.pull_hops;
  if (q.flags & TH_WANT_PATHS) {
    out->path_off = static_cast<const int64_t*>(s->p_off.p);
    out->path_count = static_cast<const int64_t*>(s->p_cnt.p);
    out->path_truncated = static_cast<const uint8_t*>(s->p_trunc.p);
    out->path_tids = static_cast<const int32_t*>(s->p_tids.p);
    out->path_total = c.path_used;
  }
  if (c.err == 2) {
    set_error("malformed exchange record (row not owned by this rank)");
    return TH_ERR_STATE;
  }
  if (c.err) {
    set_error("seed id out of range for the graph's entity count");
    return TH_ERR_RANGE;
  }
  bool overflow = false;
  if (c.ids_used > s->f_cap) {
    s->last_f_need = c.ids_used + c.ids_used / 4;
    overflow = true;
  }
  if (c.act_used > s->a_cap) {
    s->last_a_need = c.act_used + c.act_used / 4;
    overflow = true;
  }
  if ((q.flags & TH_WANT_PATHS) && c.path_used > s->p_cap) {
    s->last_p_need = c.path_used + c.path_used / 4;
    overflow = true;
  }
  if (overflow) {
    set_error("result capacity exceeded; capacities grown, re-run the query");
    return TH_ERR_OVERFLOW;
  }
  return TH_OK;
}

void session_free(Session* s) {
  drop_graph(s);
  for_each_session_buf(s, [&](DBuf* d) {
    if (d->p) cudaFreeAsync(d->p, s->st);
    d->p = nullptr;
    d->bytes = 0;
  });
  cudaStreamSynchronize(s->st);
  for (cudaEvent_t e : s->ev_pool) cudaEventDestroy(e);
  s->ev_pool.clear();
  if (s->side) {
    cudaStreamSynchronize(s->side);
    for (int i = 0; i < kMaxK + 2; ++i) {
      cudaEventDestroy(s->ev_expand[i]);
      cudaEventDestroy(s->ev_mat[i]);
      cudaEventDestroy(s->ev_cnt[i]);
    }
    cudaStreamSynchronize(s->side2);
    cudaStreamDestroy(s->side);
    cudaStreamDestroy(s->side2);
    s->side = s->side2 = nullptr;
  }
  if (s->cap) {
    cudaStreamDestroy(s->cap);
    s->cap = nullptr;
  }
}

// partition.py:80-84 multiplicative hash; -1 for entities without out-edges
__global__ void plan_owner_hash_kernel(const int32_t* __restrict__ indptr, int64_t E, int32_t m,
                                       int32_t* owner) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const bool subject = indptr[e + 1] > indptr[e];
    const uint32_t h = (uint32_t)((uint64_t)e * 0x9E3779B1ull);
    owner[e] = subject ? (int32_t)(h % (uint32_t)m) : -1;
  }
}

void plan_owner_hash(const Graph* g, int32_t m, int32_t* d_owner, cudaStream_t st) {
  if (g->E == 0) return;
  plan_owner_hash_kernel<<<grid_for(g->E), kThreads, 0, st>>>(g->indptr, g->E, m, d_owner);
  TH_LAUNCHED();
}


// ============================================================ K6 shards
// One rank's partitioned-graph session (see k6_shard.cuh).  The host issues
// a wave hop by hop in three phases (send / receive / end) separated by a
// barrier across ranks; all data movement between ranks is peers writing
// into each other's exchange regions from the kernels, so the host never
// waits on a count or a collective inside a wave.

struct Shard {
  Graph g;                         // rows [0,n_local) owned, then hub slices
  int32_t* tid_l2g = nullptr;      // local triple -> global tid (ascending)
  int32_t* lidx = nullptr;         // [E] row at the owner
  int32_t* hub_index = nullptr;    // [E]
  int32_t* hub_ids = nullptr;      // [H]
  int32_t* l2g = nullptr;          // [n_local] owned rows -> global ids (ascending)
  int64_t E = 0, n_local = 0, H = 0, T_global = 0;
  int32_t rank = 0, world = 1;
  Session s;
  DBuf O, Of, olist;               // remote staging (world > 1)
  Graph gin;                       // in-edges of owned objects (pull hops)
  bool can_pull = false;
  double pull_divisor = 8.0;
  // exchange region (peers write into it) and the peers' regions
  uint8_t* xr = nullptr;
  size_t xr_bytes = 0;
  int64_t xcap = 0;                // inbox records
  size_t off_keys = 0, off_bits = 0, off_hubs = 0;
  std::vector<uint8_t*> peers;     // host copy of the peer bases ([world])
  std::vector<bool> peer_ipc;      // opened through cudaIpcOpenMemHandle
  uint8_t** d_peers = nullptr;     // device copy
  int W = 0;
  bool in_wave = false;
  int next_hop = 0, next_phase = 0;
  HubCache* hc = nullptr;          // K7: hub slices paged in on demand (hubcache.cuh)
  struct WaveGraph* group = nullptr;  // in-process worlds: the wave's CUDA graph (when members[0])
  bool retired = false;            // the wave's retire kernels are issued already (shards_run_wave)
  int64_t rows() const { return n_local + H; }
};

// A whole wave of an in-process world (every rank on one stream) as one
// CUDA graph: begin + every hop's phases of every shard, captured once per
// shape and replayed (inputs staged into session buffers first, as
// run_graphed does for single graphs).
struct WaveGraph {
  std::vector<Shard*> members;
  std::vector<GraphKey> keys;
  std::vector<uint64_t> sigs;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap = nullptr;
  bool seen = false, valid = false;
  int failures = 0;
  int64_t launches = 0;
};

namespace {

template <typename T>
T* dcopy(const T* src, int64_t n, cudaStream_t st) {
  T* p = nullptr;
  TH_CUDA(cudaMalloc(&p, sizeof(T) * std::max<int64_t>(n, 1)));
  if (n > 0) TH_CUDA(cudaMemcpyAsync(p, src, sizeof(T) * n, cudaMemcpyDeviceToDevice, st));
  return p;
}

// exchange region layout for an inbox of `cap` records and H hubs
void shard_layout(Shard* sh, int64_t cap) {
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  sh->xcap = cap;
  sh->off_keys = kXCtrlBytes;
  sh->off_bits = up(sh->off_keys + sizeof(uint64_t) * (size_t)cap);
  sh->off_hubs = up(sh->off_bits + sizeof(uint32_t) * (size_t)cap);
  sh->xr_bytes = up(sh->off_hubs + sizeof(uint32_t) * (size_t)std::max<int64_t>(sh->H, 1) * 32);
}

void shard_alloc_region(Shard* sh, int64_t cap, cudaStream_t st) {
  if (sh->xr) TH_CUDA(cudaFree(sh->xr));
  sh->xr = nullptr;
  shard_layout(sh, cap);
  TH_CUDA(cudaMalloc(&sh->xr, sh->xr_bytes));
  TH_CUDA(cudaMemsetAsync(sh->xr, 0, sh->xr_bytes, st));
  TH_CUDA(cudaStreamSynchronize(st));  // (peers may map it right away)
  sh->peers.assign(sh->world, nullptr);
  sh->peer_ipc.assign(sh->world, false);
  sh->peers[sh->rank] = sh->xr;
}

void shard_close_peers(Shard* sh) {
  for (int d = 0; d < (int)sh->peers.size(); ++d)
    if (sh->peer_ipc[d] && sh->peers[d]) cudaIpcCloseMemHandle(sh->peers[d]);
  for (int d = 0; d < (int)sh->peers.size(); ++d) {
    if (d != sh->rank) sh->peers[d] = nullptr;
    sh->peer_ipc[d] = false;
  }
}

bool shard_connected(const Shard* sh) {
  for (uint8_t* p : sh->peers)
    if (!p) return false;
  return !sh->peers.empty();
}

// the kernels' copy of the peer table, once every peer is known
void shard_publish_peers(Shard* sh) {
  if (sh->d_peers && shard_connected(sh))
    TH_CUDA(cudaMemcpy(sh->d_peers, sh->peers.data(), sizeof(uint8_t*) * sh->world,
                       cudaMemcpyHostToDevice));
}

template <int W>
ShardArgs shard_args(Shard* sh) {
  Session* s = &sh->s;
  const Graph* g = &sh->g;
  ShardArgs sa{};
  WaveArgs& a = sa.a;
  a.indptr = g->indptr;
  a.csr_obj = g->csr_obj;
  a.csr_rel = g->csr_rel;
  a.E = sh->rows();
  a.T = g->T;
  a.X = static_cast<uint32_t*>(s->X.p);
  a.N = static_cast<uint32_t*>(s->N.p);
  a.V = static_cast<uint32_t*>(s->V.p);
  a.S = static_cast<uint32_t*>(s->S.p);
  a.Xf = static_cast<uint32_t*>(s->Xf.p);
  a.Nf = static_cast<uint32_t*>(s->Nf.p);
  a.Vf = static_cast<uint32_t*>(s->Vf.p);
  a.M = s->last.d_rel_masks ? static_cast<uint32_t*>(s->M.p) : nullptr;
  a.lists = static_cast<int32_t*>(s->lists.p);
  a.heavy = static_cast<int32_t*>(s->heavy.p);
  a.heavy_off = static_cast<int64_t*>(s->heavy_off.p);
  a.ctl = static_cast<Ctl*>(s->ctl.p);
  a.nq = s->last.n_queries;
  a.sem = s->last.semantics;
  a.h = sh->next_hop;
  sa.lidx = sh->lidx;
  sa.hub_index = sh->hub_index;
  sa.hub_ids = sh->hub_ids;
  sa.O = static_cast<uint32_t*>(sh->O.p);
  sa.Of = static_cast<uint32_t*>(sh->Of.p);
  sa.olist = static_cast<int32_t*>(sh->olist.p);
  sa.olen = &a.ctl->olen;
  sa.E_global = sh->E;
  sa.n_local = sh->n_local;
  sa.n_hubs = sh->H;
  sa.rank = sh->rank;
  sa.world = sh->world;
  sa.px.base = sh->d_peers;
  sa.px.cap = sh->xcap;
  sa.px.off_keys = sh->off_keys;
  sa.px.off_bits = sh->off_bits;
  sa.px.off_hubs = sh->off_hubs;
  return sa;
}

template <int W>
WaveBufs shard_bufs(Shard* sh) {
  Session* s = &sh->s;
  WaveBufs b{};
  b.W = W;
  b.X = static_cast<uint32_t*>(s->X.p);
  b.N = static_cast<uint32_t*>(s->N.p);
  b.V = static_cast<uint32_t*>(s->V.p);
  b.S = static_cast<uint32_t*>(s->S.p);
  b.Xf = static_cast<uint32_t*>(s->Xf.p);
  b.Nf = static_cast<uint32_t*>(s->Nf.p);
  b.Vf = static_cast<uint32_t*>(s->Vf.p);
  b.M = static_cast<uint32_t*>(s->M.p);
  b.lists = static_cast<int32_t*>(s->lists.p);
  b.heavy = static_cast<int32_t*>(s->heavy.p);
  b.counts = static_cast<int32_t*>(s->counts.p);
  b.totals = static_cast<int64_t*>(s->totals.p);
  b.counts2 = static_cast<int32_t*>(s->counts2.p);  // second K4 slot (overlapped layers)
  b.totals2 = static_cast<int64_t*>(s->totals2.p);
  b.ctl = static_cast<Ctl*>(s->ctl.p);
  return b;
}

// edge counts come from the seeds / the previous layer's K4 (unfiltered
// FRONTIER/EXACT waves without hub slices, whose rows K4 does not cover)
bool shard_fused_edges(const Shard* sh) {
  const th_query& q = sh->s.last;
  return sh->H == 0 && !q.d_rel_masks && q.semantics != TH_CUMULATIVE;
}

template <int W>
void shard_begin_w(Shard* sh, const th_query* q) {
  Session* s = &sh->s;
  cudaStream_t st = s->st;
  const int64_t rows = std::max<int64_t>(sh->rows(), 1);
  const int64_t k = q->k;
  const int64_t fwords = ceil_div(rows, 32) + 1;
  for (DBuf* d : {&s->X, &s->N, &s->V, &s->S}) {
    if (d == &s->S && q->semantics != TH_CUMULATIVE) continue;
    if (d->bytes < (size_t)rows * W * 4) {
      ensure<uint32_t>(*d, rows * W, st);
      TH_CUDA(cudaMemsetAsync(d->p, 0, d->bytes, st));
    }
  }
  ensure<uint32_t>(s->Xf, fwords, st);
  ensure<uint32_t>(s->Nf, fwords, st);
  ensure<uint32_t>(s->Vf, fwords, st);
  ensure<int32_t>(s->lists, (k + 1) * rows, st);
  ensure<int32_t>(s->heavy, rows, st);
  ensure<int64_t>(s->heavy_off, rows + 1, st);
  if (q->d_rel_masks) ensure<uint32_t>(s->M, std::max<int64_t>(sh->g.R, 1) * W, st);
  ensure<int32_t>(s->counts, (int64_t)kMaxWave * (kMatBlocks + 64), st);
  ensure<int64_t>(s->totals, kMaxWave + 1, st);
  ensure<int32_t>(s->counts2, (int64_t)kMaxWave * (kMatBlocks + 64), st);
  ensure<int64_t>(s->totals2, kMaxWave + 1, st);
  if (sh->world > 1) {
    // remote staging, global-indexed (push pre-dedupe, pull frontier copy)
    const int64_t E = std::max<int64_t>(sh->E, 1);
    if (sh->O.bytes < (size_t)E * W * 4) {
      ensure<uint32_t>(sh->O, E * W, st);
      TH_CUDA(cudaMemsetAsync(sh->O.p, 0, sh->O.bytes, st));
    }
    if (sh->Of.bytes < (size_t)(ceil_div(E, 32) + 1) * 4) {
      ensure<uint32_t>(sh->Of, ceil_div(E, 32) + 1, st);
      TH_CUDA(cudaMemsetAsync(sh->Of.p, 0, sh->Of.bytes, st));
    }
    ensure<int32_t>(sh->olist, E, st);
  }
  Ctl* ctl = static_cast<Ctl*>(s->ctl.p);
  TH_CUDA(cudaMemsetAsync(ctl, 0, sizeof(Ctl), st));
  TH_CUDA(cudaMemsetAsync(s->Xf.p, 0, fwords * 4, st));
  TH_CUDA(cudaMemsetAsync(s->Nf.p, 0, fwords * 4, st));
  TH_CUDA(cudaMemsetAsync(s->Vf.p, 0, fwords * 4, st));
  // own inbox empty, overflow flag down (peers send only after the barrier
  // that follows this call)
  TH_CUDA(cudaMemsetAsync(sh->xr, 0, 16, st));
  sh->next_hop = 0;
  ShardArgs sa = shard_args<W>(sh);
  if (q->d_rel_masks) {
    build_mask_kernel<W><<<grid_for(sh->g.R * W), kThreads, 0, st>>>(
        q->d_rel_masks, q->mask_words, 0, q->n_queries, sh->g.R, static_cast<uint32_t*>(s->M.p));
    TH_LAUNCHED();
    s->launches += 1;
  }
  shard_seed_kernel<W><<<grid_for((int64_t)q->n_queries * 32), kThreads, 0, st>>>(
      sa, q->d_seed_offsets, q->d_seeds,
      shard_fused_edges(sh) ? static_cast<int64_t*>(s->edges.p) : nullptr);
  TH_LAUNCHED();
  shard_publish_cost_kernel<<<1, kMaxWorld, 0, st>>>(sa, 0);  // hop 1's frontier = the seeds
  TH_LAUNCHED();
  s->launches += 2;
  sh->next_hop = 1;
  sh->next_phase = 0;
}

// frontier-only waves overlap each layer's K4 with the next hop
bool shard_overlaps(Shard* sh) {
  const th_query& q = sh->s.last;
  const bool on = sh->s.overlap && (q.flags & TH_WANT_FRONTIERS) && !(q.flags & TH_WANT_ACTIVATED) &&
                  q.semantics != TH_CUMULATIVE;
  if (on) ensure_side_stream(&sh->s);
  return on;
}

// phase 0: direction, edge counts, activated triples, then push (local
// test-and-set + remote staging -> owners' inboxes) or pull (owned frontier
// rows -> every inbox); the unchosen direction's kernels exit at once
template <int W>
void shard_send_w(Shard* sh, int h) {
  Session* s = &sh->s;
  cudaStream_t st = s->st;
  const th_query& q = s->last;
  const bool filter = q.d_rel_masks != nullptr;
  const int64_t B = q.n_queries;
  WaveBufs b = shard_bufs<W>(sh);
  ShardArgs sa = shard_args<W>(sh);
  sa.a.h = h;
  const unsigned pg = persistent_grid();
  {
    ProfScope ps(s, TH_PROF_SETUP);
    shard_begin_hop_kernel<<<1, 1, 0, st>>>(sa, h, sh->T_global, sh->pull_divisor, sh->can_pull ? 1 : 0);
    TH_LAUNCHED();
    s->launches += 1;
  }
  int64_t* e_out = static_cast<int64_t*>(s->edges.p) + (h - 1) * B;
  // (no hub slices and no filter: the previous layer's K4 (or the seeds)
  // already summed the expanded rows' out-degrees)
  if (!shard_fused_edges(sh)) {
    ProfScope ps(s, TH_PROF_EDGES);
    if (filter) {
      edge_count_filtered_kernel<W><<<pg, kThreads, 0, st>>>(sa.a, e_out, 0);
      TH_LAUNCHED();
      heavy_scan_kernel<<<1, 1024, 0, st>>>(sa.a.indptr, sa.a.heavy, sa.a.ctl, sa.a.heavy_off, -1);
      TH_LAUNCHED();
      edge_count_filtered_kernel<W><<<pg, kThreads, 0, st>>>(sa.a, e_out, 1);
      TH_LAUNCHED();
      s->launches += 3;
    } else {
      edge_count_kernel<W><<<pg, kThreads, 0, st>>>(sa.a, e_out);
      TH_LAUNCHED();
      s->launches += 1;
    }
  }
  if (q.flags & TH_WANT_ACTIVATED) {
    ProfScope ps(s, TH_PROF_ACTIVATED);
    materialize_triples<W>(s, b, (int)B, static_cast<int64_t*>(s->a_off.p) + (h - 1) * B,
                           static_cast<int64_t*>(s->a_len.p) + (h - 1) * B,
                           static_cast<int32_t*>(s->a_ids.p), s->a_cap, &b.ctl->act_used);
  }
  {
    ProfScope ps(s, TH_PROF_PUSH);
    const int sem = q.semantics == TH_EXACT ? TH_EXACT : TH_FRONTIER;
#define TH_SHARD_PUSH(SEM, F)                                                      \
  shard_push_light_kernel<W, SEM, F><<<pg, kThreads, 0, st>>>(sa);               \
  TH_LAUNCHED();                                                                 \
  heavy_scan_kernel<<<1, 1024, 0, st>>>(sa.a.indptr, sa.a.heavy, sa.a.ctl,         \
                                       sa.a.heavy_off, h);                       \
  TH_LAUNCHED();                                                                 \
  shard_push_heavy_kernel<W, SEM, F><<<pg, kThreads, 0, st>>>(sa);               \
  TH_LAUNCHED();
    if (filter) {
      if (sem == TH_EXACT) { TH_SHARD_PUSH(TH_EXACT, true) } else { TH_SHARD_PUSH(TH_FRONTIER, true) }
    } else {
      if (sem == TH_EXACT) { TH_SHARD_PUSH(TH_EXACT, false) } else { TH_SHARD_PUSH(TH_FRONTIER, false) }
    }
#undef TH_SHARD_PUSH
    s->launches += 3;  // light, heavy-chunk scan, heavy
    if (sh->world > 1) {
      shard_send_kernel<W><<<pg, kThreads, 0, st>>>(sa);
      TH_LAUNCHED();
      shard_frontier_send_kernel<W><<<pg, kThreads, 0, st>>>(sa, h - 1, sh->l2g);
      TH_LAUNCHED();
      s->launches += 2;
    }
  }
}

// phase 1: apply what the peers sent (push: inbox records; pull: staged
// frontier + pull over the owned in-edges), empty the inbox, publish the
// owned hubs' next-layer rows
template <int W>
void shard_receive_w(Shard* sh, int h) {
  Session* s = &sh->s;
  cudaStream_t st = s->st;
  ShardArgs sa = shard_args<W>(sh);
  sa.a.h = h;
  const unsigned pg = persistent_grid();
  const bool filter = s->last.d_rel_masks != nullptr;
  const int sem = s->last.semantics;
  if (sh->world > 1) {
    ProfScope ps(s, TH_PROF_PUSH);
    if (sem == TH_EXACT) shard_absorb_kernel<W, TH_EXACT><<<pg, kThreads, 0, st>>>(sa);
    else shard_absorb_kernel<W, TH_FRONTIER><<<pg, kThreads, 0, st>>>(sa);
    TH_LAUNCHED();
    s->launches += 1;
  }
  if (sh->can_pull) {
    ProfScope ps(s, TH_PROF_PULL);
    WaveArgs pa = sa.a;
    if (sh->world > 1) {
      shard_gather_frontier_kernel<W><<<pg, kThreads, 0, st>>>(sa, h - 1);
      TH_LAUNCHED();
      pa.X = sa.O;
      pa.Xf = sa.Of;
      s->launches += 1;
    }
    // (one rank: the frontier is X itself, global rows = local rows)
    pa.rsrc = sh->gin.rsrc;
    pa.rrel = sh->gin.rrel;
    pa.item_v = sh->gin.item_v;
    pa.item_lo = sh->gin.item_lo;
    pa.item_hi = sh->gin.item_hi;
    pa.n_items = sh->gin.n_items;
    if (sem == TH_EXACT) {
      if (filter) launch_pull<W, TH_EXACT, true>(s, &sh->gin, pa, st);
      else launch_pull<W, TH_EXACT, false>(s, &sh->gin, pa, st);
    } else {
      if (filter) launch_pull<W, TH_FRONTIER, true>(s, &sh->gin, pa, st);
      else launch_pull<W, TH_FRONTIER, false>(s, &sh->gin, pa, st);
    }
    if (sh->world > 1) {
      shard_clear_frontier_kernel<W><<<pg, kThreads, 0, st>>>(sa, h - 1);
      TH_LAUNCHED();
      s->launches += 1;
    }
  }
  shard_inbox_reset_kernel<<<1, 32, 0, st>>>(sa);
  TH_LAUNCHED();
  s->launches += 1;
  if (h < s->last.k && sh->H > 0) {  // the last layer is never expanded
    shard_hub_out_kernel<W><<<grid_for(sh->H * W), kThreads, 0, st>>>(sa);
    TH_LAUNCHED();
    s->launches += 1;
  }
}

// phase 2: hub frontier rows from the board, K4 over the owned rows, retire
// X, publish the new layer's cost
template <int W>
void shard_end_w(Shard* sh, int h) {
  Session* s = &sh->s;
  cudaStream_t st = s->st;
  const th_query& q = s->last;
  const int64_t B = q.n_queries;
  WaveBufs b = shard_bufs<W>(sh);
  ShardArgs sa = shard_args<W>(sh);
  sa.a.h = h;
  const int64_t rows = std::max<int64_t>(sh->rows(), 1);
  const int64_t fwords = ceil_div(rows, 32) + 1;
  if (h < q.k && sh->H > 0) {
    shard_hub_in_kernel<W><<<grid_for(sh->H), kThreads, 0, st>>>(sa);
    TH_LAUNCHED();
    s->launches += 1;
  }
  // as in run_wave: the layer's K4 runs on a side stream (consecutive
  // layers alternate between two, with their own scratch) and overlaps the
  // next hop's phases, which only read the layer
  const bool overlap = shard_overlaps(sh);
  if (q.flags & TH_WANT_FRONTIERS) {
    const int slot = overlap ? (int)(h & 1) : 0;
    cudaStream_t kst = slot ? s->side2 : s->side;
    if (overlap) {
      TH_CUDA(cudaEventRecord(s->ev_expand[h], st));
      TH_CUDA(cudaStreamWaitEvent(kst, s->ev_expand[h], 0));
    }
    StreamScope scope(s, overlap ? kst : st);
    s->k4_slot = slot;
    s->mark_counted = overlap ? s->ev_cnt[h] : nullptr;
    s->counted_recorded = false;
    {
      ProfScope ps(s, TH_PROF_FRONTIER);
      int64_t* f_off = static_cast<int64_t*>(s->f_off.p) + (h - 1) * B;
      int64_t* f_len = static_cast<int64_t*>(s->f_len.p) + (h - 1) * B;
      int32_t* ids = static_cast<int32_t*>(s->f_ids.p);
      if (q.semantics == TH_CUMULATIVE) {
        materialize_dense<W>(s, b, b.V, b.S, b.Vf, (int)B, f_off, f_len, ids, s->f_cap, &b.ctl->ids_used);
      } else {
        // the layer is the next hop's frontier: its K4 count pass also
        // yields |T_{h+1}(q)| (all of this rank's expanded rows when there
        // are no hub slices)
        EdgeSum es{};
        if (h < q.k && shard_fused_edges(sh)) {
          int nplanes = 0;
          while (nplanes < 31 && (int64_t(1) << nplanes) <= sh->g.max_out) ++nplanes;
          es.indptr = sh->g.indptr;
          es.nplanes = nplanes;
          es.out = static_cast<int64_t*>(s->edges.p) + h * B;
        }
        materialize_dense<W>(s, b, b.N, nullptr, b.Nf, (int)B, f_off, f_len, ids, s->f_cap,
                             &b.ctl->ids_used, es);
      }
    }
    if (overlap) {
      TH_CUDA(cudaEventRecord(s->ev_mat[h], kst));
      if (!s->counted_recorded) TH_CUDA(cudaEventRecord(s->ev_cnt[h], kst));
    }
    s->mark_counted = nullptr;
    s->k4_slot = 0;
  }
  {
    // retiring X (layer h-1) waits until that layer's K4 read it
    if (overlap && h > 1) TH_CUDA(cudaStreamWaitEvent(st, s->ev_cnt[h - 1], 0));
    ProfScope ps(s, TH_PROF_CLEAR);
    clear_rows_kernel<W><<<grid_for(rows * W), kThreads, 0, st>>>(b.X, b.lists, b.ctl, h - 1, h - 1, rows);
    TH_LAUNCHED();
    TH_CUDA(cudaMemsetAsync(b.Xf, 0, fwords * 4, st));
    s->launches += 1;
  }
  if (h < q.k) {
    shard_publish_cost_kernel<<<1, kMaxWorld, 0, st>>>(sa, h);
    TH_LAUNCHED();
    s->launches += 1;
  }
  std::swap(s->X, s->N);
  std::swap(s->Xf, s->Nf);
}

template <int W>
void shard_retire_w(Shard* sh) {
  Session* s = &sh->s;
  cudaStream_t st = s->st;
  const th_query& q = s->last;
  const int k = q.k;
  WaveBufs b = shard_bufs<W>(sh);
  const int64_t rows = std::max<int64_t>(sh->rows(), 1);
  const bool overlap = shard_overlaps(sh);
  if (overlap) TH_CUDA(cudaStreamWaitEvent(st, s->ev_cnt[k], 0));
  clear_rows_kernel<W><<<grid_for(rows * W), kThreads, 0, st>>>(b.X, b.lists, b.ctl, k, k, rows);
  TH_LAUNCHED();
  if (overlap) {
    // results of the last two layers' K4s are complete before th_finish
    TH_CUDA(cudaStreamWaitEvent(st, s->ev_mat[k], 0));
    if (k > 1) TH_CUDA(cudaStreamWaitEvent(st, s->ev_mat[k - 1], 0));
  }
  if (q.semantics != TH_EXACT) {
    clear_rows_kernel<W><<<grid_for(rows * W), kThreads, 0, st>>>(b.V, b.lists, b.ctl, 0, k, rows);
    TH_LAUNCHED();
  }
  if (q.semantics == TH_CUMULATIVE) {
    clear_rows_kernel<W><<<grid_for(rows * W), kThreads, 0, st>>>(b.S, b.lists, b.ctl, 0, 0, rows);
    TH_LAUNCHED();
  }
  s->launches += 3;
}

#define TH_W_DISPATCH(W_, CALL)             \
  switch (W_) {                             \
    case 1: { constexpr int WW = 1; CALL; } break;   \
    case 2: { constexpr int WW = 2; CALL; } break;   \
    case 4: { constexpr int WW = 4; CALL; } break;   \
    case 8: { constexpr int WW = 8; CALL; } break;   \
    case 16: { constexpr int WW = 16; CALL; } break; \
    default: { constexpr int WW = 32; CALL; } break; \
  }

}  // namespace

int shard_create(Shard** out, const int32_t* d_subj, const int32_t* d_rel, const int32_t* d_obj,
                 int64_t T, int64_t E, int64_t R, const int32_t* d_lidx,
                 const int32_t* d_hub_index, const int32_t* d_hub_ids, int64_t H,
                 const int32_t* d_l2g, int64_t n_local, int32_t rank, int32_t world,
                 int64_t inbox_records, cudaStream_t st) {
  if (world > kMaxWorld) {
    set_error("world above " + std::to_string(kMaxWorld) + " ranks");
    return TH_ERR_INVALID;
  }
  auto* sh = new Shard();
  *out = sh;
  sh->E = E;
  sh->n_local = n_local;
  sh->H = H;
  sh->T_global = T;
  sh->rank = rank;
  sh->world = world;
  sh->lidx = dcopy(d_lidx, E, st);
  sh->hub_index = dcopy(d_hub_index, E, st);
  sh->hub_ids = dcopy(d_hub_ids, H, st);
  sh->l2g = dcopy(d_l2g, n_local, st);
  // select + compact this rank's triples (tid order kept)
  int32_t* key = nullptr;
  TH_CUDA(cudaMalloc(&key, sizeof(int32_t) * std::max<int64_t>(T, 1)));
  const int nb = (int)std::max<int64_t>(1, ceil_div(T, kCompactWords));
  int32_t* bsum = nullptr;
  TH_CUDA(cudaMalloc(&bsum, sizeof(int32_t) * (nb + 1)));
  if (T > 0) {
    shard_select_kernel<<<grid_for(T), kThreads, 0, st>>>(d_subj, T, sh->lidx, sh->hub_index,
                                                         n_local, rank, world, key);
    TH_LAUNCHED();
    shard_count_kernel<<<nb, kCompactThreads, 0, st>>>(key, T, bsum);
    TH_LAUNCHED();
    flag_scan_kernel<<<1, 1024, 0, st>>>(bsum, nb, bsum + nb);
    TH_LAUNCHED();
  } else {
    TH_CUDA(cudaMemsetAsync(bsum + nb, 0, sizeof(int32_t), st));
  }
  int32_t tl = 0;
  TH_CUDA(cudaMemcpyAsync(&tl, bsum + nb, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  TH_CUDA(cudaStreamSynchronize(st));
  int32_t *okey = nullptr, *orel = nullptr, *oobj = nullptr;
  const int64_t tcap = std::max<int32_t>(tl, 1);
  TH_CUDA(cudaMalloc(&okey, sizeof(int32_t) * tcap));
  TH_CUDA(cudaMalloc(&orel, sizeof(int32_t) * tcap));
  TH_CUDA(cudaMalloc(&oobj, sizeof(int32_t) * tcap));
  TH_CUDA(cudaMalloc(&sh->tid_l2g, sizeof(int32_t) * tcap));
  if (T > 0) {
    shard_gather_kernel<<<nb, kCompactThreads, 0, st>>>(key, T, bsum, d_rel, d_obj, okey, orel, oobj,
                                                        sh->tid_l2g);
    TH_LAUNCHED();
  }
  int rc = graph_build(&sh->g, okey, orel, oobj, tl, n_local + H, R, false, st, E);
  TH_CUDA(cudaStreamSynchronize(st));
  for (void* p : {(void*)okey, (void*)orel, (void*)oobj}) cudaFree(p);
  if (rc != TH_OK) {
    cudaFree(key);
    cudaFree(bsum);
    return rc;
  }
  // in-edges of the owned objects (global sources) for pull hops; pull
  // records carry 64-bit keys, so every graph size qualifies
  if (T > 0) {
    shard_select_in_kernel<<<grid_for(T), kThreads, 0, st>>>(d_obj, T, sh->lidx, rank, world, key);
    TH_LAUNCHED();
    shard_count_kernel<<<nb, kCompactThreads, 0, st>>>(key, T, bsum);
    TH_LAUNCHED();
    flag_scan_kernel<<<1, 1024, 0, st>>>(bsum, nb, bsum + nb);
    TH_LAUNCHED();
    int32_t ti = 0;
    TH_CUDA(cudaMemcpyAsync(&ti, bsum + nb, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    TH_CUDA(cudaStreamSynchronize(st));
    const int64_t icap = std::max<int32_t>(ti, 1);
    int32_t *ikey = nullptr, *irel = nullptr, *isub = nullptr, *itid = nullptr;
    TH_CUDA(cudaMalloc(&ikey, sizeof(int32_t) * icap));
    TH_CUDA(cudaMalloc(&irel, sizeof(int32_t) * icap));
    TH_CUDA(cudaMalloc(&isub, sizeof(int32_t) * icap));
    TH_CUDA(cudaMalloc(&itid, sizeof(int32_t) * icap));
    shard_gather_kernel<<<nb, kCompactThreads, 0, st>>>(key, T, bsum, d_rel, d_subj, ikey, irel, isub,
                                                        itid);
    TH_LAUNCHED();
    // forward side keyed by the global subject (unused), reverse side by the
    // object's local row: items cover the owned rows
    rc = graph_build(&sh->gin, isub, irel, ikey, ti, E, R, true, st, E);
    TH_CUDA(cudaStreamSynchronize(st));
    for (void* p : {(void*)ikey, (void*)irel, (void*)isub, (void*)itid}) cudaFree(p);
    if (rc != TH_OK) {
      cudaFree(key);
      cudaFree(bsum);
      return rc;
    }
    sh->can_pull = true;
  }
  cudaFree(key);
  cudaFree(bsum);
  TH_CUDA(cudaMalloc(&sh->d_peers, sizeof(uint8_t*) * world));
  shard_alloc_region(sh, std::max<int64_t>(inbox_records, 1024), st);
  shard_publish_peers(sh);  // (one rank: connected to itself already)
  Session* s = &sh->s;
  s->g = &sh->g;
  s->st = st;
  s->pull_divisor = 0.0;
  s->mat_rows = n_local;
  // (one rank owns every entity and triple in id order: both maps are the
  // identity, and K4 skips the per-id lookups)
  s->row_map = world > 1 ? sh->l2g : nullptr;
  s->tid_map = world > 1 ? sh->tid_l2g : nullptr;
  return TH_OK;
}

int64_t shard_local_triples(const Shard* sh) { return sh->g.T; }

int shard_region(const Shard* sh, void** base, uint64_t* bytes, int64_t* records) {
  *base = sh->xr;
  *bytes = sh->xr_bytes;
  if (records) *records = sh->xcap;
  return TH_OK;
}

int shard_ipc_handle(const Shard* sh, void* out64) {
  cudaIpcMemHandle_t h;
  TH_CUDA(cudaIpcGetMemHandle(&h, sh->xr));
  static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
  std::memcpy(out64, &h, sizeof(h));
  return TH_OK;
}

int shard_connect(Shard* sh, int32_t peer, void* base, bool ipc) {
  if (peer < 0 || peer >= sh->world) {
    set_error("peer rank out of range");
    return TH_ERR_INVALID;
  }
  if (peer == sh->rank) {
    if (base != sh->xr) {
      set_error("a shard's own region is its own");
      return TH_ERR_INVALID;
    }
  } else {
    if (sh->peer_ipc[peer] && sh->peers[peer]) cudaIpcCloseMemHandle(sh->peers[peer]);
    sh->peers[peer] = static_cast<uint8_t*>(base);
    sh->peer_ipc[peer] = ipc;
  }
  shard_publish_peers(sh);
  return TH_OK;
}

int shard_ipc_open(Shard* sh, int32_t peer, const void* handle64) {
  if (peer == sh->rank) return shard_connect(sh, peer, sh->xr, false);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  void* p = nullptr;
  TH_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  return shard_connect(sh, peer, p, true);
}

int shard_grow_inbox(Shard* sh, int64_t records) {
  if (records <= sh->xcap) return TH_OK;
  shard_close_peers(sh);
  shard_alloc_region(sh, records, sh->s.st);
  shard_publish_peers(sh);
  return TH_OK;
}

int shard_begin(Shard* sh, const th_query* q) {
  Session* s = &sh->s;
  if (q->k < 1 || q->k > kMaxK) {
    set_error("hop count must be in [1, " + std::to_string(kMaxK) + "]");
    return TH_ERR_INVALID;
  }
  if (q->semantics < TH_EXACT || q->semantics > TH_CUMULATIVE) {
    set_error("unknown hop semantics");
    return TH_ERR_INVALID;
  }
  if (q->n_queries < 0 || q->n_queries > kMaxWave ||
      (q->n_queries > 0 && (!q->d_seed_offsets || !q->d_seeds))) {
    set_error("a partitioned wave takes 0..1024 queries with device seed arrays");
    return TH_ERR_INVALID;
  }
  if (q->d_rel_masks && q->mask_words < ceil_div(sh->g.R, 32)) {
    set_error("mask_words too small for the relation count");
    return TH_ERR_INVALID;
  }
  if (q->flags & TH_WANT_PATHS) {
    set_error("path reconstruction is not available on partitioned graphs");
    return TH_ERR_INVALID;
  }
  if (!shard_connected(sh)) {
    set_error("exchange regions of the peers are not connected (th_shard_connect / th_shard_ipc_open)");
    return TH_ERR_STATE;
  }
  cudaStream_t st = s->st;
  const int64_t B = q->n_queries, k = q->k;
  const int64_t kb = std::max<int64_t>(k * B, 1);
  ensure<Ctl>(s->ctl, 1, st);
  for (DBuf* d : {&s->f_off, &s->f_len, &s->a_off, &s->a_len, &s->edges}) {
    ensure<int64_t>(*d, kb, st);
    TH_CUDA(cudaMemsetAsync(d->p, 0, sizeof(int64_t) * kb, st));
  }
  s->f_cap = std::max<int64_t>({s->f_cap, s->last_f_need, 1 << 16});
  s->a_cap = std::max<int64_t>({s->a_cap, s->last_a_need, 1 << 16});
  ensure<int32_t>(s->f_ids, s->f_cap, st);
  ensure<int32_t>(s->a_ids, s->a_cap, st);
  s->last = *q;
  s->has_run = true;
  sh->W = pick_words((int)std::max<int64_t>(B, 1));
  sh->in_wave = true;
  sh->retired = false;
  TH_W_DISPATCH(sh->W, shard_begin_w<WW>(sh, q));
  return TH_OK;
}

int shard_hop(Shard* sh, int h, int phase) {
  if (!sh->in_wave) {
    set_error("no wave in progress (th_shard_begin first)");
    return TH_ERR_STATE;
  }
  if (h != sh->next_hop || h > sh->s.last.k || phase != sh->next_phase) {
    set_error("hop or phase out of sequence");
    return TH_ERR_STATE;
  }
  NvtxRange nvtx_phase("th shard hop %d phase %d", h, phase);
  if (phase == 0 && sh->hc) {
    // the frontier's hub pages resident before any kernel of the hop reads
    // them (the host waits for the flags; the loads queue on the stream)
    TH_CUDA(cudaStreamSynchronize(sh->s.st));
    const int rc = hubcache_step(sh->hc, static_cast<const uint32_t*>(sh->s.Xf.p), sh->s.st);
    if (rc != TH_OK) {
      sh->in_wave = false;
      return rc;
    }
  }
  if (phase == 0) TH_W_DISPATCH(sh->W, shard_send_w<WW>(sh, h))
  else if (phase == 1) TH_W_DISPATCH(sh->W, shard_receive_w<WW>(sh, h))
  else TH_W_DISPATCH(sh->W, shard_end_w<WW>(sh, h))
  sh->next_phase = (phase + 1) % 3;
  if (phase == 2) sh->next_hop = h + 1;
  return TH_OK;
}

int shard_can_pull(const Shard* sh) { return sh->can_pull ? 1 : 0; }

void shard_set_pull_divisor(Shard* sh, double d) { sh->pull_divisor = d; }

int shard_finish(Shard* sh, th_result* out) {
  if (!sh->in_wave || sh->next_hop != sh->s.last.k + 1) {
    set_error("th_shard_finish before the last hop ended");
    return TH_ERR_STATE;
  }
  if (!sh->retired) TH_W_DISPATCH(sh->W, shard_retire_w<WW>(sh));
  sh->in_wave = false;
  const int rc = session_finish(&sh->s, out);
  XCtrl xc;
  TH_CUDA(cudaMemcpy(&xc, sh->xr, sizeof(XCtrl), cudaMemcpyDeviceToHost));
  if (xc.overflow) {
    // the inbox must grow: every rank reallocates and reconnects, then the
    // wave runs again (th_shard_grow_inbox)
    set_error("exchange inbox overflowed; grow it and run the wave again");
    return TH_ERR_OVERFLOW;
  }
  return rc;
}

int shard_columns(const Shard* sh, th_shard_cols* out) {
  out->n_triples = sh->g.T;
  out->n_local = sh->n_local;
  out->n_hubs = sh->H;
  out->subj_row = sh->g.subj;
  out->rel = sh->g.rel;
  out->obj = sh->g.obj;
  out->tid_l2g = sh->tid_l2g;
  out->l2g = sh->l2g;
  out->hub_ids = sh->hub_ids;
  return TH_OK;
}

int shard_sent(Shard* sh, int64_t* per_hop, int n) {
  TH_CUDA(cudaStreamSynchronize(sh->s.st));
  Ctl c;
  TH_CUDA(cudaMemcpy(&c, sh->s.ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; ++i) per_hop[i] = i + 1 <= sh->s.last.k ? (int64_t)c.sent[i + 1] : 0;
  return TH_OK;
}

int shard_inbox_overflowed(const Shard* sh) {
  XCtrl xc;
  if (cudaMemcpy(&xc, sh->xr, sizeof(XCtrl), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return xc.overflow ? 1 : 0;
}

Session* shard_session(Shard* sh) { return &sh->s; }

int shard_hub_cache(Shard* sh, int64_t capacity) {
  if (sh->in_wave) {
    set_error("the hub cache cannot be enabled during a wave");
    return TH_ERR_STATE;
  }
  if (sh->hc) {
    set_error("the shard's hub cache is enabled already");
    return TH_ERR_STATE;
  }
  TH_CUDA(cudaStreamSynchronize(sh->s.st));
  return hubcache_create(&sh->hc, &sh->g, sh->n_local, capacity, sh->s.st);
}

HubCache* shard_hub_cache_of(Shard* sh) { return sh->hc; }

namespace {

// the shard-side buffers a captured wave bakes in (exchange region, staging)
uint64_t shard_sig(const Shard* sh) {
  uint64_t h = 1469598103934665603ull;
  for (uint64_t v : {(uint64_t)(uintptr_t)sh->xr, (uint64_t)sh->xcap, (uint64_t)sh->off_keys,
                     (uint64_t)sh->off_bits, (uint64_t)sh->off_hubs, (uint64_t)(uintptr_t)sh->O.p,
                     (uint64_t)sh->O.bytes, (uint64_t)(uintptr_t)sh->Of.p, (uint64_t)(uintptr_t)sh->olist.p,
                     (uint64_t)(uintptr_t)sh->d_peers, (uint64_t)(sh->pull_divisor * 1024.0),
                     // (the graph arrays too: a shard built later at a freed shard's address)
                     (uint64_t)(uintptr_t)sh->g.indptr, (uint64_t)(uintptr_t)sh->g.csr_obj,
                     (uint64_t)(uintptr_t)sh->g.csr_rel, (uint64_t)(uintptr_t)sh->g.csr_tid,
                     (uint64_t)(uintptr_t)sh->g.subj, (uint64_t)(uintptr_t)sh->gin.rsrc,
                     (uint64_t)(uintptr_t)sh->gin.item_v, (uint64_t)(uintptr_t)sh->lidx,
                     (uint64_t)(uintptr_t)sh->l2g, (uint64_t)(uintptr_t)sh->tid_l2g}) {
    h ^= v;
    h *= 1099511628211ull;
  }
  return h;
}

// host-side state a begin + all hops leave behind (a replayed graph ran them)
void shard_mark_wave(Shard* sh, const th_query* q) {
  Session* s = &sh->s;
  s->f_cap = std::max<int64_t>({s->f_cap, s->last_f_need, 1 << 16});
  s->a_cap = std::max<int64_t>({s->a_cap, s->last_a_need, 1 << 16});
  s->last = *q;
  s->has_run = true;
  sh->W = pick_words((int)std::max<int64_t>(q->n_queries, 1));
  sh->in_wave = true;
  sh->next_hop = q->k + 1;
  sh->next_phase = 0;
  sh->retired = true;
}

int shards_issue(Shard* const* sh, int n, const th_query* q) {
  for (int i = 0; i < n; ++i) {
    const int rc = shard_begin(sh[i], &q[i]);
    if (rc != TH_OK) return rc;
  }
  for (int h = 1; h <= q[0].k; ++h)
    for (int phase = 0; phase < 3; ++phase)
      for (int i = 0; i < n; ++i) {
        const int rc = shard_hop(sh[i], h, phase);
        if (rc != TH_OK) return rc;
      }
  // the retire kernels too (they join the K4 side streams back)
  for (int i = 0; i < n; ++i) {
    TH_W_DISPATCH(sh[i]->W, shard_retire_w<WW>(sh[i]));
    sh[i]->retired = true;
  }
  return TH_OK;
}

void wave_keys(Shard* const* sh, int n, const th_query* q, std::vector<GraphKey>& keys,
               std::vector<uint64_t>& sigs) {
  keys.resize(n);
  sigs.resize(n);
  for (int i = 0; i < n; ++i) {
    keys[i] = graph_key(&sh[i]->s, &q[i]);
    sigs[i] = shard_sig(sh[i]);
  }
}

}  // namespace

int shards_run_wave(Shard* const* sh, int n, const th_query* q, const int64_t* n_seeds) {
  cudaStream_t st = sh[0]->s.st;
  bool graphable = n >= 1;
  for (int i = 0; i < n && graphable; ++i)
    graphable = !sh[i]->hc && !sh[i]->s.prof && sh[i]->s.st == st && q[i].n_queries > 0 &&
                q[i].k == q[0].k && shard_connected(sh[i]);
  if (!graphable) return shards_issue(sh, n, q);
  // stage the inputs into session buffers (their addresses are baked in)
  std::vector<th_query> qs(q, q + n);
  for (int i = 0; i < n; ++i) {
    Session* s = &sh[i]->s;
    const int64_t B = q[i].n_queries;
    qs[i].d_seed_offsets = stage(s->in_offs, q[i].d_seed_offsets, B + 1, st);
    qs[i].d_seeds = stage(s->in_seeds, q[i].d_seeds, std::max<int64_t>(n_seeds[i], 1), st);
    if (q[i].d_rel_masks)
      qs[i].d_rel_masks = stage(s->in_masks, q[i].d_rel_masks, B * (int64_t)q[i].mask_words, st);
  }
  if (!sh[0]->group) sh[0]->group = new WaveGraph();
  WaveGraph* G = sh[0]->group;
  std::vector<GraphKey> keys;
  std::vector<uint64_t> sigs;
  wave_keys(sh, n, qs.data(), keys, sigs);
  const bool same = G->members == std::vector<Shard*>(sh, sh + n) && G->keys == keys && G->sigs == sigs;
  if (G->exec && G->valid && same) {
    TH_CUDA(cudaGraphLaunch(G->exec, st));
    for (int i = 0; i < n; ++i) shard_mark_wave(sh[i], &qs[i]);
    sh[0]->s.launches += G->launches;
    return TH_OK;
  }
  if (G->exec) cudaGraphExecDestroy(G->exec);
  G->exec = nullptr;
  G->valid = false;
  static const bool dbg_w = std::getenv("TH_GRAPH_DEBUG") != nullptr;
  if (dbg_w)
    std::fprintf(stderr, "[th] wave: exec=%d valid=%d seen=%d same=%d failures=%d\n", (int)(G->exec != nullptr),
                 (int)G->valid, (int)G->seen, (int)same, G->failures);
  if (!(G->seen && same) || G->failures >= 3) {
    // first wave of this shape: eager (sizes every buffer), remembered
    const int rc = shards_issue(sh, n, qs.data());
    G->members.assign(sh, sh + n);
    wave_keys(sh, n, qs.data(), G->keys, G->sigs);
    G->seen = rc == TH_OK;
    return rc;
  }
  // second wave of the same shape: capture on a session-owned stream
  if (!G->cap) {
    int least = 0, greatest = 0;
    TH_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    TH_CUDA(cudaStreamCreateWithPriority(&G->cap, cudaStreamNonBlocking, greatest));
  }
  // (the capture stream must see the staged inputs)
  cudaEvent_t staged;
  TH_CUDA(cudaEventCreateWithFlags(&staged, cudaEventDisableTiming));
  TH_CUDA(cudaEventRecord(staged, st));
  TH_CUDA(cudaStreamWaitEvent(G->cap, staged, 0));
  cudaEventDestroy(staged);
  std::vector<int64_t> l0(n);
  for (int i = 0; i < n; ++i) {
    l0[i] = sh[i]->s.launches;
    sh[i]->s.st = G->cap;
  }
  TH_CUDA(cudaStreamBeginCapture(G->cap, cudaStreamCaptureModeThreadLocal));
  int rc = TH_OK;
  bool threw = false;
  try {
    rc = shards_issue(sh, n, qs.data());
  } catch (const CudaError&) {
    threw = true;
  }
  for (int i = 0; i < n; ++i) sh[i]->s.st = st;
  cudaGraph_t graph = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(G->cap, &graph);
  std::vector<GraphKey> after;
  std::vector<uint64_t> after_sigs;
  wave_keys(sh, n, qs.data(), after, after_sigs);
  if (threw || rc != TH_OK || ce != cudaSuccess || after != keys || after_sigs != sigs) {
    // capture is an optimisation: drop it and run this wave eagerly
    static const bool dbg = std::getenv("TH_GRAPH_DEBUG") != nullptr;
    if (dbg)
      std::fprintf(stderr, "[th] wave capture dropped: threw=%d rc=%d end=%s keys=%d sigs=%d\n", (int)threw, rc,
                   cudaGetErrorString(ce), (int)(after == keys), (int)(after_sigs == sigs));
    if (graph) cudaGraphDestroy(graph);
    (void)cudaGetLastError();
    G->failures += 1;
    G->seen = false;
    for (int i = 0; i < n; ++i) sh[i]->s.launches = l0[i];
    return shards_issue(sh, n, qs.data());
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, graph, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(graph);
  TH_CUDA(ie);
  G->exec = exec;
  G->valid = true;
  G->launches = 0;
  for (int i = 0; i < n; ++i) G->launches += sh[i]->s.launches - l0[i];
  TH_CUDA(cudaGraphLaunch(G->exec, st));
  return TH_OK;
}

void shard_free(Shard* sh) {
  if (sh->group) {
    if (sh->group->exec) cudaGraphExecDestroy(sh->group->exec);
    if (sh->group->cap) cudaStreamDestroy(sh->group->cap);
    delete sh->group;
  }
  session_free(&sh->s);
  if (sh->hc) hubcache_free(sh->hc, &sh->g);
  shard_close_peers(sh);
  for (DBuf* d : {&sh->O, &sh->Of, &sh->olist}) {
    if (d->p) cudaFree(d->p);
    d->p = nullptr;
  }
  for (void* p : {(void*)sh->tid_l2g, (void*)sh->lidx, (void*)sh->hub_index, (void*)sh->hub_ids,
                  (void*)sh->l2g, (void*)sh->xr, (void*)sh->d_peers})
    if (p) cudaFree(p);
  graph_free(&sh->g);
  graph_free(&sh->gin);
  delete sh;
}

}  // namespace th
