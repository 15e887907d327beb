// Part of engine.cu (included inside namespace th::{anonymous}).
//
// K6: one rank's side of the partitioned (multi-GPU) hop, the B200 form of
// the reference's Algorithm 1 (engine.py:94-135 _partitioned_expand: route
// -> local expand -> union).  One owner map serves both roles
//   own(v) = ((v * 0x9E3779B1) mod 2^32) mod world     (partition.py:80-84)
// -- the rank that stores v's out-row (subject-cohesive, partition.py:3-4)
// and the rank that holds v's per-query visited/next bits.  Hubs (the top
// out-degree entities) are the exception to subject cohesion: their rows
// are edge-split over all ranks (triple t of a hub lives on rank
// hash(t) mod world), and a hub in the frontier is expanded by every rank on
// its slice.
//
// Exchange: every rank owns an exchange region in its HBM -- control words
// (inbox cursor, overflow flag, the ranks' published frontier costs), an
// inbox of (int64 key, uint32 bits) records and a hub-row board -- and its
// peers WRITE INTO IT DIRECTLY: remote atomics reserve inbox space, plain
// stores deliver records, costs and hub rows (NVLink P2P within a box; the
// regions of other processes are CUDA-IPC mappings; on one device, plain
// pointers).  Nothing is read back to the host during a wave.  A hop runs in
// three phases separated by a barrier across ranks (the peers' writes of
// the previous phase are complete):
//   0 send     direction from the published costs (pull when the summed
//              frontier out-edges exceed T / pull_divisor, as K2/K3);
//              push: expand the local frontier rows + hub slices, owned
//              targets test-and-set directly, remote ones OR-ed into the
//              staging matrix O (each (query, target) leaves a rank at most
//              once per hop), then staged rows -> records in the owners'
//              inboxes; pull: the owned frontier rows -> records in EVERY
//              rank's inbox (an all-gather)
//   1 receive  push: test-and-set the inbox records; pull: stage the
//              gathered frontier (global rows), pull over the owned
//              in-edges; owners write their hubs' next-layer rows onto
//              every rank's hub board
//   2 end      install the hub frontier rows, K4 over the owned rows (ids
//              mapped to global), retire X, publish the new layer's cost
// Local row space: [0, n_local) owned entities in ascending id order, then
// [n_local, n_local + n_hubs) hub slices.
#pragma once

constexpr int kMaxWorld = 64;

// control words at the start of every exchange region
struct XCtrl {
  unsigned long long cursor;            // inbox records appended this hop
  unsigned int overflow;                // an append did not fit the inbox (sticky per wave)
  unsigned int pad;
  unsigned long long cost[kMaxWorld];   // frontier out-edge totals published by each rank
};
constexpr size_t kXCtrlBytes = 1024;
static_assert(sizeof(XCtrl) <= kXCtrlBytes, "control block");

// the peers' exchange regions as this rank's kernels see them
struct XPeers {
  uint8_t* const* base;  // [world] device base addresses (own included)
  int64_t cap;           // inbox records per region
  size_t off_keys, off_bits, off_hubs;
  __device__ __forceinline__ XCtrl* ctrl(int d) const { return reinterpret_cast<XCtrl*>(base[d]); }
  __device__ __forceinline__ uint64_t* keys(int d) const {
    return reinterpret_cast<uint64_t*>(base[d] + off_keys);
  }
  __device__ __forceinline__ uint32_t* bits(int d) const {
    return reinterpret_cast<uint32_t*>(base[d] + off_bits);
  }
  __device__ __forceinline__ uint32_t* hubs(int d) const {
    return reinterpret_cast<uint32_t*>(base[d] + off_hubs);
  }
};

struct ShardArgs {
  WaveArgs a;              // local rows = n_local + n_hubs
  const int32_t* lidx;     // [E_global] row of an entity at its owner
  const int32_t* hub_index;  // [E_global] -1 or hub number
  const int32_t* hub_ids;  // [n_hubs]
  uint32_t* O;             // [E_global][W] staged remote bits
  uint32_t* Of;            // [E_global / 32] staged-row flags
  int32_t* olist;          // staged global ids
  int32_t* olen;
  int64_t E_global, n_local, n_hubs;
  int32_t rank, world;
  XPeers px;
};

__device__ __forceinline__ int32_t owner_of(int64_t v, int32_t world) {
  return (int32_t)((uint32_t)((uint64_t)v * 0x9E3779B1ull) % (uint32_t)world);
}

// test-and-set of (local row, word j) with bits w (K2's PushOp on a row)
template <int W, int SEM>
__device__ __forceinline__ bool local_set(const WaveArgs& a, int32_t row, int j, uint32_t w) {
  const size_t r = (size_t)row * W + j;
  if (SEM == TH_EXACT) {
    if (!(w & ~__ldcg(&a.N[r]))) return false;
    const uint32_t old = atomicOr(&a.N[r], w);
    return old == 0u && flag_next(a, row);
  }
  if (!(w & ~__ldcg(&a.V[r]))) return false;
  const uint32_t old = atomicOr(&a.V[r], w);
  const uint32_t nb = w & ~old;
  if (!nb) return false;
  atomicOr(&a.N[r], nb);
  return flag_next(a, row);
}

// stage bits for a remote target; true for the first toucher of v this hop
template <int W>
__device__ __forceinline__ bool remote_stage(const ShardArgs& sa, int32_t v, int j, uint32_t w) {
  uint32_t* o = &sa.O[(size_t)v * W + j];
  if (!(w & ~__ldcg(o))) return false;
  atomicOr(o, w);
  const uint32_t fb = 1u << (v & 31);
  return !(atomicOr(&sa.Of[v >> 5], fb) & fb);
}

// seeds: owned seeds set local rows; hub seeds set their hub rows (every rank
// sees every seed, so hub rows need no exchange at hop 0)
// (e_out: |T_1(q)| = out-degree sum of q's distinct owned seeds, when the
// edge counts are fused -- no hub slices)
template <int W>
__global__ void shard_seed_kernel(ShardArgs sa, const int32_t* __restrict__ qoff,
                                  const int32_t* __restrict__ seeds, int64_t* e_out) {
  const WaveArgs& a = sa.a;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int q = gw; q < a.nq; q += nw) {
    const int32_t lo = qoff[q], hi = qoff[q + 1];
    const uint32_t qb = 1u << (q & 31);
    const int qw = q >> 5;
    unsigned long long dsum = 0ull;
    for (int32_t i0 = lo; i0 < hi; i0 += 32) {
      const int32_t i = i0 + lane;
      int32_t row = -1, hrow = -1;
      if (i < hi) {
        const int32_t e = seeds[i];
        if (e < 0 || e >= sa.E_global) {
          a.ctl->err = 1;
        } else {
          if (owner_of(e, sa.world) == sa.rank) row = sa.lidx[e];
          const int32_t hx = sa.hub_index[e];
          if (hx >= 0) hrow = (int32_t)(sa.n_local + hx);
        }
      }
      bool fresh = false, hfresh = false;
      if (row >= 0) {
        const size_t r = (size_t)row * W + qw;
        const uint32_t was = atomicOr(&a.X[r], qb);
        if (e_out && !(was & qb)) dsum += (unsigned long long)(a.indptr[row + 1] - a.indptr[row]);
        if (a.sem != TH_EXACT) atomicOr(&a.V[r], qb);
        if (a.sem == TH_CUMULATIVE) atomicOr(&a.S[r], qb);
        const uint32_t fb = 1u << (row & 31);
        fresh = !(atomicOr(&a.Xf[row >> 5], fb) & fb);
        if (fresh && a.sem != TH_EXACT) atomicOr(&a.Vf[row >> 5], fb);
      }
      if (hrow >= 0) {
        atomicOr(&a.X[(size_t)hrow * W + qw], qb);
        const uint32_t fb = 1u << (hrow & 31);
        hfresh = !(atomicOr(&a.Xf[hrow >> 5], fb) & fb);
      }
      const uint32_t d = fresh ? (uint32_t)(a.indptr[row + 1] - a.indptr[row]) : 0u;
      warp_append_all(fresh, row, d, a.lists, &a.ctl->list_len[0], a.E, &a.ctl->push_cost[0]);
      const uint32_t hd = hfresh ? (uint32_t)(a.indptr[hrow + 1] - a.indptr[hrow]) : 0u;
      warp_append_all(hfresh, hrow, hd, a.lists, &a.ctl->list_len[0], a.E, &a.ctl->push_cost[0]);
    }
    if (e_out) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) dsum += __shfl_xor_sync(TH_FULL, dsum, o);
      if (lane == 0) e_out[q] = (int64_t)dsum;
    }
  }
}

// K2's pair enumeration over CSR slots [lo, hi) of local row u, with the
// owner split of every target
template <int W, int SEM, bool FILTER>
__device__ __forceinline__ void shard_row_pairs(const ShardArgs& sa, int32_t u, int32_t lo,
                                                int32_t hi, WarpAppender& app) {
  const WaveArgs& a = sa.a;
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
    bool fresh = false, rfresh = false;
    int32_t row = 0, v = 0;
    if (p < pairs) {
      const int32_t pos = lo + e;
      uint32_t w = x;
      if (FILTER) w &= a.M[(size_t)a.csr_rel[pos] * W + j];
      if (w) {
        v = a.csr_obj[pos];
        if (sa.world == 1) {  // (one rank: every row is owned, local row = id)
          row = v;
          fresh = local_set<W, SEM>(a, row, j, w);
        } else if (owner_of(v, sa.world) == sa.rank) {
          row = sa.lidx[v];
          fresh = local_set<W, SEM>(a, row, j, w);
        } else {
          rfresh = remote_stage<W>(sa, v, j, w);
        }
      }
    }
    app.add(a, fresh, row);
    warp_append_all(rfresh, v, 0u, sa.olist, sa.olen, sa.E_global, (unsigned long long*)nullptr);
  }
}

template <int W, int SEM, bool FILTER>
__global__ void __launch_bounds__(kThreads) shard_push_light_kernel(ShardArgs sa) {
  const WaveArgs& a = sa.a;
  if (a.ctl->mode[a.h] != 0) return;
  __shared__ int32_t abuf[kThreads / 32][kAppendRun + 32];
  WarpAppender app{abuf[threadIdx.x >> 5]};
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int32_t n = a.ctl->list_len[a.h - 1];
  const int32_t* list = a.lists + a.ctl->list_off[a.h - 1];
  for (int32_t i = gw; i < n; i += nw) {
    const int32_t u = list[i];
    const int32_t lo = a.indptr[u], hi = a.indptr[u + 1];
    if (hi - lo > kHeavyPush) {
      // with a relation filter the edge-count pass already built the heavy list
      if (!FILTER && lane_id() == 0) a.heavy[atomicAdd(&a.ctl->heavy_len, 1)] = u;
      continue;
    }
    shard_row_pairs<W, SEM, FILTER>(sa, u, lo, hi, app);
  }
  app.finish(a);
}

template <int W, int SEM, bool FILTER>
__global__ void __launch_bounds__(kThreads) shard_push_heavy_kernel(ShardArgs sa) {
  const WaveArgs& a = sa.a;
  if (a.ctl->mode[a.h] != 0) return;
  __shared__ int32_t abuf[kThreads / 32][kAppendRun + 32];
  WarpAppender app{abuf[threadIdx.x >> 5]};
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int32_t nh = a.ctl->heavy_len;
  if (nh == 0) return;
  if (nh <= kSmallHeavy) {
    int64_t base = 0;
    for (int32_t i = 0; i < nh; ++i) {
      const int32_t u = a.heavy[i];
      const int32_t lo = a.indptr[u], hi = a.indptr[u + 1];
      const int32_t nc = (hi - lo + kPushChunk - 1) / kPushChunk;
      for (int64_t c = ((gw - base) % nw + nw) % nw; c < nc; c += nw) {
        const int32_t clo = lo + (int32_t)c * kPushChunk;
        shard_row_pairs<W, SEM, FILTER>(sa, u, clo, min(hi, clo + kPushChunk), app);
      }
      base += nc;
    }
    app.finish(a);
    return;
  }
  const int64_t total = a.heavy_off[nh];
  for (int64_t g = gw; g < total; g += nw) {
    int32_t lo_i = 0, hi_i = nh - 1;
    while (lo_i < hi_i) {
      const int32_t mid = (lo_i + hi_i + 1) >> 1;
      if (a.heavy_off[mid] <= g) lo_i = mid;
      else hi_i = mid - 1;
    }
    const int32_t u = a.heavy[lo_i];
    const int32_t lo = a.indptr[u], hi = a.indptr[u + 1];
    const int32_t clo = lo + (int32_t)(g - a.heavy_off[lo_i]) * kPushChunk;
    shard_row_pairs<W, SEM, FILTER>(sa, u, clo, min(hi, clo + kPushChunk), app);
  }
  app.finish(a);
}

// reserve n records in rank d's inbox; returns the first slot (records at or
// beyond the capacity are dropped and flag the receiver's overflow)
__device__ __forceinline__ unsigned long long inbox_reserve(const XPeers& px, int d, int n) {
  return atomicAdd(&px.ctrl(d)->cursor, (unsigned long long)n);
}

__device__ __forceinline__ void inbox_put(const XPeers& px, int d, unsigned long long at, uint64_t key,
                                          uint32_t bits) {
  if ((int64_t)at < px.cap) {
    px.keys(d)[at] = key;
    px.bits(d)[at] = bits;
  } else {
    px.ctrl(d)->overflow = 1u;
  }
}

// staged rows -> records ((row_at_owner * W + word), bits) written straight
// into the owners' inboxes (warp-aggregated: one remote atomic per (warp,
// owner)); staged rows and flags are cleared behind
template <int W>
__global__ void __launch_bounds__(kThreads) shard_send_kernel(ShardArgs sa) {
  if (sa.a.ctl->mode[sa.a.h] != 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int32_t n = *sa.olen;
  for (int64_t base = gw * 32; base < n; base += nw * 32) {
    const int64_t i = base + lane;
    int32_t v = -1, dest = -1;
    uint32_t words[W];
    int nzc = 0;
    if (i < n) {
      v = sa.olist[i];
      dest = owner_of(v, sa.world);
#pragma unroll
      for (int j = 0; j < W; ++j) {
        words[j] = sa.O[(size_t)v * W + j];
        nzc += words[j] != 0u;
      }
    }
    unsigned pending = __ballot_sync(TH_FULL, dest >= 0 && nzc > 0);
    while (pending) {
      // one owner per round: the lanes bound for it append together
      const int d = __shfl_sync(TH_FULL, dest, __ffs(pending) - 1);
      const bool mine = dest == d && nzc > 0;
      pending &= ~__ballot_sync(TH_FULL, mine);
      int incl = mine ? nzc : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(TH_FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const int tot = __shfl_sync(TH_FULL, incl, 31);
      unsigned long long b0 = 0;
      if (lane == 0) {
        b0 = inbox_reserve(sa.px, d, tot);
        if (d != sa.rank) atomicAdd(&sa.a.ctl->sent[sa.a.h], (unsigned long long)tot);
      }
      b0 = __shfl_sync(TH_FULL, b0, 0);
      if (mine) {
        unsigned long long o = b0 + (unsigned long long)(incl - nzc);
        const uint64_t key0 = (uint64_t)sa.lidx[v] * W;
#pragma unroll
        for (int j = 0; j < W; ++j)
          if (words[j]) inbox_put(sa.px, d, o++, key0 + j, words[j]);
      }
    }
    if (v >= 0) {
#pragma unroll
      for (int j = 0; j < W; ++j) sa.O[(size_t)v * W + j] = 0u;
      atomicAnd(&sa.Of[v >> 5], ~(1u << (v & 31)));
    }
  }
}

// this rank's inbox records -> local test-and-set, appended to the hop's list
template <int W, int SEM>
__global__ void __launch_bounds__(kThreads) shard_absorb_kernel(ShardArgs sa) {
  const WaveArgs& a = sa.a;
  if (a.ctl->mode[a.h] != 0) return;
  const int lane = threadIdx.x & 31;
  __shared__ int32_t abuf[kThreads / 32][kAppendRun + 32];
  WarpAppender app{abuf[threadIdx.x >> 5]};
  const XCtrl* xc = sa.px.ctrl(sa.rank);
  const int64_t n = (int64_t)min(xc->cursor, (unsigned long long)sa.px.cap);
  const uint64_t* keys = sa.px.keys(sa.rank);
  const uint32_t* bits = sa.px.bits(sa.rank);
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = gw * 32; base < n; base += nw * 32) {
    const int64_t i = base + lane;
    bool fresh = false;
    int32_t row = 0;
    if (i < n) {
      const uint64_t key = keys[i];
      row = (int32_t)(key / W);
      if (key / W >= (uint64_t)sa.n_local) {
        a.ctl->err = 2;  // malformed record: not an owned row
        row = 0;
      } else {
        fresh = local_set<W, SEM>(a, row, (int)(key % W), bits[i]);
      }
    }
    app.add(a, fresh, row);
  }
  app.finish(a);
}

// hop h begins: the ranks' published frontier costs decide push or pull
// (every rank sees the same costs, so all choose alike); list segment h
__global__ void shard_begin_hop_kernel(ShardArgs sa, int h, int64_t T_global, double pull_divisor,
                                       int can_pull) {
  Ctl* ctl = sa.a.ctl;
  const int32_t prev = ctl->list_len[h - 1];
  ctl->list_off[h] = ctl->list_off[h - 1] + prev;
  ctl->list_len[h] = 0;
  ctl->push_cost[h] = 0;
  ctl->heavy_len = 0;
  ctl->olen = 0;
  const XCtrl* xc = sa.px.ctrl(sa.rank);
  unsigned long long cost = 0ull;
  for (int d = 0; d < sa.world; ++d) cost += xc->cost[d];
  const int pull = can_pull && pull_divisor > 0 && (double)cost * pull_divisor > (double)T_global;
  ctl->mode[h] = pull;
  ctl->dense[h] = pull && (double)cost * 2.0 > (double)T_global;
  if (pull) ctl->pull_hops++;
  else ctl->push_hops++;
}

// this rank's frontier cost of list segment `seg` onto every rank's board
__global__ void shard_publish_cost_kernel(ShardArgs sa, int seg) {
  const int d = threadIdx.x;
  if (d < sa.world) sa.px.ctrl(d)->cost[sa.rank] = sa.a.ctl->push_cost[seg];
}

// the inbox is consumed: empty it for the peers' next sends
__global__ void shard_inbox_reset_kernel(ShardArgs sa) {
  if (threadIdx.x == 0) sa.px.ctrl(sa.rank)->cursor = 0ull;
}

// owners write their hubs' next-layer rows onto every rank's hub board
// ([n_hubs][W]); each hub has exactly one owner, so every board ends up
// holding every hub's row with no reduction
template <int W>
__global__ void shard_hub_out_kernel(ShardArgs sa) {
  const int64_t n = sa.n_hubs * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = i / W;
    const int j = (int)(i % W);
    const int32_t v = sa.hub_ids[h];
    if (owner_of(v, sa.world) != sa.rank) continue;
    const uint32_t w = sa.a.N[(size_t)sa.lidx[v] * W + j];
    for (int d = 0; d < sa.world; ++d) sa.px.hubs(d)[i] = w;
  }
}

// install the board's hub rows as next-layer hub slice rows (frontier only:
// a hub's visited bits stay with its owner)
template <int W>
__global__ void shard_hub_in_kernel(ShardArgs sa) {
  const WaveArgs& a = sa.a;
  const uint32_t* rows = sa.px.hubs(sa.rank);
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t base = gw * 32; base < sa.n_hubs; base += nw * 32) {
    const int64_t h = base + lane;
    bool any = false;
    int32_t row = 0;
    if (h < sa.n_hubs) {
      row = (int32_t)(sa.n_local + h);
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const uint32_t w = rows[h * W + j];
        a.N[(size_t)row * W + j] = w;
        any |= w != 0u;
      }
      if (any) {
        const uint32_t fb = 1u << (row & 31);
        any = !(atomicOr(&a.Nf[row >> 5], fb) & fb);
      }
    }
    const uint32_t d = any ? (uint32_t)(a.indptr[row + 1] - a.indptr[row]) : 0u;
    warp_append_all(any, row, d, a.lists + a.ctl->list_off[a.h], &a.ctl->list_len[a.h], a.E,
                    &a.ctl->push_cost[a.h]);
  }
}

// mark the local triples of the rank and their local row keys, in tid order
__global__ void shard_select_kernel(const int32_t* __restrict__ subj, int64_t T,
                                    const int32_t* __restrict__ lidx,
                                    const int32_t* __restrict__ hub_index, int64_t n_local,
                                    int32_t rank, int32_t world, int32_t* key) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = subj[t];
    const int32_t hx = hub_index[u];
    int32_t k = -1;
    if (hx >= 0) {
      if (owner_of(t, world) == rank) k = (int32_t)(n_local + hx);
    } else if (owner_of(u, world) == rank) {
      k = lidx[u];
    }
    key[t] = k;
  }
}

// ordered compaction of the selected triples (key >= 0) via per-block scans
__global__ void __launch_bounds__(kCompactThreads) shard_count_kernel(const int32_t* __restrict__ key,
                                                                       int64_t T, int32_t* bcount) {
  __shared__ int ws[32];
  const int64_t t0 = (int64_t)blockIdx.x * kCompactWords + threadIdx.x * kCompactPerThread;
  int c = 0;
#pragma unroll
  for (int i = 0; i < kCompactPerThread; ++i) c += (t0 + i < T && key[t0 + i] >= 0);
  int total;
  block_excl_scan(c, ws, &total);
  if (threadIdx.x == 0) bcount[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kCompactThreads) shard_gather_kernel(
    const int32_t* __restrict__ key, int64_t T, const int32_t* __restrict__ boff,
    const int32_t* __restrict__ rel, const int32_t* __restrict__ obj, int32_t* okey, int32_t* orel,
    int32_t* oobj, int32_t* otid) {
  __shared__ int ws[32];
  const int64_t t0 = (int64_t)blockIdx.x * kCompactWords + threadIdx.x * kCompactPerThread;
  int c = 0;
#pragma unroll
  for (int i = 0; i < kCompactPerThread; ++i) c += (t0 + i < T && key[t0 + i] >= 0);
  int total;
  int o = boff[blockIdx.x] + block_excl_scan(c, ws, &total);
  for (int i = 0; i < kCompactPerThread; ++i) {
    const int64_t t = t0 + i;
    if (t < T && key[t] >= 0) {
      okey[o] = key[t];
      orel[o] = rel[t];
      oobj[o] = obj[t];
      otid[o] = (int32_t)t;
      ++o;
    }
  }
}

// ---------------------------------------------------------------------------
// Pull hops across partitions (dense frontiers).  Instead of pushing every
// frontier edge's candidates to the target's owner, every rank writes its
// owned frontier rows -- records ((gid * W + word), bits) -- into every
// rank's inbox (an all-gather over peer memory); each rank stages them into
// a global-indexed copy of the frontier (the push staging matrix O, empty
// between hops) and pulls for the entities it owns over its in-edge CSR
// (global sources).  Hub frontier rows are already replicated and are
// copied in locally.  On a single rank the frontier is its own X (global
// rows = local rows) and nothing is staged.

// in-edges of owned objects: key = object's local row, or -1
__global__ void shard_select_in_kernel(const int32_t* __restrict__ obj, int64_t T,
                                       const int32_t* __restrict__ lidx, int32_t rank,
                                       int32_t world, int32_t* key) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = obj[t];
    key[t] = owner_of(v, world) == rank ? lidx[v] : -1;
  }
}

// owned frontier rows of list segment `seg` -> records in every rank's inbox
template <int W>
__global__ void __launch_bounds__(kThreads) shard_frontier_send_kernel(ShardArgs sa, int seg,
                                                                       const int32_t* __restrict__ l2g) {
  const WaveArgs& a = sa.a;
  if (a.ctl->mode[a.h] != 1) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int32_t n = a.ctl->list_len[seg];
  const int32_t* list = a.lists + a.ctl->list_off[seg];
  for (int64_t base = gw * 32; base < n; base += nw * 32) {
    const int64_t i = base + lane;
    int32_t row = -1;
    uint32_t words[W];
    int nzc = 0;
    if (i < n) {
      row = list[i];
      if (row < sa.n_local) {
#pragma unroll
        for (int j = 0; j < W; ++j) {
          words[j] = a.X[(size_t)row * W + j];
          nzc += words[j] != 0u;
        }
      } else {
        row = -1;  // hub rows: every rank holds them already
      }
    }
    int incl = nzc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(TH_FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int tot = __shfl_sync(TH_FULL, incl, 31);
    if (!tot) continue;
    const uint64_t key0 = row >= 0 ? (uint64_t)l2g[row] * W : 0ull;
    for (int d = 0; d < sa.world; ++d) {
      unsigned long long b0 = 0;
      if (lane == 0) {
        b0 = inbox_reserve(sa.px, d, tot);
        if (d != sa.rank) atomicAdd(&a.ctl->sent[a.h], (unsigned long long)tot);
      }
      b0 = __shfl_sync(TH_FULL, b0, 0);
      if (row >= 0) {
        unsigned long long o = b0 + (unsigned long long)(incl - nzc);
#pragma unroll
        for (int j = 0; j < W; ++j)
          if (words[j]) inbox_put(sa.px, d, o++, key0 + j, words[j]);
      }
    }
  }
}

// gathered records (and the local hub frontier rows) -> global staging O, Of
template <int W>
__global__ void shard_gather_frontier_kernel(ShardArgs sa, int seg) {
  const WaveArgs& a = sa.a;
  if (a.ctl->mode[a.h] != 1) return;
  const int64_t n = (int64_t)min(sa.px.ctrl(sa.rank)->cursor, (unsigned long long)sa.px.cap);
  const uint64_t* keys = sa.px.keys(sa.rank);
  const uint32_t* bits = sa.px.bits(sa.rank);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[i];
    const int64_t g = (int64_t)(key / W);
    sa.O[key] = bits[i];
    atomicOr(&sa.Of[g >> 5], 1u << (g & 31));
  }
  // hub rows of the segment (rows >= n_local), one thread per (row, word)
  const int32_t nl = a.ctl->list_len[seg];
  const int32_t* list = a.lists + a.ctl->list_off[seg];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)nl * W;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t row = list[i / W];
    if (row < sa.n_local) continue;
    const int j = (int)(i % W);
    const int32_t g = sa.hub_ids[row - sa.n_local];
    const uint32_t w = a.X[(size_t)row * W + j];
    if (w) {
      sa.O[(size_t)g * W + j] = w;
      atomicOr(&sa.Of[g >> 5], 1u << (g & 31));
    }
  }
}

// undo the staging: zero the gathered words, the hub rows' words and their
// flag words (every staged entity is cleared here, so whole flag words can go)
template <int W>
__global__ void shard_clear_frontier_kernel(ShardArgs sa, int seg) {
  const WaveArgs& a = sa.a;
  if (a.ctl->mode[a.h] != 1) return;
  const int64_t n = (int64_t)min(sa.px.ctrl(sa.rank)->cursor, (unsigned long long)sa.px.cap);
  const uint64_t* keys = sa.px.keys(sa.rank);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[i];
    sa.O[key] = 0u;
    sa.Of[(key / W) >> 5] = 0u;
  }
  const int32_t nl = a.ctl->list_len[seg];
  const int32_t* list = a.lists + a.ctl->list_off[seg];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)nl * W;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t row = list[i / W];
    if (row < sa.n_local) continue;
    const int32_t g = sa.hub_ids[row - sa.n_local];
    sa.O[(size_t)g * W + (i % W)] = 0u;
    sa.Of[g >> 5] = 0u;
  }
}
