// Part of engine.cu (included inside namespace th::{anonymous}); kept in its
// own file so the kernel can be revised in isolation.
#pragma once

// ------------------------------------------------------------ pull hop

// VEC words per lane, LPR lanes per entity row, GPW rows (groups) per warp
template <int W>
struct RowShape {
  static constexpr int VEC = W >= 4 ? 4 : W;
  static constexpr int LPR = W / VEC;
  static constexpr int GPW = 32 / LPR;
};

template <int VEC>
__device__ __forceinline__ void ld_words(const uint32_t* p, uint32_t (&o)[VEC]) {
  if constexpr (VEC == 4) {
    const uint4 t = *reinterpret_cast<const uint4*>(p);
    o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
  } else if constexpr (VEC == 2) {
    const uint2 t = *reinterpret_cast<const uint2*>(p);
    o[0] = t.x; o[1] = t.y;
  } else {
    o[0] = *p;
  }
}

// read-only path for data the kernel never writes (frontier rows, masks)
template <int VEC>
__device__ __forceinline__ void ldg_words(const uint32_t* p, uint32_t (&o)[VEC]) {
  if constexpr (VEC == 4) {
    const uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
    o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
  } else if constexpr (VEC == 2) {
    const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
    o[0] = t.x; o[1] = t.y;
  } else {
    o[0] = __ldg(p);
  }
}

template <int VEC>
__device__ __forceinline__ void st_words(uint32_t* p, const uint32_t (&v)[VEC]) {
  if constexpr (VEC == 4) {
    *reinterpret_cast<uint4*>(p) = make_uint4(v[0], v[1], v[2], v[3]);
  } else if constexpr (VEC == 2) {
    *reinterpret_cast<uint2*>(p) = make_uint2(v[0], v[1]);
  } else {
    *p = v[0];
  }
}

// Pull hop over the static in-edge items of the reverse CSR.  Each lane
// group (LPR lanes, 16 B per lane) owns one item and ORs the frontier rows of
// its active in-neighbours (4 rows in flight per group, GPW groups per warp,
// all in lockstep so the warp stays convergent).  A group stops early once
// every live query has visited or reached the entity.  Whole in-rows are
// finished with plain stores; rows split over several items merge with
// atomicOr (the union of the pieces is exactly R_h & ~V_{h-1}).
// (newly reached entities are appended through a WarpAppender)
template <int W, int SEM, bool FILTER, bool SCREEN>
__global__ void __launch_bounds__(kThreads) pull_kernel(WaveArgs a) {
  if (a.ctl->mode[a.h] != 1) return;
  // (beside the two-phase pull's kernels: dense hops only)
  if (a.pull_only_dense && a.ctl->dense[a.h] == 0) return;
  const bool dense = a.ctl->dense[a.h] != 0;
  using RS = RowShape<W>;
  constexpr int VEC = RS::VEC, LPR = RS::LPR, GPW = RS::GPW;
  // nth-set-bit table for the LPR-bit group masks: entry m holds the
  // positions of m's set bits, ascending, one per nibble (replaces __fns,
  // a software loop)
  __shared__ uint32_t nth_bit[LPR >= 4 ? (1 << LPR) : 1];
  __shared__ int32_t abuf[kThreads / 32][kAppendRun + 32];
  if constexpr (LPR >= 4) {
    for (int m = threadIdx.x; m < (1 << LPR); m += blockDim.x) {
      uint32_t e = 0u;
      int n = 0;
      for (int b = 0; b < LPR; ++b)
        if ((m >> b) & 1) e |= (uint32_t)b << (4 * n++);
      nth_bit[m] = e;
    }
    __syncthreads();
  }
  WarpAppender app{abuf[threadIdx.x >> 5]};
  const unsigned lane = lane_id();
  const int part = (int)lane % LPR, grp = (int)lane / LPR;
  const unsigned gbits = (LPR == 32 ? TH_FULL : ((1u << LPR) - 1u)) << (grp * LPR);
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t valid[VEC];
#pragma unroll
  for (int c = 0; c < VEC; ++c) valid[c] = valid_word(part * VEC + c, a.nq);
  const int64_t n = a.n_items_dev ? (int64_t)*a.n_items_dev : a.n_items;
  // SCREEN (graphs of low mean in-degree, chosen on the host): items are
  // first screened 32 at a time, one per lane -- an item takes part only if
  // one of its in-edges comes from the frontier (any edge when the hop is
  // dense).  At C4 (1.6 in-edges per entity, ~90% of items without a
  // frontier in-neighbour at hop 3) this replaces a lane group's item /
  // visited-row / flag round trips per item with one screening pass, and
  // the visited row is loaded only for items that can change (C4 k=3 13.8
  // -> 11.3 ms); the lane groups then take the surviving items GPW at a
  // time.  Without SCREEN each lane group takes the next item directly
  // (high in-degree: C2's screened pull was 12% slower).
  constexpr int64_t kStep = SCREEN ? 32 : GPW;
  for (int64_t base = warp * kStep; base < n; base += nwarps * kStep) {
    int32_t s_vv = 0, s_lo = 0, s_hi = 0;
    bool s_act = false;
    if constexpr (SCREEN) {
      const int64_t it = base + lane;
      if (it < n) {
        s_vv = __ldg(a.item_v + it);
        s_lo = __ldg(a.item_lo + it);
        s_hi = __ldg(a.item_hi + it);
        s_act = s_hi > s_lo;
        if (s_act && !dense) {
          s_act = false;
          for (int32_t e = s_lo; e < s_hi; ++e) {
            const int32_t u = __ldg(a.rsrc + e);
            if ((__ldg(a.Xf + (u >> 5)) >> (u & 31)) & 1u) {
              s_act = true;
              break;
            }
          }
        }
      }
    }
    unsigned am = SCREEN ? __ballot_sync(TH_FULL, s_act) : 1u;
    while (am) {
    bool live;
    int32_t vv = 0, lo = 0, hi = 0;
    if constexpr (SCREEN) {
      // group grp takes the grp-th surviving item of this round
      const int navail = __popc(am);
      const int src_lane = grp < navail ? select_bit(am, grp) : 0;
      live = grp < navail;
      for (int r = 0; r < GPW && am; ++r) am &= am - 1u;
      vv = __shfl_sync(TH_FULL, s_vv, src_lane);
      lo = __shfl_sync(TH_FULL, s_lo, src_lane);
      hi = __shfl_sync(TH_FULL, s_hi, src_lane);
      if (!live) vv = lo = hi = 0;
    } else {
      am = 0u;
      const int64_t it = base + grp;
      live = it < n;
      if (live) {
        vv = a.item_v[it];
        lo = a.item_lo[it];
        hi = a.item_hi[it];
      }
    }
    const bool split = vv < 0;
    const int32_t v = split ? ~vv : vv;
    const size_t row = (size_t)v * W + part * VEC;
    uint32_t seen[VEC], acc[VEC];
#pragma unroll
    for (int c = 0; c < VEC; ++c) {
      seen[c] = 0u;
      acc[c] = 0u;
    }
    // (a row no earlier layer reached has an all-zero visited row: its Vf
    // bit says so without the 4W-byte load -- at C4's hop 3 ~80% of the
    // screened items)
    if (SEM != TH_EXACT && live && ((__ldcg(a.Vf + (v >> 5)) >> (v & 31)) & 1u))
      ld_words<VEC>(a.V + row, seen);
    bool sat = true;
#pragma unroll
    for (int c = 0; c < VEC; ++c) sat &= (seen[c] & valid[c]) == valid[c];
    // the full-mask ballot must run on every lane (no short-circuit around it)
    const bool group_sat = (__ballot_sync(TH_FULL, sat) & gbits) == gbits;
    bool done = !live || (SEM != TH_EXACT && group_sat);
    const int len = done ? 0 : hi - lo;
    int maxlen = len;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(TH_FULL, maxlen, o));
    if constexpr (LPR >= 4) {
      // LPR in-edges per step: lane p of a group loads edge e0+p and tests
      // its frontier flag (coalesced, no redundant loads), the group's
      // active edges are compacted with one __fns per lane, then their
      // frontier rows are loaded back to back (up to LPR loads in flight)
      // the next step's in-edge sources are loaded one step ahead, so their
      // latency hides behind this step's flag and row loads
      int32_t u_nx = 0;
      uint32_t rr_nx = 0u;
      if (!done && part < len) {
        u_nx = __ldg(a.rsrc + lo + part);
        if (FILTER) rr_nx = (uint32_t)__ldg(a.rrel + lo + part);
      }
      for (int e0 = 0; e0 < maxlen; e0 += LPR) {
        const int ei = e0 + part;
        bool act = !done && ei < len;
        const int32_t u = u_nx;
        const uint32_t rr = rr_nx;
        const int en = ei + LPR;
        if (!done && en < len) {
          u_nx = __ldg(a.rsrc + lo + en);
          if (FILTER) rr_nx = (uint32_t)__ldg(a.rrel + lo + en);
        }
        int cnt;
        int32_t uc;
        uint32_t rc;
        if (dense) {
          // most in-edges come from the frontier: gather every source row
          // (a non-frontier row is zero) instead of testing flags first,
          // which saves a dependent L2 round trip and the compaction
          cnt = done ? 0 : min(max(len - e0, 0), LPR);
          uc = u;
          rc = rr;
        } else {
          if (act) act = (__ldg(a.Xf + (u >> 5)) >> (u & 31)) & 1u;
          const unsigned gm = (__ballot_sync(TH_FULL, act) & gbits) >> (grp * LPR);
          cnt = __popc(gm);
          const int srcp = part < cnt ? (int)((nth_bit[gm] >> (4 * part)) & 0xfu) : 0;
          uc = __shfl_sync(TH_FULL, u, grp * LPR + srcp);
          rc = FILTER ? __shfl_sync(TH_FULL, rr, grp * LPR + srcp) : 0u;
        }
        // steps where no group of the warp found a frontier in-edge skip the
        // (fully unrolled, up to LPR loads in flight) row gathers entirely;
        // bounding the unrolled loop by the busiest group measured slower at
        // C4 (serialised or branchy loads)
        const int maxcnt = (int)__reduce_max_sync(TH_FULL, (unsigned)cnt);
        auto take = [&](int it) {
          const int32_t uu = __shfl_sync(TH_FULL, uc, grp * LPR + it);
          const uint32_t r2 = FILTER ? __shfl_sync(TH_FULL, rc, grp * LPR + it) : 0u;
          if (it < cnt) {
            uint32_t x[VEC];
            ldg_words<VEC>(a.X + (size_t)uu * W + part * VEC, x);
            if (FILTER) {
              uint32_t m[VEC];
              ldg_words<VEC>(a.M + (size_t)r2 * W + part * VEC, m);
#pragma unroll
              for (int c = 0; c < VEC; ++c) x[c] &= m[c];
            }
#pragma unroll
            for (int c = 0; c < VEC; ++c) acc[c] |= x[c];
          }
        };
        if (maxcnt > 0) {
#pragma unroll
          for (int it = 0; it < LPR; ++it) take(it);
        }
        bool full = true;
#pragma unroll
        for (int c = 0; c < VEC; ++c) full &= ((acc[c] | seen[c]) & valid[c]) == valid[c];
        if ((__ballot_sync(TH_FULL, full) & gbits) == gbits) done = true;
        if (__all_sync(TH_FULL, done)) break;
      }
    } else {
      for (int e0 = 0; e0 < maxlen; e0 += 4) {
        int32_t u[4];
        uint32_t rr[4];
        bool act[4];
  #pragma unroll
        for (int k = 0; k < 4; ++k) {
          act[k] = !done && e0 + k < len;
          u[k] = act[k] ? __ldg(a.rsrc + lo + e0 + k) : 0;
          rr[k] = (FILTER && act[k]) ? (uint32_t)__ldg(a.rrel + lo + e0 + k) : 0u;
        }
  #pragma unroll
        for (int k = 0; k < 4; ++k)
          if (act[k]) act[k] = (__ldg(a.Xf + (u[k] >> 5)) >> (u[k] & 31)) & 1u;
  #pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (act[k]) {
            uint32_t x[VEC];
            ldg_words<VEC>(a.X + (size_t)u[k] * W + part * VEC, x);
            if (FILTER) {
              uint32_t m[VEC];
              ldg_words<VEC>(a.M + (size_t)rr[k] * W + part * VEC, m);
  #pragma unroll
              for (int c = 0; c < VEC; ++c) x[c] &= m[c];
            }
  #pragma unroll
            for (int c = 0; c < VEC; ++c) acc[c] |= x[c];
          }
        }
        bool full = true;
  #pragma unroll
        for (int c = 0; c < VEC; ++c) full &= ((acc[c] | seen[c]) & valid[c]) == valid[c];
        if ((__ballot_sync(TH_FULL, full) & gbits) == gbits) done = true;
        if (__all_sync(TH_FULL, done)) break;
      }
    }
    uint32_t nb[VEC];
    bool any = false;
#pragma unroll
    for (int c = 0; c < VEC; ++c) {
      nb[c] = acc[c] & ~seen[c] & valid[c];
      any |= nb[c] != 0u;
    }
    any = (__ballot_sync(TH_FULL, any) & gbits) != 0u;
    bool fresh = false;
    if (live && any) {
      // (FRONTIER's last hop skips the visited-row update: the wave ends
      // with the layer, and the visited matrix is only cleared after it)
      if (!split) {
        st_words<VEC>(a.N + row, nb);
        if (SEM != TH_EXACT && !a.last_frontier) {
          uint32_t nv[VEC];
#pragma unroll
          for (int c = 0; c < VEC; ++c) nv[c] = seen[c] | nb[c];
          st_words<VEC>(a.V + row, nv);
        }
        // (a whole row is reached by its one item only: set its flags
        // without waiting for the old value)
        if (part == 0) {
          const uint32_t fb = 1u << (v & 31);
          atomicOr(&a.Nf[v >> 5], fb);
          if (SEM != TH_EXACT) atomicOr(&a.Vf[v >> 5], fb);
          fresh = true;
        }
      } else {
#pragma unroll
        for (int c = 0; c < VEC; ++c) {
          if (nb[c]) {
            atomicOr(a.N + row + c, nb[c]);
            if (SEM != TH_EXACT && !a.last_frontier) atomicOr(a.V + row + c, nb[c]);
          }
        }
        if (part == 0) fresh = flag_next(a, v);
      }
    }
    app.add(a, fresh, v);
    }
  }
  app.finish(a);
}


// Two-phase pull (pull_screen 2).  Phase 1, pull_screen_kernel, finds the
// in-edges of the hop that come from the frontier; phase 2 gathers them.
//
// The in-kernel screen (SCREEN = true) walks an item's in-edges on one lane,
// two dependent loads (source, frontier flag) per step, and the lane groups
// then redo the flag tests before their row loads: a 5-deep dependent chain
// per item (item, visited flag, sources, flags, rows), with 4 items per warp
// in flight (C4 hop 3: 13M surviving items, 2.3 ms, 44% issue, DRAM 16%).
//   non-dense hops: pull_screen_edges_kernel streams the in-edges (source
//     and target row of each, rdst) and compacts the frontier ones as
//     (vv, u[, rel]) -- a whole row's entries stay consecutive -- through a
//     per-warp shared run stored with one global atomic per >= 128 entries;
//     pull_edges_kernel gathers them: one dependent step (the entry) in
//     front of the row loads instead of four.
//   dense hops (every in-edge is taken): pull_kernel<.., SCREEN = false>
//     over the static items.
// ctl->pull_items[h] counts the entries.
constexpr int kScreenRun = 32;

// non-dense hops: the frontier in-edges as (vv, u[, rel]).  Each warp
// streams a contiguous range of 32-edge chunks (source and target row of
// each edge, coalesced; the frontier flag from the L2-resident bitmap),
// software-pipelined three chunks deep: chunk c+3's edges and chunk c+2's
// flag words are loaded while chunk c is compacted.  A whole row's in-edges
// (vv >= 0, at most kPullChunk) stay consecutive in the output: a warp
// skips the leading edges of a row that started before its range and takes
// the rest of its own last row past the range end; a flush stores the run
// up to the start of a row still open at the chunk boundary.  Split rows'
// edges may fall anywhere (their rows merge with atomics).
template <bool FILTER>
__global__ void __launch_bounds__(kThreads) pull_screen_edges_kernel(WaveArgs a, int32_t* cv,
                                                                     int32_t* cu, int32_t* cr) {
  if (a.ctl->mode[a.h] != 1 || a.ctl->dense[a.h] != 0) return;
  constexpr int kRun = 128;  // entries per counter atomic
  constexpr int kBuf = kRun + 2 * 32;  // < kRun left + a chunk + a row's continuation
  __shared__ int32_t sb[kThreads / 32][FILTER ? 3 : 2][kBuf];
  const int wib = threadIdx.x >> 5;
  int32_t* bv = sb[wib][0];
  int32_t* bu = sb[wib][1];
  int32_t* br = sb[wib][FILTER ? 2 : 1];
  int fill = 0;
  const unsigned lane = lane_id();
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t T = a.T;
  const int64_t nch = (T + 31) / 32;
  const int64_t per = (nch + nwarps - 1) / nwarps;
  const int64_t c_begin = warp * per;
  const int64_t c_end = c_begin + per < nch ? c_begin + per : nch;
  if (c_begin >= c_end) return;
  int32_t* count = &a.ctl->pull_items[a.h];
  auto ld = [&](int64_t c, int32_t& d, int32_t& u) {
    const int64_t e = c * 32 + lane;
    d = INT32_MIN;
    u = 0;
    if (e < T) {
      d = __ldg(a.rdst + e);
      u = __ldg(a.rsrc + e);
    }
  };
  auto append = [&](bool take, int32_t v, int32_t u, int32_t r) {
    const unsigned m = __ballot_sync(TH_FULL, take);
    if (take) {
      const int p = fill + __popc(m & lanemask_lt());
      bv[p] = v;
      bu[p] = u;
      if (FILTER) br[p] = r;
    }
    fill += __popc(m);
  };
  // stores run [0, n) and moves [n, fill) to the front
  auto flush = [&](int n) {
    __syncwarp();
    int32_t at = 0;
    if (lane == 0) at = atomicAdd(count, n);
    at = __shfl_sync(TH_FULL, at, 0);
    for (int i = (int)lane; i < n; i += 32) {
      cv[at + i] = bv[i];
      cu[at + i] = bu[i];
      if (FILTER) cr[at + i] = br[i];
    }
    __syncwarp();
    const int rest = fill - n;
    int32_t tv = 0, tu = 0, tr = 0;
    if ((int)lane < rest) {
      tv = bv[n + lane];
      tu = bu[n + lane];
      if (FILTER) tr = br[n + lane];
    }
    __syncwarp();
    if ((int)lane < rest) {
      bv[lane] = tv;
      bu[lane] = tu;
      if (FILTER) br[lane] = tr;
    }
    fill = rest;
    __syncwarp();
  };
  auto xf = [&](int32_t d, int32_t u) { return d != INT32_MIN ? __ldg(a.Xf + (u >> 5)) : 0u; };
  int32_t d0, u0, d1, u1, d2, u2, d3, u3;
  ld(c_begin, d0, u0);
  ld(c_begin + 1, d1, u1);
  ld(c_begin + 2, d2, u2);
  uint32_t x0 = xf(d0, u0), x1 = xf(d1, u1), x2;
  int32_t last = c_begin > 0 ? __ldg(a.rdst + c_begin * 32 - 1) : INT32_MIN;
  bool first = true;
  for (int64_t c = c_begin; c < c_end; ++c) {
    x2 = xf(d2, u2);
    ld(c + 3, d3, u3);
    int32_t pd = __shfl_up_sync(TH_FULL, d0, 1);
    if (lane == 0) pd = last;
    int lead = 0;
    if (first) {
      // a whole row that started before the range: the previous warp's
      const unsigned chg = __ballot_sync(TH_FULL, d0 != pd);
      if (__shfl_sync(TH_FULL, d0, 0) >= 0 && !(chg & 1u)) lead = chg ? __ffs(chg) - 1 : 32;
      first = false;
    }
    const bool take = (int)lane >= lead && d0 != INT32_MIN && ((x0 >> (u0 & 31)) & 1u);
    int32_t r = 0;
    if (FILTER && take) r = (int32_t)__ldg(a.rrel + c * 32 + lane);
    append(take, d0, u0, r);
    last = __shfl_sync(TH_FULL, d0, 31);
    const bool open = last >= 0 && __shfl_sync(TH_FULL, d1, 0) == last;  // row runs into c+1
    if (c + 1 == c_end && open) {
      // the range's last whole row: its edges in the next chunk
      const unsigned ne = __ballot_sync(TH_FULL, d1 != last);
      const int cont = ne ? __ffs(ne) - 1 : 32;
      const bool t2 = (int)lane < cont && ((x1 >> (u1 & 31)) & 1u);
      int32_t r2 = 0;
      if (FILTER && t2) r2 = (int32_t)__ldg(a.rrel + (c + 1) * 32 + lane);
      append(t2, last, u1, r2);
    } else if (fill >= kRun) {
      // keep a row still open at the boundary with its next entries
      int tail = 0;
      if (open) {
        const bool ok = (int)lane < fill && bv[fill - 1 - (int)lane] == last;
        const unsigned nm = __ballot_sync(TH_FULL, !ok);
        tail = nm ? __ffs(nm) - 1 : 32;
      }
      if (fill - tail > 0) flush(fill - tail);
    }
    d0 = d1;
    u0 = u1;
    x0 = x1;
    d1 = d2;
    u1 = u2;
    x1 = x2;
    d2 = d3;
    u2 = u3;
  }
  if (fill) flush(fill);
}

// Two-phase pull, phase 2 over compacted frontier in-edges (vv, u[, rel])
// of a non-dense hop.  A warp takes a window of 32 entries; runs of equal
// vv are segments (one target row each), handed to the lane groups GPW at a
// time.  A whole row's run (vv >= 0, at most kPullChunk entries) belongs to
// the window it starts in, which reads up to 31 entries past its end; split
// rows' runs are cut at window edges and merged with atomicOr.  Per segment:
// the frontier rows of its sources are loaded 4 at a time with the visited
// row, then N (and V) are written; a whole row is flagged with a
// non-returning atomic (only its own segment can reach it this hop).
template <int W, int SEM, bool FILTER, int SPG = 2>
__global__ void __launch_bounds__(kThreads) pull_edges_kernel(WaveArgs a, const int32_t* __restrict__ cv,
                                                              const int32_t* __restrict__ cu,
                                                              const int32_t* __restrict__ cr) {
  if (a.ctl->mode[a.h] != 1 || a.ctl->dense[a.h] != 0) return;
  using RS = RowShape<W>;
  constexpr int VEC = RS::VEC, LPR = RS::LPR, GPW = RS::GPW;
  __shared__ int32_t abuf[kThreads / 32][kAppendRun + 32];
  __shared__ int32_t segs[kThreads / 32][33];
  WarpAppender app{abuf[threadIdx.x >> 5]};
  int32_t* seg = segs[threadIdx.x >> 5];
  const unsigned lane = lane_id();
  const int part = (int)lane % LPR, grp = (int)lane / LPR;
  const unsigned gbits = (LPR == 32 ? TH_FULL : ((1u << LPR) - 1u)) << (grp * LPR);
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t valid[VEC];
#pragma unroll
  for (int c = 0; c < VEC; ++c) valid[c] = valid_word(part * VEC + c, a.nq);
  const int64_t n = a.ctl->pull_items[a.h];
  // a window's loads, issued one window ahead: its entries, the 32 after it
  // (the continuation of its last run) and the entry before it
  int32_t ev, eu, er, ev2, eu2, er2, pv;
  auto ld = [&](int64_t b) {
    const int64_t i = b + lane, j = i + 32;
    ev = ev2 = pv = INT32_MIN;
    eu = eu2 = er = er2 = 0;
    if (i < n) {
      ev = __ldg(cv + i);
      eu = __ldg(cu + i);
      if (FILTER) er = __ldg(cr + i);
    }
    if (j < n) {
      ev2 = __ldg(cv + j);
      eu2 = __ldg(cu + j);
      if (FILTER) er2 = __ldg(cr + j);
    }
    if (lane == 0 && b > 0 && b <= n) pv = __ldg(cv + b - 1);
  };
  ld(warp * 32);
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t i = base + lane;
    const int32_t cev = ev, ceu = eu, cer = er, cev2 = ev2, ceu2 = eu2, cer2 = er2, cpv = pv;
    ld(base + nwarps * 32);
    // each lane's entry row: its visited flag, fetched ahead of the rounds
    uint32_t vis = 0u;
    if (SEM != TH_EXACT && i < n) {
      const int32_t vi = cev < 0 ? ~cev : cev;
      vis = (__ldcg(a.Vf + (vi >> 5)) >> (vi & 31)) & 1u;
    }
    int32_t prev = __shfl_up_sync(TH_FULL, cev, 1);
    if (lane == 0) prev = cpv;
    // a run starts where vv changes; a split row's run also at the window
    // start; a whole row's run continuing from the previous window is its
    const bool start = i < n && (cev != prev || (lane == 0 && cev < 0));
    const unsigned S = __ballot_sync(TH_FULL, start);
    if (!S) continue;
    const int nseg = __popc(S);
    const int wend = n - base >= 32 ? 32 : (int)(n - base);
    // the last run continues past the window when it is a whole row's
    const int ls = 31 - __clz((int)S);
    const int32_t lv = __shfl_sync(TH_FULL, cev, ls);
    int cont = 0;
    if (lv >= 0) {
      const unsigned ne = __ballot_sync(TH_FULL, cev2 != lv);
      cont = ne ? __ffs(ne) - 1 : 32;
    }
    if (start) seg[__popc(S & lanemask_lt())] = (int)lane;
    if (lane == 0) seg[nseg] = wend + cont;
    __syncwarp();
    // SPG runs per lane group per round, their row loads issued together
    for (int r0 = 0; r0 < nseg; r0 += GPW * SPG) {
      bool live[SPG], split[SPG];
      int s[SPG], len[SPG];
      int32_t v[SPG];
      size_t row[SPG];
      uint32_t seen[SPG][VEC], acc[SPG][VEC];
      int maxlen = 0;
#pragma unroll
      for (int g = 0; g < SPG; ++g) {
        const int si = r0 + g * GPW + grp;
        live[g] = si < nseg;
        s[g] = live[g] ? seg[si] : 0;
        len[g] = live[g] ? seg[si + 1] - s[g] : 0;
        const int32_t vv = __shfl_sync(TH_FULL, cev, s[g]);
        const uint32_t vs = __shfl_sync(TH_FULL, vis, s[g]);
        split[g] = vv < 0;
        v[g] = split[g] ? ~vv : vv;
        row[g] = (size_t)v[g] * W + part * VEC;
#pragma unroll
        for (int c = 0; c < VEC; ++c) {
          seen[g][c] = 0u;
          acc[g][c] = 0u;
        }
        if (SEM != TH_EXACT && live[g] && vs) ld_words<VEC>(a.V + row[g], seen[g]);
        maxlen = max(maxlen, len[g]);
      }
      maxlen = (int)__reduce_max_sync(TH_FULL, (unsigned)maxlen);
      for (int t0 = 0; t0 < maxlen; t0 += 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (t0 + k >= maxlen) break;  // (warp-uniform: most runs hold one or two edges)
#pragma unroll
          for (int g = 0; g < SPG; ++g) {
            const int t = s[g] + t0 + k;
            const int32_t ua = __shfl_sync(TH_FULL, ceu, t & 31);
            const int32_t ub = __shfl_sync(TH_FULL, ceu2, t & 31);
            int32_t ra = 0, rb = 0;
            if (FILTER) {
              ra = __shfl_sync(TH_FULL, cer, t & 31);
              rb = __shfl_sync(TH_FULL, cer2, t & 31);
            }
            if (t0 + k < len[g]) {
              const int32_t u = t < 32 ? ua : ub;
              uint32_t x[VEC];
              ldg_words<VEC>(a.X + (size_t)u * W + part * VEC, x);
              if (FILTER) {
                uint32_t m[VEC];
                ldg_words<VEC>(a.M + (size_t)(t < 32 ? ra : rb) * W + part * VEC, m);
#pragma unroll
                for (int c = 0; c < VEC; ++c) x[c] &= m[c];
              }
#pragma unroll
              for (int c = 0; c < VEC; ++c) acc[g][c] |= x[c];
            }
          }
        }
      }
#pragma unroll
      for (int g = 0; g < SPG; ++g) {
        uint32_t nb[VEC];
        bool any = false;
#pragma unroll
        for (int c = 0; c < VEC; ++c) {
          nb[c] = acc[g][c] & ~seen[g][c] & valid[c];
          any |= nb[c] != 0u;
        }
        any = (__ballot_sync(TH_FULL, any) & gbits) != 0u;
        bool fresh = false;
        if (live[g] && any) {
          if (!split[g]) {
            st_words<VEC>(a.N + row[g], nb);
            if (SEM != TH_EXACT && !a.last_frontier) {
              uint32_t nw[VEC];
#pragma unroll
              for (int c = 0; c < VEC; ++c) nw[c] = seen[g][c] | nb[c];
              st_words<VEC>(a.V + row[g], nw);
            }
            if (part == 0) {
              const uint32_t fb = 1u << (v[g] & 31);
              atomicOr(&a.Nf[v[g] >> 5], fb);
              if (SEM != TH_EXACT) atomicOr(&a.Vf[v[g] >> 5], fb);
              fresh = true;
            }
          } else {
#pragma unroll
            for (int c = 0; c < VEC; ++c) {
              if (nb[c]) {
                atomicOr(a.N + row[g] + c, nb[c]);
                if (SEM != TH_EXACT && !a.last_frontier) atomicOr(a.V + row[g] + c, nb[c]);
              }
            }
            if (part == 0) fresh = flag_next(a, v[g]);
          }
        }
        app.add(a, fresh, v[g]);
      }
    }
    __syncwarp();
  }
  app.finish(a);
}
