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
  // (over the two-phase screen's compacted items: dense hops only)
  if (a.n_items_dev && a.ctl->dense[a.h] == 0) return;
  const bool dense = a.ctl->dense[a.h] != 0;
  using RS = RowShape<W>;
  constexpr int VEC = RS::VEC, LPR = RS::LPR, GPW = RS::GPW;
  // nth-set-bit table for the LPR-bit group masks: entry m holds the
  // positions of m's set bits, ascending, one per nibble (replaces __fns,
  // a software loop)
  __shared__ uint32_t nth_bit[LPR >= 4 ? (1 << LPR) : 1];
  __shared__ int32_t abuf[kThreads / 32][2 * kAppendRun];
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
      } else {
#pragma unroll
        for (int c = 0; c < VEC; ++c) {
          if (nb[c]) {
            atomicOr(a.N + row + c, nb[c]);
            if (SEM != TH_EXACT && !a.last_frontier) atomicOr(a.V + row + c, nb[c]);
          }
        }
      }
      if (part == 0) fresh = flag_next(a, v);
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
// Here a warp takes 32 consecutive items, whose in-edges are one contiguous
// run of the reverse CSR (items split rows in order; rows without in-edges
// have none), and tests that run 32 edges per step: coalesced source loads,
// independent flag loads, the owning item found by a 5-step search over the
// lanes' item starts.
//   non-dense hops: the frontier in-edges themselves are compacted, as
//     (vv, u[, rel]) in edge order -- an item's entries stay consecutive --
//     and pull_edges_kernel gathers them: one dependent step (the entry) in
//     front of the row loads instead of three.
//   dense hops (every in-edge is taken): the items are compacted as
//     (v, lo, hi) and pull_kernel<.., SCREEN = false> runs over that list.
// Entries go through a per-warp shared run stored with one global atomic
// per >= 32 entries (ctl->pull_items[h] counts them).
constexpr int kScreenRun = 32;
constexpr int kScreenBuf = 64;

template <bool FILTER>
__global__ void __launch_bounds__(kThreads) pull_screen_kernel(WaveArgs a, int32_t* c0, int32_t* c1,
                                                               int32_t* c2) {
  if (a.ctl->mode[a.h] != 1) return;
  const bool dense = a.ctl->dense[a.h] != 0;
  __shared__ int32_t sb[kThreads / 32][3][kScreenBuf];
  const int wib = threadIdx.x >> 5;
  int32_t* b0 = sb[wib][0];
  int32_t* b1 = sb[wib][1];
  int32_t* b2 = sb[wib][2];
  int fill = 0;
  const unsigned lane = lane_id();
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n = a.n_items;
  int32_t* count = &a.ctl->pull_items[a.h];
  // (dense: items, three words each; else edges, two or three)
  const bool third = dense || FILTER;
  auto flush = [&]() {
    __syncwarp();
    int32_t at = 0;
    if (lane == 0) at = atomicAdd(count, fill);
    at = __shfl_sync(TH_FULL, at, 0);
    for (int i = (int)lane; i < fill; i += 32) {
      c0[at + i] = b0[i];
      c1[at + i] = b1[i];
      if (third) c2[at + i] = b2[i];
    }
    fill = 0;
    __syncwarp();
  };
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t it = base + lane;
    int32_t vv = 0, lo = INT32_MAX, hi = INT32_MAX;
    if (it < n) {
      vv = __ldg(a.item_v + it);
      lo = __ldg(a.item_lo + it);
      hi = __ldg(a.item_hi + it);
    }
    if (dense) {
      const bool act = it < n;
      const unsigned fm = __ballot_sync(TH_FULL, act);
      if (act) {
        const int p = fill + __popc(fm & lanemask_lt());
        b0[p] = vv;
        b1[p] = lo;
        b2[p] = hi;
      }
      fill += __popc(fm);
      if (fill >= kScreenRun) flush();
      continue;
    }
    const int last = n - base >= 32 ? 31 : (int)(n - 1 - base);
    const int32_t L = __shfl_sync(TH_FULL, lo, 0), H = __shfl_sync(TH_FULL, hi, last);
    int32_t forced = -1;  // an item cut by a flush: all its entries are marked split
    for (int32_t e0 = L; e0 < H; e0 += 32) {
      const int32_t e = e0 + (int32_t)lane;
      bool ea = false;
      int32_t u = 0;
      if (e < H) {
        u = __ldg(a.rsrc + e);
        ea = (__ldg(a.Xf + (u >> 5)) >> (u & 31)) & 1u;
      }
      const unsigned em = __ballot_sync(TH_FULL, ea);
      if (!em) continue;
      // owning item: the last lane whose item starts at or before e
      int own = 0;
#pragma unroll
      for (int st = 16; st >= 1; st >>= 1) {
        const int32_t l = __shfl_sync(TH_FULL, lo, own + st);
        if (l <= e) own += st;
      }
      int32_t ev = __shfl_sync(TH_FULL, vv, own);
      const int c = __popc(em);
      if (fill + c > kScreenBuf) {
        // the item open at e0 (started in an earlier step) is cut: its
        // buffered entries (a suffix of the run) and the rest of its
        // entries become a split row's, merged with atomics in phase 2
        const int own0 = __shfl_sync(TH_FULL, own, 0);
        const int32_t v0 = __shfl_sync(TH_FULL, vv, own0);
        const int32_t lo0 = __shfl_sync(TH_FULL, lo, own0);
        if (lo0 < e0 && v0 >= 0) {
          for (int i = (int)lane; i < fill; i += 32)
            if (b0[i] == v0) b0[i] = ~v0;
          forced = v0;
        }
        flush();
      }
      if (ev >= 0 && ev == forced) ev = ~ev;
      if (ea) {
        const int p = fill + __popc(em & lanemask_lt());
        b0[p] = ev;
        b1[p] = u;
        if (FILTER) b2[p] = (int32_t)__ldg(a.rrel + e);
      }
      fill += c;
    }
    if (fill >= kScreenRun) flush();
  }
  if (fill) flush();
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
template <int W, int SEM, bool FILTER>
__global__ void __launch_bounds__(kThreads) pull_edges_kernel(WaveArgs a, const int32_t* __restrict__ cv,
                                                              const int32_t* __restrict__ cu,
                                                              const int32_t* __restrict__ cr) {
  if (a.ctl->mode[a.h] != 1 || a.ctl->dense[a.h] != 0) return;
  using RS = RowShape<W>;
  constexpr int VEC = RS::VEC, LPR = RS::LPR, GPW = RS::GPW;
  __shared__ int32_t abuf[kThreads / 32][2 * kAppendRun];
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
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t i = base + lane;
    int32_t ev = INT32_MIN, eu = 0, er = 0;
    if (i < n) {
      ev = __ldg(cv + i);
      eu = __ldg(cu + i);
      if (FILTER) er = __ldg(cr + i);
    }
    int32_t prev = __shfl_up_sync(TH_FULL, ev, 1);
    if (lane == 0) prev = base > 0 ? __ldg(cv + base - 1) : INT32_MIN;
    // a run starts where vv changes; a split row's run also at the window
    // start; a whole row's run continuing from the previous window is its
    const bool start = i < n && (ev != prev || (lane == 0 && ev < 0));
    const unsigned S = __ballot_sync(TH_FULL, start);
    if (!S) continue;
    const int nseg = __popc(S);
    const int wend = n - base >= 32 ? 32 : (int)(n - base);
    // the last run continues past the window when it is a whole row's
    const int ls = 31 - __clz((int)S);
    const int32_t lv = __shfl_sync(TH_FULL, ev, ls);
    int cont = 0;
    int32_t u2 = 0, r2 = 0;
    if (lv >= 0 && base + 32 < n) {
      const int64_t j = base + 32 + lane;
      const int32_t v2 = j < n ? __ldg(cv + j) : INT32_MIN;
      const unsigned ne = __ballot_sync(TH_FULL, v2 != lv);
      cont = ne ? __ffs(ne) - 1 : 32;
      if ((int)lane < cont) {
        u2 = __ldg(cu + j);
        if (FILTER) r2 = __ldg(cr + j);
      }
    }
    if (start) seg[__popc(S & lanemask_lt())] = (int)lane;
    if (lane == 0) seg[nseg] = wend + cont;
    __syncwarp();
    for (int r0 = 0; r0 < nseg; r0 += GPW) {
      const int si = r0 + grp;
      const bool live = si < nseg;
      const int s = live ? seg[si] : 0;
      const int len = live ? seg[si + 1] - s : 0;
      const int32_t vv = __shfl_sync(TH_FULL, ev, s);
      const bool split = vv < 0;
      const int32_t v = split ? ~vv : vv;
      const size_t row = (size_t)v * W + part * VEC;
      uint32_t seen[VEC], acc[VEC];
#pragma unroll
      for (int c = 0; c < VEC; ++c) {
        seen[c] = 0u;
        acc[c] = 0u;
      }
      if (SEM != TH_EXACT && live && ((__ldcg(a.Vf + (v >> 5)) >> (v & 31)) & 1u))
        ld_words<VEC>(a.V + row, seen);
      const int maxlen = (int)__reduce_max_sync(TH_FULL, (unsigned)len);
      for (int t0 = 0; t0 < maxlen; t0 += 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int t = s + t0 + k;
          const int32_t ua = __shfl_sync(TH_FULL, eu, t & 31);
          const int32_t ub = __shfl_sync(TH_FULL, u2, t & 31);
          int32_t ra = 0, rb = 0;
          if (FILTER) {
            ra = __shfl_sync(TH_FULL, er, t & 31);
            rb = __shfl_sync(TH_FULL, r2, t & 31);
          }
          if (t0 + k < len) {
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
            for (int c = 0; c < VEC; ++c) acc[c] |= x[c];
          }
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
        if (!split) {
          st_words<VEC>(a.N + row, nb);
          if (SEM != TH_EXACT && !a.last_frontier) {
            uint32_t nw[VEC];
#pragma unroll
            for (int c = 0; c < VEC; ++c) nw[c] = seen[c] | nb[c];
            st_words<VEC>(a.V + row, nw);
          }
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
    __syncwarp();
  }
  app.finish(a);
}
