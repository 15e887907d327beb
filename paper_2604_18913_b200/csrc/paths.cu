// K5: path reconstruction on the device.
//
// Reference: reconstruct_paths / HopAdjacency / assemble_paths
// (incidence.py:344-408).  Paths are ALL length-k walks from the query's
// seed set, ordered lexicographically by their triple-id sequence, capped at
// max_paths with a `truncated` flag (incidence.py:386-388).  Every step of a
// walk is an activated triple of its hop under exact-walk semantics, so
// level d>0 candidates are exactly the CSR row of the previous object (rows
// are tid-ascending by construction, incidence.py:186-188), filtered by the
// query's relation mask.  Level 0 is the seed's row (single-seed queries) or
// the hop-1 activated list (seed sets: rows interleave by tid).
//
// One warp per query runs an explicit-stack DFS.  Every level scans 32
// candidates per step with a ballot; the second-to-last level takes 32
// candidates at once so empty rows cost nothing and, when counting without a
// relation filter, whole rows are counted from their lengths.  Two passes:
// COUNT (saturating at max_paths+1 -> truncated flag) and WRITE into a packed
// [path][k] triple-id array whose offsets come from a device scan.
#include <climits>

#include "common.cuh"
#include "paths.cuh"
#include "prims.cuh"

namespace th {
namespace {

constexpr int kPathThreads = 128;
constexpr int kMaxDepth = 32;

struct Cand {
  int32_t tid, obj;
  uint32_t rel;
};

__device__ __forceinline__ bool rel_ok(const PathArgs& a, int q, uint32_t r) {
  if (!a.masks) return true;
  return (a.masks[(size_t)q * a.mask_words + (r >> 5)] >> (r & 31)) & 1u;
}

// level-0 candidate i (list mode) or CSR slot i (row mode)
__device__ __forceinline__ Cand cand_l0(const PathArgs& a, bool list_mode, int64_t i) {
  Cand c;
  if (list_mode) {
    c.tid = a.l0_ids[i];
    c.obj = a.t_obj[c.tid];
    c.rel = a.t_rel[c.tid];
  } else {
    c.tid = a.csr_tid[i];
    c.obj = a.csr_obj[i];
    c.rel = a.csr_rel[i];
  }
  return c;
}

__device__ __forceinline__ Cand cand_csr(const PathArgs& a, int64_t i) {
  Cand c;
  c.tid = a.csr_tid[i];
  c.obj = a.csr_obj[i];
  c.rel = a.csr_rel[i];
  return c;
}

// candidates [lo, hi) of level d in order: 4 x 32 per iteration, all loads
// issued before the four ordered ballots (a huge filtered row is the DFS's
// critical path; this cuts its dependent iterations 4x)
template <bool WRITE, bool SINGLE = false>
__device__ __forceinline__ void emit_range(const PathArgs& a, int q, int d, bool list_mode,
                                           int64_t lo, int64_t hi, const int32_t* stack_tid,
                                           int64_t& count, int64_t limit, int64_t out_base) {
  const unsigned lane = lane_id();
  for (int64_t b = lo; b < hi && count < limit; b += 128) {
    Cand c[4];
    bool pass[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = b + 32 * u + lane;
      pass[u] = i < hi;
      c[u] = Cand{0, 0, 0};
      if (pass[u]) c[u] = d == 0 ? cand_l0(a, list_mode, i) : cand_csr(a, i);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (pass[u]) pass[u] = rel_ok(a, q, c[u].rel);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned bal = __ballot_sync(TH_FULL, pass[u]);
      if (WRITE && pass[u]) {
        const int64_t idx = count + __popc(bal & lanemask_lt());
        const int64_t pp = out_base + idx;
        // SINGLE: counts run to max_paths + 1 (truncation), slots hold max_paths
        if (SINGLE ? idx < a.max_paths : (idx < limit && pp < a.cap)) {
          int32_t* dst = (SINGLE ? a.tmp : a.p_tids) + pp * a.k;
          for (int dd = 0; dd < d; ++dd) dst[dd] = stack_tid[dd];
          dst[d] = c[u].tid;
        }
      }
      count += __popc(bal);
    }
  }
}

template <bool WRITE, bool SINGLE = false>
__global__ void __launch_bounds__(kPathThreads) paths_kernel(PathArgs a) {
  __shared__ int32_t stack_tid_s[kPathThreads / 32][kMaxDepth];
  __shared__ int64_t cur_s[kPathThreads / 32][kMaxDepth];
  __shared__ int64_t end_s[kPathThreads / 32][kMaxDepth];
  const int warp = threadIdx.x >> 5;
  const unsigned lane = lane_id();
  int32_t* stack_tid = stack_tid_s[warp];
  int64_t* cur = cur_s[warp];
  int64_t* end = end_s[warp];
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int k = a.k;
  for (int q = gw; q < a.B; q += nw) {
    bool list_mode = !a.singleton;
    int64_t lo0 = 0, hi0 = 0;
    if (list_mode) {
      lo0 = a.l0_off[q];
      hi0 = lo0 + a.l0_len[q];
    } else {
      // singleton queries: query q is {seeds[q]} (offsets are not read)
      {
        const int32_t s = a.seeds[q];
        if (s >= 0 && s < a.E) {
          lo0 = a.indptr[s];
          hi0 = a.indptr[s + 1];
        }
      }
    }
    int64_t limit, out_base = 0;
    if (SINGLE) {
      limit = a.max_paths + 1;
      out_base = (int64_t)q * a.max_paths;
    } else if (WRITE) {
      limit = a.p_cnt[q];
      out_base = a.p_off[q];
    } else {
      limit = a.max_paths < 0 ? LLONG_MAX : a.max_paths + 1;
    }
    int64_t count = 0;
    if (limit > 0) {
      int d = 0;
      if (lane == 0) {
        cur[0] = lo0;
        end[0] = hi0;
      }
      __syncwarp();
      while (d >= 0 && count < limit) {
        if (d == k - 1) {
          emit_range<WRITE, SINGLE>(a, q, d, list_mode, cur[d], end[d], stack_tid, count, limit, out_base);
          --d;
          continue;
        }
        if (d == k - 2) {
          // batch of 32 candidates; their rows are the last level
          const int64_t b = cur[d], e = end[d];
          if (b >= e) {
            --d;
            continue;
          }
          const int64_t i = b + lane;
          bool pass = false;
          Cand c{0, 0, 0};
          int64_t rlo = 0, rhi = 0;
          if (i < e) {
            c = d == 0 ? cand_l0(a, list_mode, i) : cand_csr(a, i);
            pass = rel_ok(a, q, c.rel);
            if (pass) {
              rlo = a.indptr[c.obj];
              rhi = a.indptr[c.obj + 1];
            }
          }
          __syncwarp();
          if (lane == 0) cur[d] = b + 32;
          __syncwarp();
          unsigned nonempty = __ballot_sync(TH_FULL, pass && rhi > rlo);
          if (!WRITE && !SINGLE && !a.masks) {
            int64_t n = rhi - rlo;
            for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(TH_FULL, n, o);
            count += n;
            continue;
          }
          while (nonempty && count < limit) {
            const int f = __ffs(nonempty) - 1;
            nonempty &= nonempty - 1u;
            const int32_t t = __shfl_sync(TH_FULL, c.tid, f);
            const int64_t lo = __shfl_sync(TH_FULL, rlo, f), hi = __shfl_sync(TH_FULL, rhi, f);
            if (lane == 0) stack_tid[d] = t;
            __syncwarp();
            emit_range<WRITE, SINGLE>(a, q, d + 1, false, lo, hi, stack_tid, count, limit, out_base);
            __syncwarp();
          }
          // drain the skipped lanes' state when the limit was hit
          continue;
        }
        // generic level: advance to the next passing candidate
        bool found = false;
        int32_t nobj = 0;
        while (cur[d] < end[d]) {
          const int64_t b = cur[d];
          const int64_t i = b + lane;
          bool pass = false;
          Cand c{0, 0, 0};
          if (i < end[d]) {
            c = d == 0 ? cand_l0(a, list_mode, i) : cand_csr(a, i);
            pass = rel_ok(a, q, c.rel);
          }
          const unsigned bal = __ballot_sync(TH_FULL, pass);
          __syncwarp();
          if (bal) {
            const int f = __ffs(bal) - 1;
            const int32_t t = __shfl_sync(TH_FULL, c.tid, f);
            nobj = __shfl_sync(TH_FULL, c.obj, f);
            if (lane == 0) {
              stack_tid[d] = t;
              cur[d] = b + f + 1;
            }
            found = true;
            __syncwarp();
            break;
          }
          if (lane == 0) cur[d] = b + 32;
          __syncwarp();
        }
        if (!found) {
          --d;
          continue;
        }
        ++d;
        if (lane == 0) {
          cur[d] = a.indptr[nobj];
          end[d] = a.indptr[nobj + 1];
        }
        __syncwarp();
      }
    }
    if ((!WRITE || SINGLE) && lane == 0) {
      const int64_t cap = a.max_paths;
      a.p_cnt[q] = cap < 0 ? count : min(count, cap);
      a.p_trunc[q] = cap >= 0 && count > cap;
    }
    __syncwarp();
  }
}

// k = 2, singleton queries, capped (the C3 shape): the paths of a query are
// its seed's passing out-edges t1 (tid order) each followed by the passing
// out-edges t2 of obj(t1) (tid order).  A CTA takes a query and walks the
// level-0 candidates in order (compacted 256 at a time); each candidate's
// row of level-1 candidates is swept by the WHOLE CTA, 2,048 slots per step
// (8 per thread, loads issued together, one block-wide ordered compaction
// of all of them), so the long rows of hub objects -- which bounded the
// one-warp DFS on C3's hub seeds -- go 8 warps wide.  Stops once
// max_paths + 1 walks are known (truncation).  (Sweeping the candidates'
// rows laid end to end instead, with a per-slot binary search for the row,
// measured slower: C3 paths 2.55 vs 1.85 ms.)
constexpr int kPathK2Warps = 8;
constexpr int kPathK2Threads = 32 * kPathK2Warps;
constexpr int kPathK2Unroll = 8;

// block-wide ordered count of `ok`: this thread's exclusive rank and the
// block total (two barriers)
__device__ __forceinline__ int block_rank(bool ok, int* wcnt, int& total) {
  const int warp = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(TH_FULL, ok);
  if (lane_id() == 0) wcnt[warp] = __popc(bal);
  __syncthreads();
  int before = 0;
  total = 0;
#pragma unroll
  for (int w = 0; w < kPathK2Warps; ++w) {
    const int c = wcnt[w];
    before += w < warp ? c : 0;
    total += c;
  }
  __syncthreads();  // (wcnt is rewritten by the next call)
  return before + __popc(bal & lanemask_lt());
}

// block_rank over kPathK2Unroll slot groups at once (one barrier pair):
// group u's slots come after every slot of groups < u
__device__ __forceinline__ void block_rank_groups(const bool (&ok)[kPathK2Unroll], int (*wcnt)[kPathK2Warps],
                                                  int (&rank)[kPathK2Unroll], int& total) {
  const int warp = threadIdx.x >> 5;
  unsigned bal[kPathK2Unroll];
#pragma unroll
  for (int u = 0; u < kPathK2Unroll; ++u) {
    bal[u] = __ballot_sync(TH_FULL, ok[u]);
    if (lane_id() == 0) wcnt[u][warp] = __popc(bal[u]);
  }
  __syncthreads();
  int base = 0;
#pragma unroll
  for (int u = 0; u < kPathK2Unroll; ++u) {
    int before = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kPathK2Warps; ++w) {
      const int c = wcnt[u][w];
      before += w < warp ? c : 0;
      tot += c;
    }
    rank[u] = base + before + __popc(bal[u] & lanemask_lt());
    base += tot;
  }
  total = base;
  __syncthreads();  // (wcnt is rewritten by the next call)
}

__global__ void __launch_bounds__(kPathK2Threads) paths_k2_kernel(PathArgs a) {
  __shared__ int wcnt[kPathK2Warps];
  __shared__ int wcnt4[kPathK2Unroll][kPathK2Warps];
  __shared__ int32_t l0_tid[kPathK2Threads], l0_obj[kPathK2Threads];
  const int tid = threadIdx.x;
  for (int q = blockIdx.x; q < a.B; q += gridDim.x) {
    int64_t lo0 = 0, hi0 = 0;
    const int32_t s = a.seeds[q];
    if (s >= 0 && s < a.E) {
      lo0 = a.indptr[s];
      hi0 = a.indptr[s + 1];
    }
    int32_t* slot = a.tmp + (int64_t)q * a.max_paths * 2;
    int64_t total = 0;  // walks found so far (uniform across the CTA)
    for (int64_t c0 = lo0; c0 < hi0 && total <= a.max_paths; c0 += kPathK2Threads) {
      // this block's passing level-0 candidates, compacted in order
      const int64_t i = c0 + tid;
      const bool ok0 = i < hi0 && rel_ok(a, q, a.csr_rel[i]);
      int n0;
      const int r0 = block_rank(ok0, wcnt, n0);
      if (ok0) {
        l0_tid[r0] = a.csr_tid[i];
        l0_obj[r0] = a.csr_obj[i];
      }
      __syncthreads();
      for (int j = 0; j < n0 && total <= a.max_paths; ++j) {
        const int32_t t1 = l0_tid[j], o = l0_obj[j];
        const int64_t rlo = a.indptr[o], rhi = a.indptr[o + 1];
        for (int64_t b = rlo; b < rhi && total <= a.max_paths; b += kPathK2Threads * kPathK2Unroll) {
          bool ok[kPathK2Unroll];
          int32_t t2[kPathK2Unroll];
#pragma unroll
          for (int u = 0; u < kPathK2Unroll; ++u) {
            const int64_t e = b + (int64_t)u * kPathK2Threads + tid;
            ok[u] = e < rhi && rel_ok(a, q, a.csr_rel[e]);
            t2[u] = ok[u] ? a.csr_tid[e] : 0;
          }
          int rank[kPathK2Unroll], n;
          block_rank_groups(ok, wcnt4, rank, n);
#pragma unroll
          for (int u = 0; u < kPathK2Unroll; ++u) {
            const int64_t p = total + rank[u];
            if (ok[u] && p < a.max_paths) {
              slot[2 * p] = t1;
              slot[2 * p + 1] = t2[u];
            }
          }
          total += n;
        }
      }
      __syncthreads();  // (l0_* are rewritten by the next block)
    }
    if (tid == 0) {
      a.p_cnt[q] = total < a.max_paths ? total : a.max_paths;
      a.p_trunc[q] = total > a.max_paths;
    }
  }
}

// pack each query's slot of the single-pass buffer at its scanned offset
// (warp per query); nothing is written past the capacity (th_finish then
// reports the overflow and the run is repeated with room)
__global__ void paths_compact_kernel(PathArgs a) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int q = gw; q < a.B; q += nw) {
    const int64_t n = a.p_cnt[q], o = a.p_off[q];
    if (o + n > a.cap) continue;
    const int32_t* src = a.tmp + (int64_t)q * a.max_paths * a.k;
    int32_t* dst = a.p_tids + o * a.k;
    for (int64_t i = lane_id(); i < n * a.k; i += 32) dst[i] = src[i];
  }
}

__global__ void paths_total_kernel(int64_t* off, const int64_t* cnt, int32_t B, int64_t* used) {
  const int64_t tot = B > 0 ? off[B - 1] + cnt[B - 1] : 0;
  off[B] = tot;
  *used = tot;
}

}  // namespace

int64_t scan_scratch_elems_i64(int64_t n) { return scan_scratch_elems<int64_t>(n); }

int launch_paths(const PathArgs& a, cudaStream_t st) {
  if (a.k > kMaxDepth) return 0;
  int launches = 0;
  const unsigned grid =
      (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div((int64_t)a.B * 32, kPathThreads),
                                                       kNumSMs * 16));
  if (a.tmp) {
    // capped: one writing DFS into per-query slots (k = 2 singleton queries:
    // a CTA per query, see paths_k2_kernel), then pack
    if (a.B > 0) {
      if (a.k == 2 && a.singleton && a.k2_parallel) {
        const unsigned g2 = (unsigned)std::min<int64_t>(a.B, kNumSMs * 8);
        paths_k2_kernel<<<g2, kPathK2Threads, 0, st>>>(a);
      } else {
        paths_kernel<true, true><<<grid, kPathThreads, 0, st>>>(a);
      }
      TH_LAUNCHED();
      launches += 1 + scan_exclusive<int64_t>(a.p_cnt, a.p_off, a.B, a.scratch, st);
    }
    paths_total_kernel<<<1, 1, 0, st>>>(a.p_off, a.p_cnt, a.B, a.used);
    TH_LAUNCHED();
    launches += 1;
    if (a.B > 0) {
      paths_compact_kernel<<<grid, kPathThreads, 0, st>>>(a);
      TH_LAUNCHED();
      launches += 1;
    }
    return launches;
  }
  if (a.B > 0) {
    paths_kernel<false><<<grid, kPathThreads, 0, st>>>(a);
    TH_LAUNCHED();
    launches += 1 + scan_exclusive<int64_t>(a.p_cnt, a.p_off, a.B, a.scratch, st);
  }
  paths_total_kernel<<<1, 1, 0, st>>>(a.p_off, a.p_cnt, a.B, a.used);
  TH_LAUNCHED();
  launches += 1;
  if (a.B > 0) {
    paths_kernel<true><<<grid, kPathThreads, 0, st>>>(a);
    TH_LAUNCHED();
    launches += 1;
  }
  return launches;
}

}  // namespace th
