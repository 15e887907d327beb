// K1: device CSR build, replacing build_incidence (incidence.py:154-196).
//
//   degrees   = histogram of subjects            (np.bincount,   :183)
//   indptr    = exclusive scan of degrees        (np.cumsum,     :184)
//   csr_tid   = stable LSD radix sort of tids by subject (argsort stable, :188)
//   csr_obj/csr_rel = gathers through csr_tid (row-ordered copies so a hop
//               streams one contiguous segment per frontier entity)
//   reverse CSR = the same by object, for pull hops.
#include <algorithm>
#include <vector>

#include "../../include/th_b200.h"
#include "graph.cuh"
#include "prims.cuh"

namespace th {
namespace {

__global__ void minmax_kernel(const int32_t* __restrict__ s, const int32_t* __restrict__ r,
                              const int32_t* __restrict__ o, int64_t n, int32_t* mm) {
  int32_t lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v[3] = {s[i], r[i], o[i]};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = min(lo[c], v[c]);
      hi[c] = max(hi[c], v[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    for (int off = 16; off; off >>= 1) {
      lo[c] = min(lo[c], __shfl_xor_sync(TH_FULL, lo[c], off));
      hi[c] = max(hi[c], __shfl_xor_sync(TH_FULL, hi[c], off));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&mm[2 * c], lo[c]);
      atomicMax(&mm[2 * c + 1], hi[c]);
    }
  }
}

__global__ void histogram_kernel(const int32_t* __restrict__ key, int64_t n, int32_t* cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = key[i];
    const unsigned peers = __match_any_sync(__activemask(), k);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&cnt[k], __popc(peers));
  }
}

__global__ void iota_copy_kernel(const int32_t* __restrict__ key, int32_t* kout, int32_t* vout,
                                 int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    kout[i] = key[i];
    vout[i] = (int32_t)i;
  }
}

__global__ void narrow_rel_kernel(const int32_t* __restrict__ r, uint16_t* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint16_t)r[i];
}

// row-ordered copies: dst_a[i] = src_a[perm[i]], dst_r[i] = src_r[perm[i]]
__global__ void gather_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ src_a,
                              const uint16_t* __restrict__ src_r, int32_t* dst_a, uint16_t* dst_r,
                              int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = perm[i];
    dst_a[i] = src_a[p];
    dst_r[i] = src_r[p];
  }
}

__global__ void max_degree_kernel(const int32_t* __restrict__ ptr, int64_t E, int32_t* out) {
  int32_t m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
       i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, ptr[i + 1] - ptr[i]);
  for (int off = 16; off; off >>= 1) m = max(m, __shfl_xor_sync(TH_FULL, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// items per in-row (cnt[v], cnt[E] = 0) and the number of split rows
__global__ void item_count_kernel(const int32_t* __restrict__ rptr, int64_t E, int32_t* cnt,
                                  int32_t* n_split) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= E;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (v == E) {
      cnt[v] = 0;
      continue;
    }
    const int32_t d = rptr[v + 1] - rptr[v];
    const int32_t c = (d + kPullChunk - 1) / kPullChunk;
    cnt[v] = c;
    if (c > 1) atomicAdd(n_split, 1);
  }
}

__global__ void rdst_kernel(const int32_t* __restrict__ rperm, const int32_t* __restrict__ obj,
                            const int32_t* __restrict__ rptr, int64_t T, int32_t* rdst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < T;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = obj[rperm[e]];
    rdst[e] = rptr[v + 1] - rptr[v] > kPullChunk ? ~v : v;
  }
}

__global__ void item_fill_kernel(const int32_t* __restrict__ rptr, const int32_t* __restrict__ off,
                                 int64_t E, int32_t* iv, int32_t* ilo, int32_t* ihi) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < E;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t lo = rptr[v], hi = rptr[v + 1];
    const int32_t o = off[v], c = off[v + 1] - o;
    for (int32_t i = 0; i < c; ++i) {
      iv[o + i] = c > 1 ? ~(int32_t)v : (int32_t)v;
      ilo[o + i] = lo + i * kPullChunk;
      ihi[o + i] = min(hi, lo + (i + 1) * kPullChunk);
    }
  }
}

template <typename T>
T* talloc(int64_t n) {
  void* p = nullptr;
  TH_CUDA(cudaMalloc(&p, (size_t)std::max<int64_t>(n, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

template <typename T>
T* dalloc(Graph* g, int64_t n) {
  void* p = nullptr;
  const size_t bytes = (size_t)std::max<int64_t>(n, 1) * sizeof(T);
  TH_CUDA(cudaMalloc(&p, bytes));
  g->bytes += bytes;
  return static_cast<T*>(p);
}

unsigned grid_for(int64_t n, int threads = 256) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), kNumSMs * 16));
}

int bits_for(int64_t n) {
  int b = 0;
  while ((int64_t(1) << b) < n) ++b;
  return b;
}

// stable sort of triple ids by `key`, producing a CSR (ptr, perm)
void sorted_rows(Graph* g, const int32_t* key, int64_t T, int64_t E, int32_t* ptr, int32_t* perm,
                 cudaStream_t st) {
  int32_t* cnt = talloc<int32_t>(E + 1);
  TH_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (E + 1), st));
  histogram_kernel<<<grid_for(T), 256, 0, st>>>(key, T, cnt);
  TH_LAUNCHED();
  int32_t* scratch = talloc<int32_t>(std::max(scan_scratch_elems<int32_t>(E + 1),
                                              scan_scratch_elems<int32_t>(radix_hist_elems(T))));
  g->launches += 1 + scan_exclusive<int32_t>(cnt, ptr, E + 1, scratch, st);
  int32_t *k0 = talloc<int32_t>(T), *k1 = talloc<int32_t>(T), *v1 = talloc<int32_t>(T);
  int32_t* hist = talloc<int32_t>(radix_hist_elems(T));
  iota_copy_kernel<<<grid_for(T), 256, 0, st>>>(key, k0, perm, T);
  TH_LAUNCHED();
  g->launches += 1;
  const int where = radix_sort_pairs(k0, perm, k1, v1, T, bits_for(E), hist, scratch, st,
                                     &g->launches);
  if (where == 1)
    TH_CUDA(cudaMemcpyAsync(perm, v1, sizeof(int32_t) * T, cudaMemcpyDeviceToDevice, st));
  TH_CUDA(cudaStreamSynchronize(st));
  for (void* p : {(void*)cnt, (void*)scratch, (void*)k0, (void*)k1, (void*)v1, (void*)hist}) {
    cudaFree(p);
  }
}

}  // namespace

int graph_build(Graph* g, const int32_t* d_subj, const int32_t* d_rel, const int32_t* d_obj,
                int64_t T, int64_t E, int64_t R, bool reverse, cudaStream_t st, int64_t obj_bound) {
  if (obj_bound < 0) obj_bound = E;
  g->E = E;
  g->T = T;
  g->R = R;
  if (T > 0) {
    int32_t* mm = nullptr;
    TH_CUDA(cudaMalloc(&mm, 6 * sizeof(int32_t)));
    const int32_t init[6] = {INT32_MAX, INT32_MIN, INT32_MAX, INT32_MIN, INT32_MAX, INT32_MIN};
    TH_CUDA(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, st));
    minmax_kernel<<<grid_for(T), 256, 0, st>>>(d_subj, d_rel, d_obj, T, mm);
    TH_LAUNCHED();
    g->launches += 1;
    int32_t h[6];
    TH_CUDA(cudaMemcpyAsync(h, mm, sizeof(h), cudaMemcpyDeviceToHost, st));
    TH_CUDA(cudaStreamSynchronize(st));
    cudaFree(mm);
    const char* names[3] = {"subject", "relation", "object"};
    const int64_t bound[3] = {E, R, obj_bound};
    for (int c = 0; c < 3; ++c) {
      if (h[2 * c] < 0 || h[2 * c + 1] >= bound[c]) {
        set_error(std::string(names[c]) + " id out of range (bound " + std::to_string(bound[c]) +
                  ")");
        return TH_ERR_RANGE;
      }
    }
  }
  g->subj = dalloc<int32_t>(g, T);
  g->obj = dalloc<int32_t>(g, T);
  g->rel = dalloc<uint16_t>(g, T);
  if (T > 0) {
    TH_CUDA(cudaMemcpyAsync(g->subj, d_subj, sizeof(int32_t) * T, cudaMemcpyDeviceToDevice, st));
    TH_CUDA(cudaMemcpyAsync(g->obj, d_obj, sizeof(int32_t) * T, cudaMemcpyDeviceToDevice, st));
    narrow_rel_kernel<<<grid_for(T), 256, 0, st>>>(d_rel, g->rel, T);
    TH_LAUNCHED();
    g->launches += 1;
  }
  g->indptr = dalloc<int32_t>(g, E + 1);
  g->csr_tid = dalloc<int32_t>(g, T);
  g->csr_obj = dalloc<int32_t>(g, T);
  g->csr_rel = dalloc<uint16_t>(g, T);
  sorted_rows(g, g->subj, T, E, g->indptr, g->csr_tid, st);
  if (T > 0) {
    gather_kernel<<<grid_for(T), 256, 0, st>>>(g->csr_tid, g->obj, g->rel, g->csr_obj, g->csr_rel, T);
    TH_LAUNCHED();
    g->launches += 1;
  }
  int32_t* dmax = nullptr;
  TH_CUDA(cudaMalloc(&dmax, 2 * sizeof(int32_t)));
  TH_CUDA(cudaMemsetAsync(dmax, 0, 2 * sizeof(int32_t), st));
  if (E > 0) {
    max_degree_kernel<<<grid_for(E), 256, 0, st>>>(g->indptr, E, dmax);
    TH_LAUNCHED();
    g->launches += 1;
  }
  if (reverse) {
    g->rindptr = dalloc<int32_t>(g, E + 1);
    int32_t* rperm = talloc<int32_t>(T);
    g->rsrc = dalloc<int32_t>(g, T);
    g->rrel = dalloc<uint16_t>(g, T);
    g->rdst = dalloc<int32_t>(g, T);
    sorted_rows(g, g->obj, T, E, g->rindptr, rperm, st);
    if (T > 0) {
      gather_kernel<<<grid_for(T), 256, 0, st>>>(rperm, g->subj, g->rel, g->rsrc, g->rrel, T);
      TH_LAUNCHED();
      rdst_kernel<<<grid_for(T), 256, 0, st>>>(rperm, g->obj, g->rindptr, T, g->rdst);
      TH_LAUNCHED();
      g->launches += 2;
    }
    TH_CUDA(cudaStreamSynchronize(st));
    cudaFree(rperm);
    if (E > 0) {
      max_degree_kernel<<<grid_for(E), 256, 0, st>>>(g->rindptr, E, dmax + 1);
      TH_LAUNCHED();
      g->launches += 1;
    }
    // static pull items: scan of per-row item counts, then fill
    int32_t* cnt = talloc<int32_t>(E + 2);
    int32_t* off = talloc<int32_t>(E + 1);
    int32_t* nsplit = cnt + E + 1;
    TH_CUDA(cudaMemsetAsync(nsplit, 0, sizeof(int32_t), st));
    item_count_kernel<<<grid_for(E + 1), 256, 0, st>>>(g->rindptr, E, cnt, nsplit);
    TH_LAUNCHED();
    int32_t* scratch = talloc<int32_t>(scan_scratch_elems<int32_t>(E + 1));
    g->launches += 1 + scan_exclusive<int32_t>(cnt, off, E + 1, scratch, st);
    int32_t hc[2];
    TH_CUDA(cudaMemcpyAsync(&hc[0], off + E, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    TH_CUDA(cudaMemcpyAsync(&hc[1], nsplit, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    TH_CUDA(cudaStreamSynchronize(st));
    g->n_items = hc[0];
    g->n_split = hc[1];
    g->item_v = dalloc<int32_t>(g, g->n_items);
    g->item_lo = dalloc<int32_t>(g, g->n_items);
    g->item_hi = dalloc<int32_t>(g, g->n_items);
    if (E > 0) {
      item_fill_kernel<<<grid_for(E), 256, 0, st>>>(g->rindptr, off, E, g->item_v, g->item_lo,
                                                    g->item_hi);
      TH_LAUNCHED();
      g->launches += 1;
    }
    TH_CUDA(cudaStreamSynchronize(st));
    for (void* p : {(void*)cnt, (void*)off, (void*)scratch}) cudaFree(p);
  }
  int32_t hm[2];
  TH_CUDA(cudaMemcpyAsync(hm, dmax, sizeof(hm), cudaMemcpyDeviceToHost, st));
  TH_CUDA(cudaStreamSynchronize(st));
  cudaFree(dmax);
  g->max_out = hm[0];
  g->max_in = hm[1];
  return TH_OK;
}

void graph_free(Graph* g) {
  for (void* p : {(void*)g->indptr, (void*)g->csr_tid, (void*)g->csr_obj, (void*)g->csr_rel,
                  (void*)g->subj, (void*)g->obj, (void*)g->rel, (void*)g->rindptr, (void*)g->rsrc,
                  (void*)g->rrel, (void*)g->rdst, (void*)g->item_v, (void*)g->item_lo, (void*)g->item_hi}) {
    if (p) cudaFree(p);
  }
  *g = Graph{};
}

}  // namespace th
