// K7: on-demand hub-adjacency cache (see hubcache.cuh).
//
// Layout after hubcache_create (e = edges per page = granularity / 2, so a
// page of the 2-byte relation column is one granule):
//
//   CSR position  [0, shift)            padding
//                 [shift, hub_base)     the owned rows' edges (mapped for good)
//                 [hub_base + p*e, +e)  hub page p: mapped while resident
//
// with hub_base = round_up(old hub start, e) and every indptr entry moved by
// shift = hub_base - old hub start, so the hub region starts on a page
// boundary.  Each slot of the pool is three physical allocations (object,
// relation, tid column pieces of one page) that are mapped at the virtual
// address of whichever page the slot holds.  The driver's VMM entry points
// are fetched through the runtime (cudaGetDriverEntryPoint), so the library
// has no link-time dependency on libcuda.
#include <cuda.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/th_b200.h"
#include "common.cuh"
#include "hubcache.cuh"

namespace th {

namespace {

struct Drv {
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) unreserve = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) access = nullptr;
  bool ok = false;
};

template <class F>
bool entry(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}

const Drv& drv() {
  static const Drv d = [] {
    Drv x;
    x.ok = entry("cuMemGetAllocationGranularity", &x.granularity) &&
           entry("cuMemAddressReserve", &x.reserve) && entry("cuMemAddressFree", &x.unreserve) &&
           entry("cuMemCreate", &x.create) && entry("cuMemRelease", &x.release) &&
           entry("cuMemMap", &x.map) && entry("cuMemUnmap", &x.unmap) &&
           entry("cuMemSetAccess", &x.access);
    return x;
  }();
  return d;
}

struct DrvError {
  CUresult code;
  const char* where;
};

#define TH_CU(expr)                                          \
  do {                                                       \
    CUresult _r = (expr);                                    \
    if (_r != CUDA_SUCCESS) throw DrvError{_r, #expr};       \
  } while (0)

__global__ void shift_indptr_kernel(int32_t* indptr, int64_t n, int32_t shift) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    indptr[i] += shift;
}

constexpr int kCols = 3;  // object, relation, tid
constexpr size_t kElem[kCols] = {4, 2, 4};

}  // namespace

struct HubCache {
  int device = 0;
  size_t gran = 0;
  int64_t row0 = 0, n_rows = 0;
  int64_t page_edges = 0, n_pages = 0, capacity = 0;
  int64_t hub_base = 0, hub_edges = 0;
  CUdeviceptr va[kCols] = {};
  size_t va_bytes[kCols] = {};
  CUmemGenericAllocationHandle prefix[kCols] = {};
  size_t prefix_bytes[kCols] = {};
  std::vector<CUmemGenericAllocationHandle> slot_mem;  // [capacity][kCols]
  std::vector<int64_t> slot_page;                      // page held, -1 = free
  std::vector<uint64_t> slot_stamp;                    // tick of the last access
  std::vector<int64_t> page_slot;                      // [n_pages] slot or -1
  void* host[kCols] = {};                              // pinned store of the hub pages
  std::vector<int32_t> hub_ptr;                        // shifted indptr[row0 .. row0 + n_rows]
  std::vector<uint32_t> flags;                         // staging for the row flag words
  uint64_t tick = 0;
  int64_t hits = 0, misses = 0, evictions = 0, resident = 0;
  std::vector<int64_t> log;

  CUdeviceptr page_va(int c, int64_t p) const {
    return va[c] + (CUdeviceptr)((hub_base + p * page_edges) * (int64_t)kElem[c]);
  }
  size_t page_bytes(int c) const { return (size_t)page_edges * kElem[c]; }
};

namespace {

void map_rw(const HubCache* hc, CUdeviceptr at, size_t bytes, CUmemGenericAllocationHandle h) {
  const Drv& d = drv();
  TH_CU(d.map(at, bytes, 0, h, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = hc->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  TH_CU(d.access(at, bytes, &acc, 1));
}

void evict(HubCache* hc, int64_t slot) {
  const int64_t p = hc->slot_page[slot];
  for (int c = 0; c < kCols; ++c) TH_CU(drv().unmap(hc->page_va(c, p), hc->page_bytes(c)));
  hc->page_slot[p] = -1;
  hc->slot_page[slot] = -1;
  hc->resident -= 1;
}

void load(HubCache* hc, int64_t slot, int64_t p, cudaStream_t st) {
  const int64_t n = std::min(hc->page_edges, hc->hub_edges - p * hc->page_edges);
  for (int c = 0; c < kCols; ++c) {
    map_rw(hc, hc->page_va(c, p), hc->page_bytes(c), hc->slot_mem[slot * kCols + c]);
    TH_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(hc->page_va(c, p)),
                            static_cast<char*>(hc->host[c]) + (size_t)p * hc->page_bytes(c),
                            (size_t)n * kElem[c], cudaMemcpyHostToDevice, st));
  }
  hc->page_slot[p] = slot;
  hc->slot_page[slot] = p;
  hc->resident += 1;
}

void release_all(HubCache* hc) {
  const Drv& d = drv();
  for (size_t s = 0; s < hc->slot_page.size(); ++s)
    if (hc->slot_page[s] >= 0) evict(hc, (int64_t)s);
  for (CUmemGenericAllocationHandle h : hc->slot_mem)
    if (h) d.release(h);
  hc->slot_mem.clear();
  for (int c = 0; c < kCols; ++c) {
    if (hc->prefix[c]) {
      d.unmap(hc->va[c], hc->prefix_bytes[c]);
      d.release(hc->prefix[c]);
      hc->prefix[c] = 0;
    }
    if (hc->va[c]) d.unreserve(hc->va[c], hc->va_bytes[c]);
    hc->va[c] = 0;
    if (hc->host[c]) cudaFreeHost(hc->host[c]);
    hc->host[c] = nullptr;
  }
}

template <class F>
int drv_guard(F&& f) {
  try {
    return f();
  } catch (const DrvError& e) {
    set_error(std::string(e.where) + ": CUDA driver error " + std::to_string((int)e.code));
    return e.code == CUDA_ERROR_OUT_OF_MEMORY ? TH_ERR_NOMEM : TH_ERR_CUDA;
  } catch (const CudaError& e) {
    set_error(std::string(e.where) + ": " + cudaGetErrorString(e.code));
    return e.code == cudaErrorMemoryAllocation ? TH_ERR_NOMEM : TH_ERR_CUDA;
  }
}

}  // namespace

int hubcache_create(HubCache** out, Graph* g, int64_t row0, int64_t capacity, cudaStream_t st) {
  *out = nullptr;
  if (capacity < 1) {
    set_error("hub cache capacity must be >= 1 page");
    return TH_ERR_INVALID;
  }
  if (row0 < 0 || row0 > g->E) {
    set_error("hub rows out of range");
    return TH_ERR_INVALID;
  }
  const Drv& d = drv();
  if (!d.ok) {
    set_error("the CUDA driver's virtual memory entry points are unavailable");
    return TH_ERR_CUDA;
  }
  auto* hc = new HubCache();
  const int rc = drv_guard([&]() -> int {
    TH_CUDA(cudaGetDevice(&hc->device));
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = hc->device;
    TH_CU(d.granularity(&hc->gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
    hc->row0 = row0;
    hc->n_rows = g->E - row0;
    hc->capacity = capacity;
    hc->page_edges = (int64_t)(hc->gran / 2);
    hc->hub_ptr.resize(hc->n_rows + 1);
    TH_CUDA(cudaMemcpyAsync(hc->hub_ptr.data(), g->indptr + row0, sizeof(int32_t) * (hc->n_rows + 1),
                            cudaMemcpyDeviceToHost, st));
    TH_CUDA(cudaStreamSynchronize(st));
    const int64_t base = hc->hub_ptr[0];
    const int64_t end = hc->hub_ptr[hc->n_rows];
    const int64_t e = hc->page_edges;
    hc->hub_edges = end - base;
    hc->n_pages = ceil_div(hc->hub_edges, e);
    hc->hub_base = ceil_div(base, e) * e;
    const int64_t shift = hc->hub_base - base;
    if ((int64_t)INT32_MAX - end < shift) {
      set_error("hub cache: shifted CSR positions exceed int32");
      return TH_ERR_INVALID;
    }
    hc->page_slot.assign(hc->n_pages, -1);
    void* old[kCols] = {g->csr_obj, g->csr_rel, g->csr_tid};
    const int64_t total = hc->hub_base + hc->n_pages * e;  // a multiple of e
    for (int c = 0; c < kCols; ++c) {
      // pinned host store of the hub pages (the tail of the last page unused)
      TH_CUDA(cudaHostAlloc(&hc->host[c], std::max<size_t>(hc->n_pages * hc->page_bytes(c), 1),
                            cudaHostAllocDefault));
      if (hc->hub_edges)
        TH_CUDA(cudaMemcpyAsync(hc->host[c], static_cast<char*>(old[c]) + base * kElem[c],
                                hc->hub_edges * kElem[c], cudaMemcpyDeviceToHost, st));
      hc->va_bytes[c] = std::max<size_t>((size_t)total * kElem[c], hc->gran);
      TH_CU(d.reserve(&hc->va[c], hc->va_bytes[c], hc->gran, 0, 0));
      // the owned rows' part: mapped for good, data moved up by `shift`
      hc->prefix_bytes[c] = (size_t)hc->hub_base * kElem[c];
      if (hc->prefix_bytes[c]) {
        TH_CU(d.create(&hc->prefix[c], hc->prefix_bytes[c], &prop, 0));
        map_rw(hc, hc->va[c], hc->prefix_bytes[c], hc->prefix[c]);
        if (base)
          TH_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(hc->va[c]) + shift * kElem[c], old[c],
                                  base * kElem[c], cudaMemcpyDeviceToDevice, st));
      }
    }
    hc->slot_mem.assign((size_t)capacity * kCols, 0);
    hc->slot_page.assign(capacity, -1);
    hc->slot_stamp.assign(capacity, 0);
    for (int64_t s = 0; s < capacity; ++s)
      for (int c = 0; c < kCols; ++c) TH_CU(d.create(&hc->slot_mem[s * kCols + c], hc->page_bytes(c), &prop, 0));
    if (shift) {
      shift_indptr_kernel<<<std::max<int64_t>(1, std::min<int64_t>(ceil_div(g->E + 1, 256), 4 * kNumSMs)), 256, 0,
                            st>>>(g->indptr, g->E + 1, (int32_t)shift);
      TH_LAUNCHED();
    }
    TH_CUDA(cudaStreamSynchronize(st));
    for (int c = 0; c < kCols; ++c) TH_CUDA(cudaFree(old[c]));
    g->csr_obj = reinterpret_cast<int32_t*>(hc->va[0]);
    g->csr_rel = reinterpret_cast<uint16_t*>(hc->va[1]);
    g->csr_tid = reinterpret_cast<int32_t*>(hc->va[2]);
    for (int32_t& x : hc->hub_ptr) x += (int32_t)shift;
    return TH_OK;
  });
  if (rc != TH_OK) {
    // (only reachable before the graph's arrays were swapped)
    drv_guard([&]() -> int {
      release_all(hc);
      return TH_OK;
    });
    delete hc;
    return rc;
  }
  *out = hc;
  return TH_OK;
}

int hubcache_step(HubCache* hc, const uint32_t* d_flags, cudaStream_t st) {
  if (hc->n_pages == 0) return TH_OK;
  return drv_guard([&]() -> int {
    const int64_t w0 = hc->row0 >> 5, w1 = (hc->row0 + hc->n_rows - 1) >> 5;
    hc->flags.resize(w1 - w0 + 1);
    TH_CUDA(cudaMemcpyAsync(hc->flags.data(), d_flags + w0, sizeof(uint32_t) * (w1 - w0 + 1),
                            cudaMemcpyDeviceToHost, st));
    TH_CUDA(cudaStreamSynchronize(st));
    // pages of the flagged hub rows, ascending
    std::vector<int64_t> want;
    int64_t last = -1;
    const int64_t e = hc->page_edges;
    for (int64_t i = 0; i < hc->n_rows; ++i) {
      const int64_t r = hc->row0 + i;
      if (!((hc->flags[(r >> 5) - w0] >> (r & 31)) & 1u)) continue;
      const int64_t lo = hc->hub_ptr[i] - hc->hub_base, hi = hc->hub_ptr[i + 1] - hc->hub_base;
      if (hi <= lo) continue;
      for (int64_t p = std::max(lo / e, last + 1); p <= (hi - 1) / e; ++p) want.push_back(p);
      last = std::max(last, (hi - 1) / e);
    }
    if ((int64_t)want.size() > hc->capacity) {
      set_error("hub cache: this hop's frontier hubs span " + std::to_string(want.size()) +
                " pages, the cache holds " + std::to_string(hc->capacity));
      return TH_ERR_INVALID;
    }
    // accesses: resident pages in recency order, then the missing ones
    std::vector<int64_t> hit, miss;
    for (int64_t p : want) (hc->page_slot[p] >= 0 ? hit : miss).push_back(p);
    std::sort(hit.begin(), hit.end(), [&](int64_t a, int64_t b) {
      return hc->slot_stamp[hc->page_slot[a]] < hc->slot_stamp[hc->page_slot[b]];
    });
    for (int64_t p : hit) {
      hc->log.push_back(p);
      hc->hits += 1;
      hc->slot_stamp[hc->page_slot[p]] = ++hc->tick;
    }
    for (int64_t p : miss) {
      hc->log.push_back(p);
      hc->misses += 1;
      int64_t slot = -1;
      for (int64_t s = 0; s < hc->capacity && slot < 0; ++s)
        if (hc->slot_page[s] < 0) slot = s;
      if (slot < 0) {  // full: the oldest stamp goes (never a page of this hop)
        slot = 0;
        for (int64_t s = 1; s < hc->capacity; ++s)
          if (hc->slot_stamp[s] < hc->slot_stamp[slot]) slot = s;
        evict(hc, slot);
        hc->evictions += 1;
      }
      load(hc, slot, p, st);
      hc->slot_stamp[slot] = ++hc->tick;
    }
    return TH_OK;
  });
}

void hubcache_stats(const HubCache* hc, int64_t out[8]) {
  out[0] = hc->hits;
  out[1] = hc->misses;
  out[2] = hc->misses;  // every miss loads once
  out[3] = hc->evictions;
  out[4] = hc->resident;
  out[5] = hc->capacity;
  out[6] = hc->n_pages;
  out[7] = hc->page_edges;
}

int64_t hubcache_trace(HubCache* hc, int64_t* out, int64_t cap) {
  const int64_t n = (int64_t)hc->log.size();
  if (out && cap >= n) {
    std::copy(hc->log.begin(), hc->log.end(), out);
    hc->log.clear();
  }
  return n;
}

int64_t hubcache_resident(const HubCache* hc, int64_t* out, int64_t cap) {
  std::vector<int64_t> slots;
  for (int64_t s = 0; s < hc->capacity; ++s)
    if (hc->slot_page[s] >= 0) slots.push_back(s);
  std::sort(slots.begin(), slots.end(),
            [&](int64_t a, int64_t b) { return hc->slot_stamp[a] < hc->slot_stamp[b]; });
  const int64_t n = (int64_t)slots.size();
  if (out && cap >= n)
    for (int64_t i = 0; i < n; ++i) out[i] = hc->slot_page[slots[i]];
  return n;
}

void hubcache_free(HubCache* hc, Graph* g) {
  if (!hc) return;
  cudaDeviceSynchronize();
  drv_guard([&]() -> int {
    release_all(hc);
    return TH_OK;
  });
  g->csr_obj = nullptr;
  g->csr_rel = nullptr;
  g->csr_tid = nullptr;
  delete hc;
}

}  // namespace th
