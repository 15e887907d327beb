/*
 * A C caller of the engine, with no Python and no torch: builds a graph from
 * (s, r, o) columns, runs one batch of per-seed queries (k hops, FRONTIER,
 * paths on) and prints every seed's frontiers, edge counts and paths.
 *
 *   gcc examples/c_abi_khop.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2604_18913_b200/lib -lth_b200 -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2604_18913_b200/lib -o /tmp/c_abi_khop
 *   /tmp/c_abi_khop E R k  < triples(s r o per line, then "--", then seeds)
 *
 * tests/test_gpu_c_abi.py compiles it and checks its output against the
 * oracle.  This is the call sequence a C/C++ host of the reference's hot
 * path would use.
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "th_b200.h"

#define CK(x)                                                                  \
  do {                                                                         \
    int rc_ = (x);                                                             \
    if (rc_) {                                                                 \
      fprintf(stderr, "%s -> %d: %s\n", #x, rc_, th_last_error());             \
      return 1;                                                                \
    }                                                                          \
  } while (0)

static int32_t* to_device(const int32_t* h, size_t n) {
  int32_t* d = NULL;
  cudaMalloc((void**)&d, (n ? n : 1) * sizeof(int32_t));
  if (n) cudaMemcpy(d, h, n * sizeof(int32_t), cudaMemcpyHostToDevice);
  return d;
}

int main(int argc, char** argv) {
  if (argc < 4) {
    fprintf(stderr, "usage: %s E R k < input\n", argv[0]);
    return 2;
  }
  const int64_t E = atoll(argv[1]), R = atoll(argv[2]);
  const int k = atoi(argv[3]);
  size_t cap = 1024, T = 0, B = 0;
  int32_t *s = malloc(cap * 4), *r = malloc(cap * 4), *o = malloc(cap * 4);
  char tok[64];
  while (scanf("%63s", tok) == 1 && strcmp(tok, "--") != 0) {
    if (T == cap) {
      cap *= 2;
      s = realloc(s, cap * 4), r = realloc(r, cap * 4), o = realloc(o, cap * 4);
    }
    s[T] = atoi(tok);
    if (scanf("%d %d", &r[T], &o[T]) != 2) return 2;
    ++T;
  }
  int32_t* seeds = malloc(4096 * 4);
  while (B < 4096 && scanf("%d", &seeds[B]) == 1) ++B;
  int32_t* offs = malloc((B + 1) * 4);
  for (size_t i = 0; i <= B; ++i) offs[i] = (int32_t)i;

  cudaStream_t st;
  cudaStreamCreate(&st);
  int32_t *ds = to_device(s, T), *dr = to_device(r, T), *dob = to_device(o, T);
  int32_t *dseeds = to_device(seeds, B), *doffs = to_device(offs, B + 1);
  th_graph* g = NULL;
  th_session* sess = NULL;
  CK(th_graph_create(ds, dr, dob, (int64_t)T, E, R, 0, st, &g));
  CK(th_session_create(g, st, &sess));
  th_query q = {(int32_t)B, doffs, dseeds, k, TH_FRONTIER, NULL, 0,
                TH_WANT_FRONTIERS | TH_WANT_PATHS | TH_SINGLETON_SEEDS, 10000};
  th_result res;
  CK(th_run(sess, &q));
  int rc = th_finish(sess, &res);
  if (rc == TH_ERR_OVERFLOW) {  /* capacities grew: issue the same run again */
    CK(th_run(sess, &q));
    rc = th_finish(sess, &res);
  }
  CK(rc);

  const size_t kb = (size_t)k * B;
  int64_t *foff = malloc(kb * 8), *flen = malloc(kb * 8), *edges = malloc(kb * 8);
  int64_t *poff = malloc((B + 1) * 8), *pcnt = malloc(B * 8 + 8);
  uint8_t* ptr = malloc(B + 1);
  int32_t* fids = malloc((res.frontier_total ? res.frontier_total : 1) * 4);
  int32_t* ptids = malloc((res.path_total ? res.path_total : 1) * (size_t)k * 4);
  cudaMemcpy(foff, res.frontier_off, kb * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(flen, res.frontier_len, kb * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(edges, res.edges, kb * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(fids, res.frontier_ids, res.frontier_total * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(poff, res.path_off, (B + 1) * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(pcnt, res.path_count, B * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(ptr, res.path_truncated, B, cudaMemcpyDeviceToHost);
  cudaMemcpy(ptids, res.path_tids, res.path_total * (size_t)k * 4, cudaMemcpyDeviceToHost);

  for (size_t i = 0; i < B; ++i) {
    printf("seed %d\n", seeds[i]);
    for (int h = 0; h < k; ++h) {
      const size_t at = (size_t)h * B + i;
      printf("hop %d edges %lld ids", h + 1, (long long)edges[at]);
      for (int64_t j = 0; j < flen[at]; ++j) printf(" %d", fids[foff[at] + j]);
      printf("\n");
    }
    printf("paths %lld truncated %d\n", (long long)pcnt[i], (int)ptr[i]);
    for (int64_t p = 0; p < pcnt[i]; ++p) {
      printf("path");
      for (int d = 0; d < k; ++d) printf(" %d", ptids[(poff[i] + p) * k + d]);
      printf("\n");
    }
  }
  th_session_destroy(sess);
  th_graph_destroy(g);
  cudaFree(ds), cudaFree(dr), cudaFree(dob), cudaFree(dseeds), cudaFree(doffs);
  cudaStreamDestroy(st);
  return 0;
}
