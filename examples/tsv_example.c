/*
 * Standalone C use of the retrieval backend's C ABI (include/tsv.h): no Python, no torch.
 * Builds a cosine index of N random 256-d rows, searches B queries that are noisy copies of
 * known rows, and checks that every query finds its row first.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/tsv_example.c \
 *       -L paper_2407_00326_b200/lib -ltsv -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2407_00326_b200/lib -o tsv_example && ./tsv_example
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "tsv.h"

#define CHECK(x)                                                             \
  do {                                                                       \
    int rc_ = (x);                                                           \
    if (rc_ != 0) {                                                          \
      fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, tsv_last_error());     \
      return 1;                                                              \
    }                                                                        \
  } while (0)

static float frand(uint64_t* s) { /* xorshift64*, uniform in (-1, 1) */
  *s ^= *s >> 12;
  *s ^= *s << 25;
  *s ^= *s >> 27;
  return (float)((*s * 2685821657736338717ull) >> 40) / (float)(1ull << 23) - 1.0f;
}

int main(void) {
  const int dim = 256, B = 64, k = 5;
  const int64_t n = 100000;
  uint64_t seed = 88172645463325252ull;
  float* rows = (float*)malloc(sizeof(float) * n * dim);
  float* queries = (float*)malloc(sizeof(float) * B * dim);
  for (int64_t i = 0; i < n * dim; ++i) rows[i] = frand(&seed);
  for (int b = 0; b < B; ++b) /* query b = row 1000 b + small noise */
    for (int d = 0; d < dim; ++d)
      queries[b * dim + d] = rows[(int64_t)(1000 * b) * dim + d] + 0.01f * frand(&seed);

  void *d_rows, *d_q, *d_s, *d_i;
  if (cudaMalloc(&d_rows, sizeof(float) * n * dim) || cudaMalloc(&d_q, sizeof(float) * B * dim) ||
      cudaMalloc(&d_s, sizeof(float) * B * k) || cudaMalloc(&d_i, sizeof(int32_t) * B * k)) {
    fprintf(stderr, "cudaMalloc failed (no GPU?)\n");
    return 2;
  }
  cudaMemcpy(d_rows, rows, sizeof(float) * n * dim, cudaMemcpyHostToDevice);
  cudaMemcpy(d_q, queries, sizeof(float) * B * dim, cudaMemcpyHostToDevice);

  tsv_index* idx = NULL;
  int64_t first = -1;
  CHECK(tsv_index_create(0, dim, TSV_METRIC_COSINE, n, &idx));
  /* fp32 rows in; the arena stores them L2-normalised as bf16 */
  CHECK(tsv_index_append(idx, d_rows, TSV_F32, n, &first, NULL));
  CHECK(tsv_search(idx, d_q, TSV_F32, B, k, 0, n, 0, (float*)d_s, (int32_t*)d_i, NULL));
  float scores[64 * 5];
  int32_t ids[64 * 5];
  cudaMemcpy(scores, d_s, sizeof(scores), cudaMemcpyDeviceToHost);
  cudaMemcpy(ids, d_i, sizeof(ids), cudaMemcpyDeviceToHost);

  int ok = 0;
  for (int b = 0; b < B; ++b) ok += ids[b * k] == 1000 * b;
  printf("tsv_example: %d/%d queries found their row first (query 0: id %d, cosine %.4f)\n", ok,
         B, ids[0], scores[0]);
  CHECK(tsv_index_destroy(idx));
  cudaFree(d_rows);
  cudaFree(d_q);
  cudaFree(d_s);
  cudaFree(d_i);
  free(rows);
  free(queries);
  return ok == B ? 0 : 3;
}
