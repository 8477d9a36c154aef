/*
 * CPU restatement of the retrieval primitives — TEST INFRASTRUCTURE / CPU BASELINE ONLY.
 * Never linked into or called by the product path (paper_2407_00326_b200/).
 *
 * Brute-force exact search over bf16 rows (fp32 or fp64 accumulation), OpenMP over corpus
 * ranges, per-thread sorted top-k lists merged at the end. Ordering (score desc, id asc),
 * padding (-inf, -1). Semantics follow oracle/oracle.py (Searching: PAPER.md:359 and
 * pkg/src/teola_sim/optimizer.py:178-197; see that file's header for the parity status —
 * the reference has no arithmetic of its own to compile).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline float bf2f(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* insert into list sorted by (score desc, id asc); precondition s > ls[k-1] */
static inline void list_insert(double* ls, int32_t* li, int k, double s, int32_t id) {
  int p = k - 1;
  while (p > 0 && ls[p - 1] < s) {
    ls[p] = ls[p - 1];
    li[p] = li[p - 1];
    --p;
  }
  ls[p] = s;
  li[p] = id;
}

static int cmp_pair(const void* a, const void* b) {
  const double* x = (const double*)a;
  const double* y = (const double*)b;
  if (x[0] > y[0]) return -1;
  if (x[0] < y[0]) return 1;
  return (x[1] < y[1]) ? -1 : (x[1] > y[1]);
}

#define RB 16 /* corpus rows per vector */
#define QB 8  /* queries per register block */
typedef float v16 __attribute__((vector_size(64)));

int tsv_oracle_threads(void) { return omp_get_max_threads(); }

/* q: [B, D] bf16 bits; c: [N, D] bf16 bits. out: [B, k]. use_double selects fp64 accumulation. */
int tsv_oracle_search(const uint16_t* q, const uint16_t* c, int64_t B, int64_t N, int D, int k,
                      int use_double, int nthreads, int64_t id_offset, float* out_s,
                      int32_t* out_i) {
  if (B <= 0 || k <= 0 || D <= 0) return 1;
  if (nthreads <= 0) nthreads = omp_get_max_threads();
  float* qf = (float*)malloc(sizeof(float) * B * D);
  if (!qf) return 2;
  for (int64_t i = 0; i < B * D; ++i) qf[i] = bf2f(q[i]);
  double* ls = (double*)malloc(sizeof(double) * (size_t)nthreads * B * k);
  int32_t* li = (int32_t*)malloc(sizeof(int32_t) * (size_t)nthreads * B * k);
  if (!ls || !li) return 2;
  for (size_t i = 0; i < (size_t)nthreads * B * k; ++i) {
    ls[i] = -INFINITY;
    li[i] = -1;
  }

#pragma omp parallel num_threads(nthreads)
  {
    const int t = omp_get_thread_num();
    const int nt = omp_get_num_threads();
    const int64_t r0 = N * t / nt, r1 = N * (t + 1) / nt;
    /* row block stored d-major: blkT[d][0..RB) so one vector holds RB rows of one dim */
    v16* blkT = (v16*)aligned_alloc(64, sizeof(v16) * (size_t)D);
    double* my_s = ls + (size_t)t * B * k;
    int32_t* my_i = li + (size_t)t * B * k;
    for (int64_t rb = r0; rb < r1; rb += RB) {
      const int nr = (int)((r1 - rb) < RB ? (r1 - rb) : RB);
      for (int d = 0; d < D; ++d) {
        v16 col;
        for (int r = 0; r < RB; ++r)
          col[r] = r < nr ? bf2f(c[(size_t)(rb + r) * D + d]) : 0.f;
        blkT[d] = col;
      }
      for (int64_t qb = 0; qb < B; qb += QB) {
        const int nq = (int)((B - qb) < QB ? (B - qb) : QB);
        double sc[QB][RB];
        if (use_double) {
          for (int j = 0; j < nq; ++j)
            for (int r = 0; r < nr; ++r) {
              const float* qq = qf + (size_t)(qb + j) * D;
              double acc = 0.0;
              for (int d = 0; d < D; ++d) acc += (double)blkT[d][r] * (double)qq[d];
              sc[j][r] = acc;
            }
        } else {
          v16 acc[QB];
          for (int j = 0; j < QB; ++j) acc[j] = (v16){0};
          const float* qrow[QB];
          for (int j = 0; j < QB; ++j) qrow[j] = qf + (size_t)(qb + (j < nq ? j : 0)) * D;
          for (int d = 0; d < D; ++d) {
            const v16 x = blkT[d];
#pragma GCC unroll 8
            for (int j = 0; j < QB; ++j) acc[j] += x * qrow[j][d];
          }
          for (int j = 0; j < nq; ++j)
            for (int r = 0; r < nr; ++r) sc[j][r] = acc[j][r];
        }
        for (int j = 0; j < nq; ++j) {
          double* s = my_s + (size_t)(qb + j) * k;
          int32_t* ii = my_i + (size_t)(qb + j) * k;
          for (int r = 0; r < nr; ++r)
            if (sc[j][r] > s[k - 1]) list_insert(s, ii, k, sc[j][r], (int32_t)(rb + r + id_offset));
        }
      }
    }
    free(blkT);
  }

  /* merge per-thread lists */
  double* tmp = (double*)malloc(sizeof(double) * 2 * (size_t)nthreads * k);
  for (int64_t b = 0; b < B; ++b) {
    int m = 0;
    for (int t = 0; t < nthreads; ++t)
      for (int j = 0; j < k; ++j) {
        const size_t o = ((size_t)t * B + b) * k + j;
        if (li[o] < 0) continue;
        tmp[2 * m] = ls[o];
        tmp[2 * m + 1] = (double)li[o];
        ++m;
      }
    qsort(tmp, m, 2 * sizeof(double), cmp_pair);
    for (int j = 0; j < k; ++j) {
      out_s[b * k + j] = j < m ? (float)tmp[2 * j] : -INFINITY;
      out_i[b * k + j] = j < m ? (int32_t)tmp[2 * j + 1] : -1;
    }
  }
  free(tmp);
  free(ls);
  free(li);
  free(qf);
  return 0;
}
