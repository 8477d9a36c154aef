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

/* ------------------------------------------------------------------------------------------
 * AMX-BF16 variant of the fp32-accumulation search (built only with -mamx-tile -mamx-bf16):
 * the CPU baseline on hosts that have Intel AMX (Sapphire Rapids and later), i.e. the strongest
 * brute-force CPU path this oracle can offer ("AMX-BF16 where available").
 * TDPBF16PS multiplies bf16 pairs exactly and accumulates in fp32, so scores agree with the
 * scalar fp32 path up to the summation order. Corpus rows are the A operand straight from the
 * row-major matrix (16 rows x 32 dims = one tile, row stride 2*D bytes); queries are packed
 * once into the VNNI B layout (pairs of dims interleaved per query), 16 queries per tile. Each
 * 32-row block of a thread's corpus range is multiplied against two query tiles at a time into
 * four 16x16 fp32 accumulator tiles, which are stored and filtered against every query's
 * current k-th score (AVX-512 compare of 16 queries at once), inserting only what beats it.
 * ------------------------------------------------------------------------------------------ */
#if defined(__AMX_BF16__) && defined(__AMX_TILE__) && defined(__AVX512F__)
#include <immintrin.h>
#include <sys/syscall.h>
#include <unistd.h>

typedef struct {
  uint8_t palette_id, start_row, reserved[14];
  uint16_t colsb[16];
  uint8_t rows[16];
} tsv_tilecfg;

/* 1 when this process may use AMX tiles (Linux grants XTILEDATA per process on request). */
int tsv_oracle_amx_available(void) {
  if (!__builtin_cpu_supports("amx-bf16")) return 0;
  return syscall(SYS_arch_prctl, 0x1023 /* ARCH_REQ_XCOMP_PERM */, 18 /* XTILEDATA */) == 0;
}

static void amx_configure(void) {
  tsv_tilecfg cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.palette_id = 1;
  for (int t = 0; t < 8; ++t) {
    cfg.colsb[t] = 64;
    cfg.rows[t] = 16;
  }
  _tile_loadconfig(&cfg);
}

static inline void filter_tile(const float* tile /* [16 rows][16 queries] */, int64_t row0,
                               int nrows, int64_t q0, int64_t B, float* thr, double* my_s,
                               int32_t* my_i, int k, int64_t id_offset) {
  const __mmask16 qmask = (q0 + 16 <= B) ? (__mmask16)0xFFFF : (__mmask16)((1u << (B - q0)) - 1u);
  const __m512 th = _mm512_loadu_ps(thr + q0);
  for (int m = 0; m < nrows; ++m) {
    const __m512 v = _mm512_loadu_ps(tile + 16 * m);
    __mmask16 hit = _mm512_mask_cmp_ps_mask(qmask, v, th, _CMP_GT_OQ);
    if (!hit) continue;
    while (hit) {
      const int n = __builtin_ctz(hit);
      hit &= hit - 1;
      const int64_t qi = q0 + n;
      const double sc = tile[16 * m + n];
      double* s = my_s + qi * k;
      if (sc > s[k - 1]) {
        list_insert(s, my_i + qi * k, k, sc, (int32_t)(row0 + m + id_offset));
        thr[qi] = (float)s[k - 1];
      }
    }
  }
}

int tsv_oracle_search_amx(const uint16_t* q, const uint16_t* c, int64_t B, int64_t N, int D,
                          int k, int nthreads, int64_t id_offset, float* out_s, int32_t* out_i) {
  if (B <= 0 || k <= 0 || D <= 0) return 1;
  if (D % 32 != 0) return 3; /* the caller uses the AVX path */
  if (nthreads <= 0) nthreads = omp_get_max_threads();
  const int KB = D / 32;
  const int64_t G = ((B + 31) / 32) * 2; /* query tiles, padded to pairs */
  /* packed queries: [G][KB][16 dim pairs][16 queries][2] */
  uint16_t* qp = (uint16_t*)aligned_alloc(64, (size_t)G * KB * 1024);
  if (!qp) return 2;
  for (int64_t g = 0; g < G; ++g)
    for (int kb = 0; kb < KB; ++kb) {
      uint16_t* t = qp + ((size_t)g * KB + kb) * 512;
      for (int kp = 0; kp < 16; ++kp)
        for (int n = 0; n < 16; ++n) {
          const int64_t qi = g * 16 + n;
          const int d = kb * 32 + 2 * kp;
          t[kp * 32 + 2 * n] = qi < B ? q[qi * D + d] : 0;
          t[kp * 32 + 2 * n + 1] = qi < B ? q[qi * D + d + 1] : 0;
        }
    }
  double* ls = (double*)malloc(sizeof(double) * (size_t)nthreads * B * k);
  int32_t* li = (int32_t*)malloc(sizeof(int32_t) * (size_t)nthreads * B * k);
  float* thr_all = (float*)malloc(sizeof(float) * (size_t)nthreads * (B + 16));
  if (!ls || !li || !thr_all) return 2;
  for (size_t i = 0; i < (size_t)nthreads * B * k; ++i) {
    ls[i] = -INFINITY;
    li[i] = -1;
  }
  int failed = 0;
#pragma omp parallel num_threads(nthreads)
  {
    const int t = omp_get_thread_num();
    const int nt = omp_get_num_threads();
    if (syscall(SYS_arch_prctl, 0x1023, 18) != 0) {
#pragma omp atomic write
      failed = 1;
    }
#pragma omp barrier
    if (!failed) {
      amx_configure();
      const int64_t r0 = N * t / nt, r1 = N * (t + 1) / nt;
      double* my_s = ls + (size_t)t * B * k;
      int32_t* my_i = li + (size_t)t * B * k;
      float* thr = thr_all + (size_t)t * (B + 16);
      for (int64_t i = 0; i < B + 16; ++i) thr[i] = -INFINITY;
      float acc[4][256] __attribute__((aligned(64)));
      uint16_t* tail = (uint16_t*)aligned_alloc(64, (size_t)32 * D * 2);
      for (int64_t rb = r0; rb < r1; rb += 32) {
        const int nr = (int)((r1 - rb) < 32 ? (r1 - rb) : 32);
        const uint16_t* a = c + (size_t)rb * D;
        if (nr < 32) { /* ragged last block: zero-padded copy */
          memset(tail, 0, (size_t)32 * D * 2);
          memcpy(tail, a, (size_t)nr * D * 2);
          a = tail;
        }
        for (int64_t g = 0; g < G; g += 2) {
          _tile_zero(0);
          _tile_zero(1);
          _tile_zero(2);
          _tile_zero(3);
          const uint16_t* b0 = qp + (size_t)g * KB * 512;
          const uint16_t* b1 = b0 + (size_t)KB * 512;
          for (int kb = 0; kb < KB; ++kb) {
            _tile_loadd(4, a + kb * 32, D * 2);
            _tile_loadd(5, a + (size_t)16 * D + kb * 32, D * 2);
            _tile_loadd(6, b0 + (size_t)kb * 512, 64);
            _tile_loadd(7, b1 + (size_t)kb * 512, 64);
            _tile_dpbf16ps(0, 4, 6);
            _tile_dpbf16ps(1, 5, 6);
            _tile_dpbf16ps(2, 4, 7);
            _tile_dpbf16ps(3, 5, 7);
          }
          _tile_stored(0, acc[0], 64);
          _tile_stored(1, acc[1], 64);
          _tile_stored(2, acc[2], 64);
          _tile_stored(3, acc[3], 64);
          const int n_lo = nr < 16 ? nr : 16, n_hi = nr > 16 ? nr - 16 : 0;
          if (g * 16 < B) {
            filter_tile(acc[0], rb, n_lo, g * 16, B, thr, my_s, my_i, k, id_offset);
            filter_tile(acc[1], rb + 16, n_hi, g * 16, B, thr, my_s, my_i, k, id_offset);
          }
          if ((g + 1) * 16 < B) {
            filter_tile(acc[2], rb, n_lo, (g + 1) * 16, B, thr, my_s, my_i, k, id_offset);
            filter_tile(acc[3], rb + 16, n_hi, (g + 1) * 16, B, thr, my_s, my_i, k, id_offset);
          }
        }
      }
      free(tail);
      _tile_release();
    }
  }
  if (failed) {
    free(qp);
    free(ls);
    free(li);
    free(thr_all);
    return 4;
  }
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
  free(qp);
  free(ls);
  free(li);
  free(thr_all);
  return 0;
}
#endif
