/*
 * O1 -- CPU ORACLE (TEST INFRASTRUCTURE ONLY).
 *
 * Plain, slow, obviously correct classical products over GF(p) and GF(p^2), in 64-bit
 * integers.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.  It shares no code, header, table or constant with the CUDA path.
 *
 * What it computes is the plain definition the paper's method reaches exactly
 * (Theorem thm:complexitybound, proves Alg. alg:MIAHMM is exact):
 *
 *   Lemma lem:transp: phi(A)_{ij} = phi(a_{ji}).  Hence
 *   (A phi(A))_{ij} = sum_t a_{it} * phi(a_{jt}).
 *
 *   - phi = transpose over GF(p):           C[i][j] = sum_t A[i][t] A[j][t]      mod p
 *   - phi = conjugate transpose over GF(p^2) = GF(p)[i]/(i^2+1), conj(x+iy) = x-iy
 *     (Frobenius):
 *        Re C[i][j] = sum_t x_it x_jt + y_it y_jt                                mod p
 *        Im C[i][j] = sum_t y_it x_jt - x_it y_jt                                mod p
 *   - phi = conjugate transpose over the quaternions H_GF(p) (§6.2): oracle_syrk_q_rows.
 *   - Low/Up: only i >= j is written (diagonal included).
 *   - A general product C = A B^T (the paper's A phi(B) over GF(p)) for gemm parity.
 *
 * Inputs are reduced mod p first (non-canonical inputs are interpreted mod p).
 * For p <= 2^16 a term is < 2^32 and a k < 2^32 sum fits in uint64 with no intermediate
 * reduction; for larger p each term is reduced before summing.
 *
 * Build: gcc -O3 -march=native -fopenmp -shared -fPIC oracle.c -o liboracle.so
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ROWP(base, ld, i) ((base) + (size_t)(i) * (size_t)(ld))

/* reduced copy of an m x k matrix with leading dimension ld (elements of width w u32) */
static uint32_t *reduced_copy(const uint32_t *A, int64_t m, int64_t k, int64_t ld, int w,
                              uint32_t p) {
  uint32_t *R = (uint32_t *)malloc((size_t)(m * k * w > 0 ? m * k * w : 1) * sizeof(uint32_t));
  if (!R) return NULL;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; i++)
    for (int64_t t = 0; t < k * w; t++) R[(size_t)i * k * w + t] = A[(size_t)i * ld * w + t] % p;
  return R;
}

static uint64_t dot_mod(const uint32_t *a, const uint32_t *b, int64_t k, uint32_t p) {
  uint64_t s = 0;
  if (p <= 65536u) {
    for (int64_t t = 0; t < k; t++) s += (uint64_t)a[t] * (uint64_t)b[t];
  } else {
    for (int64_t t = 0; t < k; t++) s += ((uint64_t)a[t] * (uint64_t)b[t]) % p;
  }
  return s % p;
}

/* Low(A A^T) mod p for rows i in [r0, r1), all j <= i.  A: m x k, lda; C: ldc. Returns 0 ok. */
int oracle_syrk_t_rows(int64_t m, int64_t k, uint32_t p, const uint32_t *A, int64_t lda,
                       uint32_t *C, int64_t ldc, int64_t r0, int64_t r1) {
  if (m < 0 || k < 0 || p < 2 || r0 < 0 || r1 > m) return 1;
  uint32_t *R = reduced_copy(A, m, k, lda, 1, p);
  if (!R) return 2;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = r0; i < r1; i++) {
    const uint32_t *ai = R + (size_t)i * k;
    for (int64_t j = 0; j <= i; j++)
      ROWP(C, ldc, i)[j] = (uint32_t)dot_mod(ai, R + (size_t)j * k, k, p);
  }
  free(R);
  return 0;
}

int oracle_syrk_t(int64_t m, int64_t k, uint32_t p, const uint32_t *A, int64_t lda,
                  uint32_t *C, int64_t ldc) {
  return oracle_syrk_t_rows(m, k, p, A, lda, C, ldc, 0, m);
}

/* Full C = A B^T mod p.  A: m x k (lda), B: n x k (ldb), C: m x n (ldc). */
int oracle_gemm_nt(int64_t m, int64_t n, int64_t k, uint32_t p, const uint32_t *A, int64_t lda,
                   const uint32_t *B, int64_t ldb, uint32_t *C, int64_t ldc) {
  if (m < 0 || n < 0 || k < 0 || p < 2) return 1;
  uint32_t *RA = reduced_copy(A, m, k, lda, 1, p);
  uint32_t *RB = reduced_copy(B, n, k, ldb, 1, p);
  if (!RA || !RB) { free(RA); free(RB); return 2; }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < m; i++)
    for (int64_t j = 0; j < n; j++)
      ROWP(C, ldc, i)[j] = (uint32_t)dot_mod(RA + (size_t)i * k, RB + (size_t)j * k, k, p);
  free(RA); free(RB);
  return 0;
}

/* Low(A A^H) over GF(p^2) = GF(p)[i]/(i^2+1) for rows [r0, r1).  A and C hold interleaved
 * (re, im) u32 pairs; lda/ldc count GF(p^2) elements. */
int oracle_syrk_h_rows(int64_t m, int64_t k, uint32_t p, const uint32_t *A, int64_t lda,
                       uint32_t *C, int64_t ldc, int64_t r0, int64_t r1) {
  if (m < 0 || k < 0 || p < 2 || r0 < 0 || r1 > m) return 1;
  const int big = p > 65536u;   /* reduce every term first so the uint64 sums cannot overflow */
  uint32_t *R = reduced_copy(A, m, k, lda, 2, p);
  if (!R) return 2;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = r0; i < r1; i++) {
    const uint32_t *ai = R + (size_t)i * k * 2;
    for (int64_t j = 0; j <= i; j++) {
      const uint32_t *aj = R + (size_t)j * k * 2;
      uint64_t re = 0, im_pos = 0, im_neg = 0;  /* (x+iy)(x'-iy') = xx'+yy' + i(yx' - xy') */
      for (int64_t t = 0; t < k; t++) {
        uint64_t x = ai[2 * t], y = ai[2 * t + 1], xp = aj[2 * t], yp = aj[2 * t + 1];
        if (big) {
          re += (x * xp) % p + (y * yp) % p;
          im_pos += (y * xp) % p;
          im_neg += (x * yp) % p;
        } else {
          re += x * xp + y * yp;
          im_pos += y * xp;
          im_neg += x * yp;
        }
      }
      uint64_t a = im_pos % p, b = im_neg % p;
      ROWP(C, ldc * 2, i)[2 * j] = (uint32_t)(re % p);
      ROWP(C, ldc * 2, i)[2 * j + 1] = (uint32_t)((a + p - b) % p);
    }
  }
  free(R);
  return 0;
}

int oracle_syrk_h(int64_t m, int64_t k, uint32_t p, const uint32_t *A, int64_t lda,
                  uint32_t *C, int64_t ldc) {
  return oracle_syrk_h_rows(m, k, p, A, lda, C, ldc, 0, m);
}

/* Low(M M^H) over the quaternions H_K, K = GF(p) (§6.2, ssec:quaternions, 1532-1560):
 * q = x1 + x2 i + x3 j + x4 k with i^2 = j^2 = k^2 = ijk = -1, conj(q) = x1 - x2 i - x3 j - x4 k,
 * (M M^H)_{ij} = sum_t M_it conj(M_jt) (Lemma lem:transp, the product taken in this order).
 * With the multiplication table w1..w4 of PAPER.md:1553-1558 and y = conj(x'):
 *   w1 = x1x1' + x2x2' + x3x3' + x4x4'
 *   w2 = x2x1' - x1x2' + x4x3' - x3x4'
 *   w3 = x3x1' - x1x3' + x2x4' - x4x2'
 *   w4 = x4x1' - x1x4' + x3x2' - x2x3'
 * M and C hold 4 interleaved u32 per element; ldm/ldc count quaternions.  Rows [r0, r1). */
int oracle_syrk_q_rows(int64_t m, int64_t k, uint32_t p, const uint32_t *M, int64_t ldm,
                       uint32_t *C, int64_t ldc, int64_t r0, int64_t r1) {
  if (m < 0 || k < 0 || p < 2 || r0 < 0 || r1 > m) return 1;
  const int big = p > 65536u;
  uint32_t *R = reduced_copy(M, m, k, ldm, 4, p);
  if (!R) return 2;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = r0; i < r1; i++) {
    const uint32_t *qi = R + (size_t)i * k * 4;
    for (int64_t j = 0; j <= i; j++) {
      const uint32_t *qj = R + (size_t)j * k * 4;
      uint64_t pos[4] = {0, 0, 0, 0}, neg[4] = {0, 0, 0, 0};
      for (int64_t t = 0; t < k; t++) {
        const uint64_t x1 = qi[4 * t], x2 = qi[4 * t + 1], x3 = qi[4 * t + 2], x4 = qi[4 * t + 3];
        const uint64_t y1 = qj[4 * t], y2 = qj[4 * t + 1], y3 = qj[4 * t + 2], y4 = qj[4 * t + 3];
        uint64_t pp[4][2] = {{x1 * y1 + x2 * y2, x3 * y3 + x4 * y4},
                             {x2 * y1, x4 * y3}, {x3 * y1, x2 * y4}, {x4 * y1, x3 * y2}};
        uint64_t nn[4][2] = {{0, 0}, {x1 * y2, x3 * y4}, {x1 * y3, x4 * y2}, {x1 * y4, x2 * y3}};
        for (int c = 0; c < 4; c++) {
          if (big) {
            pos[c] += pp[c][0] % p + pp[c][1] % p;
            neg[c] += nn[c][0] % p + nn[c][1] % p;
          } else {
            pos[c] += pp[c][0] + pp[c][1];
            neg[c] += nn[c][0] + nn[c][1];
          }
        }
      }
      for (int c = 0; c < 4; c++)
        ROWP(C, ldc * 4, i)[4 * j + c] = (uint32_t)((pos[c] % p + p - neg[c] % p) % p);
    }
  }
  free(R);
  return 0;
}

/* number of OpenMP threads the oracle runs with (for the cpu_baseline 'cores' field) */
int oracle_num_threads(void) {
  int n = 1;
#ifdef _OPENMP
#pragma omp parallel
  {
#pragma omp single
    n = omp_get_num_threads();
  }
#endif
  return n;
}
