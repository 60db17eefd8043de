/*
 * gram_oracle.c — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Factorised Gram of the join matrix of two SplitMix64 tables, for the
 * full-size parity tests (SURVEY.md §8c "large-config oracle"):
 *   J^T J = [[ sum_g m2g A_g^T A_g ,  sum_g (1^T A_g)^T (1^T B_g) ],
 *            [        (sym)        ,  sum_g m1g B_g^T B_g        ]]
 * computed in O(m1 n1^2 + m2 n2^2) without touching the join, with the table
 * entries regenerated from their seeds (element k = row * cols + col,
 * u = ((mix64(seed + (k+1) * 0x9E3779B97F4A7C15) >> 11) + 0.5) * 2^-53, the
 * recipe of oracle/datagen.py).  Keys (optional, sorted int64) define the
 * groups exactly as SPEC.md:202-207.  Row blocks are reduced by OpenMP threads
 * into private Grams that are summed in a fixed order (deterministic).
 * R_oracle = chol(J^T J)^T, sigma_oracle = sqrt(eig(J^T J)) (oracle/factorised.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline double unif(uint64_t seed, uint64_t k) {
  return ((double)(mix64(seed + (k + 1) * 0x9E3779B97F4A7C15ull) >> 11) + 0.5) * 1.1102230246251565e-16;
}

#define BLK 256

/* G[0:n,0:n] += sum_i w_i x_i x_i^T over rows of a SplitMix table (upper triangle). */
/* Row r of the table as held by the caller is generated row perm[r] (perm == NULL:
 * identity) -- tables whose rows were permuted by a stable key sort (C3 recipe). */
static inline uint64_t grow(const int64_t* perm, int64_t r) { return perm ? (uint64_t)perm[r] : (uint64_t)r; }

static void weighted_gram(uint64_t seed, int64_t m, int n, const double* w, double* G, int ld, int off,
                          const int64_t* perm) {
  int nt = omp_get_max_threads();
  double* priv = (double*)calloc((size_t)nt * n * n, sizeof(double));
  int64_t nblk = (m + BLK - 1) / BLK;
#pragma omp parallel
  {
    int tid = omp_get_thread_num();
    double* Gp = priv + (size_t)tid * n * n;
    double* x = (double*)malloc(sizeof(double) * BLK * n);
#pragma omp for schedule(static)
    for (int64_t b = 0; b < nblk; ++b) {
      int64_t r0 = b * BLK, r1 = r0 + BLK < m ? r0 + BLK : m;
      int rows = (int)(r1 - r0);
      for (int i = 0; i < rows; ++i) {
        double sw = w ? w[r0 + i] : 1.0;
        for (int c = 0; c < n; ++c) x[i * n + c] = unif(seed, grow(perm, r0 + i) * n + c);
        (void)sw;
      }
      int i = 0;
      for (; i + 4 <= rows; i += 4) {  /* 4 rows per pass: 4x fewer accumulator loads */
        const double* x0 = x + i * n; const double* x1 = x0 + n; const double* x2 = x1 + n; const double* x3 = x2 + n;
        double w0 = w ? w[r0 + i] : 1.0, w1 = w ? w[r0 + i + 1] : 1.0;
        double w2 = w ? w[r0 + i + 2] : 1.0, w3 = w ? w[r0 + i + 3] : 1.0;
        for (int p = 0; p < n; ++p) {
          const double a0 = w0 * x0[p], a1 = w1 * x1[p], a2 = w2 * x2[p], a3 = w3 * x3[p];
          double* gr = Gp + p * n;
          for (int q = p; q < n; ++q) gr[q] += a0 * x0[q] + a1 * x1[q] + a2 * x2[q] + a3 * x3[q];
        }
      }
      for (; i < rows; ++i) {
        const double sw = w ? w[r0 + i] : 1.0;
        const double* xi = x + i * n;
        for (int p = 0; p < n; ++p) {
          const double a = sw * xi[p];
          double* gr = Gp + p * n;
          for (int q = p; q < n; ++q) gr[q] += a * xi[q];
        }
      }
    }
    free(x);
  }
  for (int t = 0; t < nt; ++t)
    for (int p = 0; p < n; ++p)
      for (int q = p; q < n; ++q) G[(off + p) * ld + off + q] += priv[(size_t)t * n * n + p * n + q];
  free(priv);
}

/* Per-row weights (count of the other side's rows with the same key) and the
 * cross term sum_g colsum(A_g)^T colsum(B_g). */
int jq_oracle_gram_perm(uint64_t seed_a, int64_t m1, int n1, const int64_t* ka, const int64_t* pa,
                        uint64_t seed_b, int64_t m2, int n2, const int64_t* kb, const int64_t* pb, double* G) {
  const int n = n1 + n2;
  memset(G, 0, sizeof(double) * n * n);
  double* wa = NULL;
  double* wb = NULL;
  double* sa = (double*)calloc(n1 > 0 ? n1 : 1, sizeof(double));
  double* sb = (double*)calloc(n2 > 0 ? n2 : 1, sizeof(double));
  if (ka) {
    wa = (double*)calloc(m1 > 0 ? m1 : 1, sizeof(double));
    wb = (double*)calloc(m2 > 0 ? m2 : 1, sizeof(double));
    int64_t i = 0, j = 0;
    while (i < m1 && j < m2) {
      if (ka[i] < kb[j]) { ++i; continue; }
      if (kb[j] < ka[i]) { ++j; continue; }
      int64_t key = ka[i], i1 = i, j1 = j;
      while (i1 < m1 && ka[i1] == key) ++i1;
      while (j1 < m2 && kb[j1] == key) ++j1;
      for (int64_t r = i; r < i1; ++r) wa[r] = (double)(j1 - j);
      for (int64_t r = j; r < j1; ++r) wb[r] = (double)(i1 - i);
      /* cross term of this group (sequential, fixed order) */
      memset(sa, 0, sizeof(double) * n1);
      memset(sb, 0, sizeof(double) * n2);
      for (int64_t r = i; r < i1; ++r)
        for (int c = 0; c < n1; ++c) sa[c] += unif(seed_a, grow(pa, r) * n1 + c);
      for (int64_t r = j; r < j1; ++r)
        for (int c = 0; c < n2; ++c) sb[c] += unif(seed_b, grow(pb, r) * n2 + c);
      for (int p = 0; p < n1; ++p)
        for (int q = 0; q < n2; ++q) G[p * n + n1 + q] += sa[p] * sb[q];
      i = i1;
      j = j1;
    }
  } else {
    /* one group: column sums in parallel blocks, fixed-order reduction */
    int nt = omp_get_max_threads();
    double* part = (double*)calloc((size_t)nt * (n1 + n2 + 1), sizeof(double));
#pragma omp parallel
    {
      double* p = part + (size_t)omp_get_thread_num() * (n1 + n2 + 1);
#pragma omp for schedule(static)
      for (int64_t r = 0; r < m1; ++r)
        for (int c = 0; c < n1; ++c) p[c] += unif(seed_a, grow(pa, r) * n1 + c);
#pragma omp for schedule(static)
      for (int64_t r = 0; r < m2; ++r)
        for (int c = 0; c < n2; ++c) p[n1 + c] += unif(seed_b, grow(pb, r) * n2 + c);
    }
    for (int t = 0; t < nt; ++t) {
      for (int c = 0; c < n1; ++c) sa[c] += part[(size_t)t * (n1 + n2 + 1) + c];
      for (int c = 0; c < n2; ++c) sb[c] += part[(size_t)t * (n1 + n2 + 1) + n1 + c];
    }
    free(part);
    for (int p = 0; p < n1; ++p)
      for (int q = 0; q < n2; ++q) G[p * n + n1 + q] = sa[p] * sb[q];
  }
  /* weighted diagonal blocks: A rows weighted by m2g, B rows by m1g */
  double* G1 = (double*)calloc((size_t)n * n, sizeof(double));
  if (ka) {
    weighted_gram(seed_a, m1, n1, wa, G1, n, 0, pa);
    weighted_gram(seed_b, m2, n2, wb, G1, n, n1, pb);
  } else {
    weighted_gram(seed_a, m1, n1, NULL, G1, n, 0, pa);
    weighted_gram(seed_b, m2, n2, NULL, G1, n, n1, pb);
    for (int p = 0; p < n1; ++p) for (int q = p; q < n1; ++q) G1[p * n + q] *= (double)m2;
    for (int p = n1; p < n; ++p) for (int q = p; q < n; ++q) G1[p * n + q] *= (double)m1;
  }
  for (int p = 0; p < n; ++p)
    for (int q = p; q < n; ++q) G[p * n + q] += G1[p * n + q];
  for (int p = 0; p < n; ++p)
    for (int q = 0; q < p; ++q) G[p * n + q] = G[q * n + p];
  free(G1); free(sa); free(sb); free(wa); free(wb);
  return 0;
}

int jq_oracle_gram(uint64_t seed_a, int64_t m1, int n1, const int64_t* ka, uint64_t seed_b, int64_t m2,
                   int n2, const int64_t* kb, double* G) {
  return jq_oracle_gram_perm(seed_a, m1, n1, ka, NULL, seed_b, m2, n2, kb, NULL, G);
}
