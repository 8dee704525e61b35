/* C/OpenMP restatement of the O(R^2) stages of one NSGA-III generation
 * (TEST INFRASTRUCTURE / CPU BASELINE ONLY -- never linked into the product).
 *
 * SURVEY.md 8(d) asks for a "fair multi-core CPU" figure beside the numpy
 * restatement: the two quadratic stages, restated in plain C over all host
 * cores, with the numpy oracle as their checker (tests/test_oracle_c.py):
 *
 *   oro_nds        non_dominated_sort with stop_at (
 *                  oracle/manyobj_ref/dominance.py:36): dominator counts by an
 *                  all-pairs sweep, then peel front by front, subtracting the
 *                  front's domination of every unranked row (count-decrement,
 *                  no bit matrix: O(R^2 m) total, any R).  Ranks are exact
 *                  integers -> bit-identical to the oracle.
 *   oro_associate  canonical FP32 association (SPEC.md:349-357 with the pins
 *                  of oracle/manyobj_ref/niche.py:168 associate_canonical):
 *                  t = (((f0 z0) + f1 z1) + ...) in FP32 without contraction,
 *                  first maximum over refs in shuffled order, d = sqrt of the
 *                  FP32 sum of squared residuals.  Built with
 *                  -ffp-contract=off so the FP32 values are the oracle's.
 *
 * Rows are split over OpenMP threads; the inner loops run over SoA columns so
 * the compiler vectorises them (target_clones: AVX-512 / AVX2 / baseline,
 * chosen at load time on the host it runs on).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define ORO_MAXM 16
#define CLONES __attribute__((target_clones("avx512f", "avx2", "default")))

/* F is row-major R x m; the sweeps read SoA copies. */
static float* to_soa(const float* F, int64_t R, int m) {
  float* S = (float*)malloc(sizeof(float) * (size_t)R * (size_t)m + 64);
  if (!S) return NULL;
  for (int64_t i = 0; i < R; ++i)
    for (int k = 0; k < m; ++k) S[(size_t)k * R + i] = F[i * m + k];
  return S;
}

/* number of rows i in [0, n) of the SoA block A (stride lda) that dominate the point b */
static inline __attribute__((always_inline)) int count_dominators(const float* A, int64_t lda, int64_t n,
                                                                 const float* b, int m) {
  int c = 0;
  for (int64_t i = 0; i < n; ++i) {
    int le = 1, lt = 0;
    for (int k = 0; k < m; ++k) {
      const float a = A[(size_t)k * lda + i];
      le &= a <= b[k];
      lt |= a < b[k];
    }
    c += le & lt;
  }
  return c;
}

#define ORO_COUNT_CASE(MM) \
  case MM: return count_dominators(A, lda, n, b, MM);

CLONES static int count_dom_m(const float* A, int64_t lda, int64_t n, const float* b, int m) {
  switch (m) {
    ORO_COUNT_CASE(1) ORO_COUNT_CASE(2) ORO_COUNT_CASE(3) ORO_COUNT_CASE(4) ORO_COUNT_CASE(5)
    ORO_COUNT_CASE(6) ORO_COUNT_CASE(7) ORO_COUNT_CASE(8) ORO_COUNT_CASE(9) ORO_COUNT_CASE(10)
    ORO_COUNT_CASE(11) ORO_COUNT_CASE(12) ORO_COUNT_CASE(13) ORO_COUNT_CASE(14) ORO_COUNT_CASE(15)
    ORO_COUNT_CASE(16)
    default: return count_dominators(A, lda, n, b, m);
  }
}

/* Dominator counts of `nrows` rows (indices `rows`, or 0..nrows-1 when rows == NULL) against all R
 * rows: the sampled form the CPU baseline extrapolates from when R is large. */
int oro_dominator_counts(const float* F, int64_t R, int m, const int64_t* rows, int64_t nrows, int32_t* cnt,
                         int threads) {
  if (m < 1 || m > ORO_MAXM || R < 0) return 2;
  float* S = to_soa(F, R, m);
  if (!S) return 7;
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t q = 0; q < nrows; ++q) {
    const int64_t j = rows ? rows[q] : q;
    float b[ORO_MAXM];
    for (int k = 0; k < m; ++k) b[k] = F[j * m + k];
    cnt[q] = count_dom_m(S, R, R, b, m);
  }
  free(S);
  return 0;
}

/* non_dominated_sort(F, stop_at): ranks[i] = front index, or 2^31-1 (DROPPED) for rows past the front
 * where the cumulative size first reaches stop_at (stop_at <= 0: peel everything). */
int oro_nds(const float* F, int64_t R, int m, int64_t stop_at, int64_t* ranks, int threads) {
  if (m < 1 || m > ORO_MAXM || R < 0) return 2;
  float* S = to_soa(F, R, m);
  int32_t* cnt = (int32_t*)malloc(sizeof(int32_t) * (size_t)(R + 1));
  float* front = (float*)malloc(sizeof(float) * (size_t)R * (size_t)m + 64);
  int64_t* fidx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(R + 1));
  if (!S || !cnt || !front || !fidx) {
    free(S); free(cnt); free(front); free(fidx);
    return 7;
  }
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t j = 0; j < R; ++j) {
    float b[ORO_MAXM];
    for (int k = 0; k < m; ++k) b[k] = F[j * m + k];
    cnt[j] = count_dom_m(S, R, R, b, m);
  }
  for (int64_t i = 0; i < R; ++i) ranks[i] = -2;          /* unranked */
  int64_t cum = 0;
  for (int64_t level = 0;; ++level) {
    int64_t nf = 0;
    for (int64_t i = 0; i < R; ++i)
      if (ranks[i] == -2 && cnt[i] == 0) fidx[nf++] = i;
    if (nf == 0) break;
    for (int64_t q = 0; q < nf; ++q) {
      ranks[fidx[q]] = level;
      for (int k = 0; k < m; ++k) front[(size_t)k * nf + q] = F[fidx[q] * m + k];
    }
    cum += nf;
    if (stop_at > 0 && cum >= stop_at) break;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t j = 0; j < R; ++j) {
      if (ranks[j] != -2) continue;
      float b[ORO_MAXM];
      for (int k = 0; k < m; ++k) b[k] = F[j * m + k];
      cnt[j] -= count_dom_m(front, nf, nf, b, m);
    }
  }
  for (int64_t i = 0; i < R; ++i)
    if (ranks[i] == -2) ranks[i] = 2147483647;
  free(S); free(cnt); free(front); free(fidx);
  return 0;
}

/* t[p] = canonical FP32 dot of f with ref p (SoA zs, refs in shuffled order), no contraction */
static inline __attribute__((always_inline)) void dots(const float* zs, int64_t w, const float* f, int m,
                                                       float* t, int64_t p0, int64_t pn) {
  for (int64_t p = 0; p < pn; ++p) t[p] = f[0] * zs[p0 + p];
  for (int k = 1; k < m; ++k)
    for (int64_t p = 0; p < pn; ++p) t[p] = t[p] + f[k] * zs[(size_t)k * w + p0 + p];
}

#define ORO_DOT_CASE(MM) \
  case MM: dots(zs, w, f, MM, t, p0, pn); return;

CLONES static void dots_m(const float* zs, int64_t w, const float* f, int m, float* t, int64_t p0, int64_t pn) {
  switch (m) {
    ORO_DOT_CASE(1) ORO_DOT_CASE(2) ORO_DOT_CASE(3) ORO_DOT_CASE(4) ORO_DOT_CASE(5) ORO_DOT_CASE(6)
    ORO_DOT_CASE(7) ORO_DOT_CASE(8) ORO_DOT_CASE(9) ORO_DOT_CASE(10) ORO_DOT_CASE(11) ORO_DOT_CASE(12)
    ORO_DOT_CASE(13) ORO_DOT_CASE(14) ORO_DOT_CASE(15) ORO_DOT_CASE(16)
    default: dots(zs, w, f, m, t, p0, pn); return;
  }
}

/* Fn: R x m rows (row-major); zhat: w x m unit directions; pos_ref[j] = shuffled position of ref j.
 * For the `nrows` rows listed (all when rows == NULL): pi = ref index of the first maximum of the
 * canonical dot in shuffled order, d = perpendicular distance (FP32). */
int oro_associate(const float* Fn, int64_t R, int m, const float* zhat, int64_t w, const int64_t* pos_ref,
                  const int64_t* rows, int64_t nrows, int64_t* pi, float* d, int threads) {
  if (m < 1 || m > ORO_MAXM || w < 1 || R < 0) return 2;
  float* zs = (float*)malloc(sizeof(float) * (size_t)w * (size_t)m + 64);
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)w);
  if (!zs || !perm) {
    free(zs); free(perm);
    return 7;
  }
  for (int64_t j = 0; j < w; ++j) {
    const int64_t p = pos_ref[j];
    if (p < 0 || p >= w) { free(zs); free(perm); return 3; }
    perm[p] = j;
    for (int k = 0; k < m; ++k) zs[(size_t)k * w + p] = zhat[j * m + k];
  }
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
  {
    float t[512];
#pragma omp for schedule(dynamic, 8)
    for (int64_t q = 0; q < nrows; ++q) {
      const int64_t i = rows ? rows[q] : q;
      const float* f = Fn + i * m;
      float best = -INFINITY;
      int64_t bp = 0;
      for (int64_t p0 = 0; p0 < w; p0 += 512) {
        const int64_t pn = w - p0 < 512 ? w - p0 : 512;
        dots_m(zs, w, f, m, t, p0, pn);
        for (int64_t p = 0; p < pn; ++p)
          if (t[p] > best) { best = t[p]; bp = p0 + p; }
      }
      float s = 0.0f;
      for (int k = 0; k < m; ++k) {
        const float e = f[k] - best * zs[(size_t)k * w + bp];
        s = k ? s + e * e : e * e;
      }
      pi[q] = perm[bp];
      d[q] = sqrtf(s);
    }
  }
  free(zs); free(perm);
  return 0;
}

int oro_max_threads(void) { return omp_get_max_threads(); }
