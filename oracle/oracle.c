/*
 * oracle.c -- plain, slow, obviously-correct FP64 CPU oracle for the VIF
 * (Vecchia-inducing-points full-scale) factor and Gaussian negative
 * log-likelihood of arXiv 2507.05064.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, helper or constant with the CUDA product path under
 * paper_2507_05064_b200/ and neither imports the other.
 *
 * Citations: "P:NNN" is a line of PAPER.md (the paper's LaTeX source).
 *   covariance family ............ P:42 (c_theta), P:503-505 (ARD q_lambda)
 *   predictive process, Sigma_l .. P:72-80
 *   residual Vecchia B, D, A_i ... P:85-97 (Eq. D_A_Vecchia)
 *   L_dagger ..................... P:99-106
 *   Woodbury, M (Eq. def_M) ...... P:109-118
 *   Sylvester determinant ........ P:119-124
 * Readings of the paper where it is silent are listed in DESIGN.md (c1..c17):
 *   c1 kernel formula, c2 nugget by index identity, c3 jitter on K(Z,Z),
 *   c4 whitened U = (L_m^{-1} K(Z,X))^T stored n x m, c5 0-based small-i rule,
 *   c11 no clamping of D_i, c12 constant term included.
 *
 * Whitened form (c4): with L_m L_m^T = K(Z,Z) + eps I and u_i = L_m^{-1} k(Z, x_i),
 *   Sigma_mn^T Sigma_m^{-1} Sigma_mn = U U^T
 *   C(a,b) = k(x_a,x_b) - u_a.u_b + sigma^2 [a == b]   (P:85-94 residual cov)
 *   A_i = C_{i,N} C_{N,N}^{-1},  D_i = C_ii - A_i C_{N,i}
 *   w_i = u_i - sum_k A_ik u_{N(i)_k},  r_i = y_i - A_i . y_{N(i)}
 *   M_w = I + sum_i w_i w_i^T / D_i  ( = L_m^{-1} M L_m^{-T}, M of P:117 )
 *   logdet Sigma_dagger = sum log D_i + logdet M_w      (det B = 1)
 *   y^T Sigma_dagger^{-1} y = sum r_i^2/D_i - v^T M_w^{-1} v, v = sum w_i r_i / D_i
 *   NLL = n/2 log(2 pi) + 1/2 logdet + 1/2 quad
 *
 * Compiled with plain -O2 (no -ffast-math), OpenMP over rows, static schedule,
 * per-thread partial sums merged in thread-index order (deterministic for a
 * given thread count).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_INVALID 1
#define OR_NOT_PD 2
#define OR_NOMEM 5

typedef struct {
  int32_t family;          /* 0: Matern 1/2, 1: Matern 3/2, 2: Matern 5/2, 3: Gaussian */
  int32_t d;
  double sigma2;           /* marginal variance sigma_1^2 */
  const double *lengthscale; /* d entries (ARD) */
  double nugget;           /* error variance sigma^2 */
  double jitter;           /* eps added to diag K(Z,Z) (reading c3) */
} or_theta;

/* c_theta(a, b) = sigma_1^2 f(r), r = || (a - b) / lambda ||  (reading c1) */
static double or_cov(const or_theta *th, const double *a, const double *b) {
  double r2 = 0.0;
  for (int k = 0; k < th->d; ++k) {
    double t = (a[k] - b[k]) / th->lengthscale[k];
    r2 += t * t;
  }
  double r = sqrt(r2);
  double f;
  switch (th->family) {
    case 0: f = exp(-r); break;
    case 1: f = (1.0 + sqrt(3.0) * r) * exp(-sqrt(3.0) * r); break;
    case 2: f = (1.0 + sqrt(5.0) * r + 5.0 * r2 / 3.0) * exp(-sqrt(5.0) * r); break;
    default: f = exp(-r2); break;
  }
  return th->sigma2 * f;
}

/* In-place lower Cholesky of the leading p x p block of A (row stride lda).
 * Returns -1 on success, else the index of the first non-positive pivot. */
static int or_chol(double *A, int p, int lda) {
  for (int j = 0; j < p; ++j) {
    double s = A[(size_t)j * lda + j];
    for (int k = 0; k < j; ++k) s -= A[(size_t)j * lda + k] * A[(size_t)j * lda + k];
    if (!(s > 0.0)) return j;
    double ljj = sqrt(s);
    A[(size_t)j * lda + j] = ljj;
    for (int i = j + 1; i < p; ++i) {
      double t = A[(size_t)i * lda + j];
      for (int k = 0; k < j; ++k) t -= A[(size_t)i * lda + k] * A[(size_t)j * lda + k];
      A[(size_t)i * lda + j] = t / ljj;
    }
  }
  return -1;
}

/* forward substitution L x = b (L lower, p x p, stride lda); x overwrites b */
static void or_fwd(const double *L, int p, int lda, double *b) {
  for (int i = 0; i < p; ++i) {
    double t = b[i];
    for (int k = 0; k < i; ++k) t -= L[(size_t)i * lda + k] * b[k];
    b[i] = t / L[(size_t)i * lda + i];
  }
}

/* back substitution L^T x = b */
static void or_bwd(const double *L, int p, int lda, double *b) {
  for (int i = p - 1; i >= 0; --i) {
    double t = b[i];
    for (int k = i + 1; k < p; ++k) t -= L[(size_t)k * lda + i] * b[k];
    b[i] = t / L[(size_t)i * lda + i];
  }
}

/* ---- exported: kernel matrix (for the closed-form / library pins) ---- */
int oracle_cov_matrix(const or_theta *th, const double *A, int64_t na, const double *B, int64_t nb,
                      double *out) {
  for (int64_t i = 0; i < na; ++i)
    for (int64_t j = 0; j < nb; ++j) out[i * nb + j] = or_cov(th, A + i * th->d, B + j * th->d);
  return OR_OK;
}

/* Step 1: K_m = K(Z,Z) + eps I, L_m = chol(K_m)   (reading c3) */
static int or_build_Lm(const or_theta *th, const double *Z, int m, double *Lm) {
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b) Lm[(size_t)a * m + b] = or_cov(th, Z + (size_t)a * th->d, Z + (size_t)b * th->d);
  for (int a = 0; a < m; ++a) Lm[(size_t)a * m + a] += th->jitter;
  return or_chol(Lm, m, m) < 0 ? OR_OK : OR_NOT_PD;
}

/* Step 2: u_i = L_m^{-1} k(Z, x_i)   (whitened, reading c4) */
static void or_u_row(const or_theta *th, const double *Z, int m, const double *Lm, const double *x,
                     double *u) {
  for (int a = 0; a < m; ++a) u[a] = or_cov(th, Z + (size_t)a * th->d, x);
  or_fwd(Lm, m, m, u);
}

/* Step 3 for one row i: conditioning set S = (N(i)..., i); C = residual covariance;
 * A_i, D_i per Eq. D_A_Vecchia.  `uS` holds the s whitened rows (s x m).
 * Writes a[0..q-1] (= A_i, q = |N(i)|), returns D_i through *Di.
 * Returns -1 on success or >= 0 if C_NN is not positive definite.
 * work: s*s doubles. */
static int or_vecchia_row(const or_theta *th, const double *X, const int32_t *Sidx, int s,
                          const double *uS, int m, double *work, double *a, double *Di) {
  double *C = work;
  for (int p = 0; p < s; ++p)
    for (int q = 0; q < s; ++q) {
      double c = or_cov(th, X + (size_t)Sidx[p] * th->d, X + (size_t)Sidx[q] * th->d);
      double uu = 0.0;
      for (int k = 0; k < m; ++k) uu += uS[(size_t)p * m + k] * uS[(size_t)q * m + k];
      c -= uu;
      if (p == q) c += th->nugget; /* sigma^2 by index identity (reading c2) */
      C[(size_t)p * s + q] = c;
    }
  int qn = s - 1;
  /* c = C_{N,i}; solve C_NN a = c via Cholesky of the leading block */
  for (int p = 0; p < qn; ++p) a[p] = C[(size_t)p * s + qn];
  if (qn > 0) {
    int bad = or_chol(C, qn, s);
    if (bad >= 0) return bad;
    or_fwd(C, qn, s, a);
    or_bwd(C, qn, s, a);
  }
  double D = C[(size_t)qn * s + qn];
  for (int p = 0; p < qn; ++p) D -= a[p] * C[(size_t)qn * s + p]; /* C is symmetric: C_{i,N} row */
  *Di = D;
  return -1;
}

static int or_count_nbrs(const int32_t *row, int mv) {
  int q = 0;
  while (q < mv && row[q] >= 0) ++q;
  return q;
}

/* Validate neighbour sets: N(i) subset of {0..i-1}, no duplicates, -1 only as a trailing pad.
 * Returns -1 if valid, else the offending row. */
int64_t oracle_check_neighbors(int64_t n, int mv, const int32_t *nbr) {
  for (int64_t i = 0; i < n; ++i) {
    const int32_t *row = nbr + i * mv;
    int q = or_count_nbrs(row, mv);
    for (int p = q; p < mv; ++p)
      if (row[p] != -1) return i;
    for (int p = 0; p < q; ++p) {
      if (row[p] < 0 || row[p] >= i) return i;
      for (int t = 0; t < p; ++t)
        if (row[t] == row[p]) return i;
    }
  }
  return -1;
}

/* ---- exported: the whole factor + NLL (oracle T1) ----
 * X: n x d (Vecchia order), Z: m x d, nbr: n x mv (-1 padded), y: n.
 * U_out (n x m), B_out (n x mv, stores -A_i in N(i) order, 0 pad), D_out (n): optional.
 * terms[0..3] = nll, logdet_D, logdet_M, quad.  *bad_row: failing row (-1 = K_m or M).
 * Implements SURVEY 8(c) "Oracle T1" steps 1-7 in order. */
int oracle_factor_nll(int64_t n, int m, int mv, const double *X, const double *Z, const int32_t *nbr,
                      const double *y, const or_theta *th, double *U_out, double *B_out, double *D_out,
                      double *terms, int64_t *bad_row) {
  *bad_row = -1;
  if (n < 1 || m < 0 || mv < 0 || th->d < 1) return OR_INVALID;
  int status = OR_OK;
  double *Lm = NULL, *U = U_out;
  if (m > 0) {
    Lm = (double *)malloc(sizeof(double) * (size_t)m * m);
    if (!Lm) return OR_NOMEM;
    if (or_build_Lm(th, Z, m, Lm) != OR_OK) { free(Lm); return OR_NOT_PD; }
    if (!U) {
      U = (double *)malloc(sizeof(double) * (size_t)n * m);
      if (!U) { free(Lm); return OR_NOMEM; }
    }
    /* step 2 */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) or_u_row(th, Z, m, Lm, X + i * th->d, U + i * (size_t)m);
  }
  int nthreads = 1;
#ifdef _OPENMP
  nthreads = omp_get_max_threads();
#endif
  size_t mm = (size_t)m * m;
  double *Mt = (double *)calloc((size_t)nthreads * (mm + m + 2), sizeof(double));
  int64_t *bad = (int64_t *)malloc(sizeof(int64_t) * nthreads);
  if (!Mt || !bad) { free(Lm); if (U != U_out) free(U); free(Mt); free(bad); return OR_NOMEM; }
  for (int t = 0; t < nthreads; ++t) bad[t] = -1;

#pragma omp parallel num_threads(nthreads)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    int s_max = mv + 1;
    int32_t *S = (int32_t *)malloc(sizeof(int32_t) * s_max);
    double *uS = (double *)malloc(sizeof(double) * (size_t)s_max * (m > 0 ? m : 1));
    double *work = (double *)malloc(sizeof(double) * (size_t)s_max * s_max);
    double *a = (double *)malloc(sizeof(double) * (mv > 0 ? mv : 1));
    double *w = (double *)malloc(sizeof(double) * (m > 0 ? m : 1));
    double *Mp = Mt + (size_t)tid * (mm + m + 2);
    double *vp = Mp + mm;
    double *qp = vp + m;     /* [0] = sum r^2/D, [1] = sum log D */
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      if (bad[tid] >= 0) continue;
      const int32_t *row = nbr + i * mv;
      int q = or_count_nbrs(row, mv);
      int s = q + 1;
      for (int p = 0; p < q; ++p) S[p] = row[p];
      S[q] = (int32_t)i;
      for (int p = 0; p < s; ++p)
        for (int k = 0; k < m; ++k) uS[(size_t)p * m + k] = U[(size_t)S[p] * m + k];
      double Di;
      /* step 3 */
      int b = or_vecchia_row(th, X, S, s, uS, m, work, a, &Di);
      if (b >= 0 || !(Di > 0.0)) { bad[tid] = i; continue; }
      if (B_out) {
        for (int p = 0; p < mv; ++p) B_out[i * mv + p] = p < q ? -a[p] : 0.0;
      }
      if (D_out) D_out[i] = Di;
      /* step 4 */
      double r = y[i];
      for (int p = 0; p < q; ++p) r -= a[p] * y[S[p]];
      for (int k = 0; k < m; ++k) {
        double t = uS[(size_t)q * m + k];
        for (int p = 0; p < q; ++p) t -= a[p] * uS[(size_t)p * m + k];
        w[k] = t;
      }
      /* step 5 */
      for (int k = 0; k < m; ++k)
        for (int l = 0; l <= k; ++l) Mp[(size_t)k * m + l] += w[k] * w[l] / Di;
      for (int k = 0; k < m; ++k) vp[k] += w[k] * r / Di;
      qp[0] += r * r / Di;
      qp[1] += log(Di);
    }
    free(S); free(uS); free(work); free(a); free(w);
  }
  for (int t = 0; t < nthreads; ++t)
    if (bad[t] >= 0 && (*bad_row < 0 || bad[t] < *bad_row)) *bad_row = bad[t];
  if (*bad_row >= 0) status = OR_NOT_PD;

  if (status == OR_OK) {
    /* merge in thread-index order */
    double *M = (double *)calloc(mm + m + 2, sizeof(double));
    for (int t = 0; t < nthreads; ++t) {
      const double *src = Mt + (size_t)t * (mm + m + 2);
      for (size_t k = 0; k < mm + m + 2; ++k) M[k] += src[k];
    }
    double *v = M + mm, qsum = M[mm + m], logdetD = M[mm + m + 1];
    /* step 6 */
    double logdetM = 0.0, quad = qsum;
    if (m > 0) {
      for (int k = 0; k < m; ++k) {
        M[(size_t)k * m + k] += 1.0;
        for (int l = k + 1; l < m; ++l) M[(size_t)k * m + l] = M[(size_t)l * m + k];
      }
      if (or_chol(M, m, m) >= 0) {
        status = OR_NOT_PD;
      } else {
        for (int k = 0; k < m; ++k) logdetM += 2.0 * log(M[(size_t)k * m + k]);
        or_fwd(M, m, m, v);
        for (int k = 0; k < m; ++k) quad -= v[k] * v[k];
      }
    }
    /* step 7 */
    terms[0] = 0.5 * (double)n * log(2.0 * M_PI) + 0.5 * (logdetD + logdetM) + 0.5 * quad;
    terms[1] = logdetD;
    terms[2] = logdetM;
    terms[3] = quad;
    free(M);
  }
  free(Mt); free(bad); free(Lm);
  if (U != U_out) free(U);
  return status;
}

/* ---- exported: sampled rows (for parity at sizes where the full oracle is too slow) ----
 * For each requested row i: u_i (if U_rows != NULL, nrows x m), B row (nrows x mv), D_i.
 * Every needed u_j is recomputed from scratch from L_m (no shared state with anything). */
int oracle_rows(int64_t n, int m, int mv, const double *X, const double *Z, const int32_t *nbr,
                const or_theta *th, int64_t nrows, const int64_t *rows, double *U_rows, double *B_rows,
                double *D_rows, int64_t *bad_row) {
  *bad_row = -1;
  double *Lm = NULL;
  if (m > 0) {
    Lm = (double *)malloc(sizeof(double) * (size_t)m * m);
    if (!Lm) return OR_NOMEM;
    if (or_build_Lm(th, Z, m, Lm) != OR_OK) { free(Lm); return OR_NOT_PD; }
  }
  int status = OR_OK;
#pragma omp parallel
  {
    int s_max = mv + 1;
    int32_t *S = (int32_t *)malloc(sizeof(int32_t) * s_max);
    double *uS = (double *)malloc(sizeof(double) * (size_t)s_max * (m > 0 ? m : 1));
    double *work = (double *)malloc(sizeof(double) * (size_t)s_max * s_max);
    double *a = (double *)malloc(sizeof(double) * (mv > 0 ? mv : 1));
#pragma omp for schedule(dynamic, 4)
    for (int64_t t = 0; t < nrows; ++t) {
      int64_t i = rows[t];
      if (i < 0 || i >= n) { status = OR_INVALID; continue; }
      const int32_t *row = nbr + i * mv;
      int q = or_count_nbrs(row, mv);
      int s = q + 1;
      for (int p = 0; p < q; ++p) S[p] = row[p];
      S[q] = (int32_t)i;
      for (int p = 0; p < s && m > 0; ++p) or_u_row(th, Z, m, Lm, X + (size_t)S[p] * th->d, uS + (size_t)p * m);
      if (U_rows)
        for (int k = 0; k < m; ++k) U_rows[t * m + k] = uS[(size_t)q * m + k];
      double Di;
      int b = or_vecchia_row(th, X, S, s, uS, m, work, a, &Di);
      if (b >= 0 || !(Di > 0.0)) {
#pragma omp critical
        { if (*bad_row < 0 || i < *bad_row) *bad_row = i; status = OR_NOT_PD; }
        continue;
      }
      for (int p = 0; p < mv; ++p) B_rows[t * mv + p] = p < q ? -a[p] : 0.0;
      D_rows[t] = Di;
    }
    free(S); free(uS); free(work); free(a);
  }
  free(Lm);
  return status;
}

/* ---- exported: partial sums over an arbitrary subset of rows (sharding pins) ----
 * Given the full factor inputs, accumulate over rows[0..nrows): G (m x m lower, += w w^T/D),
 * v (m), and sums[0] += r^2/D, sums[1] += log D.  Serial, in the given row order. */
int oracle_partial(int64_t n, int m, int mv, const double *X, const double *Z, const int32_t *nbr,
                   const double *y, const or_theta *th, int64_t nrows, const int64_t *rows, double *G,
                   double *v, double *sums, int64_t *bad_row) {
  *bad_row = -1;
  double *Lm = NULL;
  if (m > 0) {
    Lm = (double *)malloc(sizeof(double) * (size_t)m * m);
    if (or_build_Lm(th, Z, m, Lm) != OR_OK) { free(Lm); return OR_NOT_PD; }
  }
  int s_max = mv + 1;
  int32_t *S = (int32_t *)malloc(sizeof(int32_t) * s_max);
  double *uS = (double *)malloc(sizeof(double) * (size_t)s_max * (m > 0 ? m : 1));
  double *work = (double *)malloc(sizeof(double) * (size_t)s_max * s_max);
  double *a = (double *)malloc(sizeof(double) * (mv > 0 ? mv : 1));
  double *w = (double *)malloc(sizeof(double) * (m > 0 ? m : 1));
  int status = OR_OK;
  for (int64_t t = 0; t < nrows; ++t) {
    int64_t i = rows[t];
    const int32_t *row = nbr + i * mv;
    int q = or_count_nbrs(row, mv);
    int s = q + 1;
    for (int p = 0; p < q; ++p) S[p] = row[p];
    S[q] = (int32_t)i;
    for (int p = 0; p < s && m > 0; ++p) or_u_row(th, Z, m, Lm, X + (size_t)S[p] * th->d, uS + (size_t)p * m);
    double Di;
    int b = or_vecchia_row(th, X, S, s, uS, m, work, a, &Di);
    if (b >= 0 || !(Di > 0.0)) { *bad_row = i; status = OR_NOT_PD; break; }
    double r = y[i];
    for (int p = 0; p < q; ++p) r -= a[p] * y[S[p]];
    for (int k = 0; k < m; ++k) {
      double tt = uS[(size_t)q * m + k];
      for (int p = 0; p < q; ++p) tt -= a[p] * uS[(size_t)p * m + k];
      w[k] = tt;
    }
    for (int k = 0; k < m; ++k)
      for (int l = 0; l <= k; ++l) G[(size_t)k * m + l] += w[k] * w[l] / Di;
    for (int k = 0; k < m; ++k) v[k] += w[k] * r / Di;
    sums[0] += r * r / Di;
    sums[1] += log(Di);
  }
  free(S); free(uS); free(work); free(a); free(w); free(Lm);
  return status;
}

/* Steps 6-7 from merged partials (G lower m x m, v, sums = {sum r^2/D, sum log D}). */
int oracle_finish(int64_t n, int m, const double *G, const double *v, const double *sums, double *terms) {
  double *M = (double *)malloc(sizeof(double) * ((size_t)m * m + m + 1));
  double *z = M + (size_t)m * m;
  for (int k = 0; k < m; ++k) {
    z[k] = v[k];
    for (int l = 0; l < m; ++l) M[(size_t)k * m + l] = (l <= k ? G[(size_t)k * m + l] : G[(size_t)l * m + k]) + (k == l ? 1.0 : 0.0);
  }
  double logdetM = 0.0, quad = sums[0];
  if (m > 0) {
    if (or_chol(M, m, m) >= 0) { free(M); return OR_NOT_PD; }
    for (int k = 0; k < m; ++k) logdetM += 2.0 * log(M[(size_t)k * m + k]);
    or_fwd(M, m, m, z);
    for (int k = 0; k < m; ++k) quad -= z[k] * z[k];
  }
  terms[0] = 0.5 * (double)n * log(2.0 * M_PI) + 0.5 * (sums[1] + logdetM) + 0.5 * quad;
  terms[1] = sums[1];
  terms[2] = logdetM;
  terms[3] = quad;
  free(M);
  return OR_OK;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* =====================================================================================
 * Gradient of the VIF Gaussian NLL with respect to theta = (sigma_1^2, lambda_1..lambda_d,
 * sigma^2)  (P:126-133 and Appendix A).
 *
 * The paper's gradient is 1/2 tr(Sigma_dagger^{-1} dSigma_dagger) - 1/2 y^T Sigma_dagger^{-1}
 * dSigma_dagger Sigma_dagger^{-1} y with dSigma_dagger = dSigma_s + dSigma_l, dB and dD from
 * Appendix A.  It is evaluated here without n x n matrices by differentiating the three terms
 * of the Woodbury/Sylvester form of the NLL that the factor above computes:
 *   NLL = n/2 log 2pi + 1/2 sum log D_i + 1/2 logdet M_w + 1/2 quad,
 *   M_w = I + sum w_i w_i^T / D_i,  v = sum w_i r_i / D_i,  quad = sum r_i^2/D_i - v^T M_w^{-1} v.
 * Per parameter p (reading g1 in DESIGN.md):
 *   dK_m, dk_i        kernel derivatives (or_dcov), jitter eps held fixed
 *   Phi = L_m^{-1} dK_m L_m^{-T},  Phi_low = tril(Phi) with halved diagonal  (d L_m = L_m Phi_low)
 *   du_i = L_m^{-1} dk_i - Phi_low u_i                                       (derivative of u_i)
 *   dC(a,b) = dk(x_a,x_b) - (du_a.u_b + u_a.du_b) + [p = nugget][a = b]     (App. A brackets)
 *   dA_i = C_NN^{-1} (dC_Ni - dC_NN A_i^T),  dD_i = dC_ii - 2 A_i.dC_Ni + A_i dC_NN A_i^T
 *                                                                            (App. A: dB = -dA)
 *   dw_i = du_i - sum_k (dA_ik u_Nk + A_ik du_Nk),  dr_i = -dA_i . y_N
 *   dM = sum (dw w^T + w dw^T)/D - w w^T dD/D^2,  dv = sum (dw r + w dr)/D - w r dD/D^2
 *   dlogdetD = sum dD/D,  dlogdetM = tr(M_w^{-1} dM),
 *   dquad = sum (2 r dr/D - r^2 dD/D^2) - 2 z.dv + z^T dM z,   z = M_w^{-1} v
 *   dNLL = 1/2 (dlogdetD + dlogdetM + dquad).
 * Pinned in tests/test_oracle_grad.py against central finite differences of oracle_factor_nll,
 * against the exact-GP gradient in the all-predecessor case, and against the paper's dense
 * formula (P:128-131 with Appendix A) assembled in numpy.
 * ===================================================================================== */

/* dk(a,b)/dtheta_p, p = 0 (sigma_1^2), 1..d (lambda_j); the nugget has no kernel derivative.
 * k = sigma_1^2 f(r): dk/dsigma_1^2 = f(r); dk/dlambda_j = sigma_1^2 (-f'(r)/r) Delta_j^2/lambda_j^3. */
static void or_dcov(const or_theta *th, const double *a, const double *b, double *dk) {
  double r2 = 0.0;
  for (int k = 0; k < th->d; ++k) {
    double t = (a[k] - b[k]) / th->lengthscale[k];
    r2 += t * t;
  }
  double r = sqrt(r2), f, h; /* h = -f'(r)/r */
  switch (th->family) {
    case 0: f = exp(-r); h = r > 0.0 ? exp(-r) / r : 0.0; break;
    case 1: f = (1.0 + sqrt(3.0) * r) * exp(-sqrt(3.0) * r); h = 3.0 * exp(-sqrt(3.0) * r); break;
    case 2:
      f = (1.0 + sqrt(5.0) * r + 5.0 * r2 / 3.0) * exp(-sqrt(5.0) * r);
      h = (5.0 / 3.0) * (1.0 + sqrt(5.0) * r) * exp(-sqrt(5.0) * r);
      break;
    default: f = exp(-r2); h = 2.0 * exp(-r2); break;
  }
  dk[0] = f;
  for (int j = 0; j < th->d; ++j) {
    double lj = th->lengthscale[j], dj = a[j] - b[j];
    dk[1 + j] = th->sigma2 * h * dj * dj / (lj * lj * lj);
  }
}

/* exported: d (kernel) matrices for the pins: out[p][i][j] = dk(A_i, B_j)/dtheta_p, p < d+1 */
int oracle_dcov_matrix(const or_theta *th, const double *A, int64_t na, const double *B, int64_t nb,
                       double *out) {
  int np = th->d + 1;
  double dk[1 + 16 + 1];
  for (int64_t i = 0; i < na; ++i)
    for (int64_t j = 0; j < nb; ++j) {
      or_dcov(th, A + i * th->d, B + j * th->d, dk);
      for (int p = 0; p < np; ++p) out[((size_t)p * na + i) * nb + j] = dk[p];
    }
  return OR_OK;
}

/* per-row quantities of the factor (same arithmetic as oracle_factor_nll steps 3-4) */
typedef struct {
  int q;
  double D, r;
} or_rowinfo;

int oracle_grad(int64_t n, int m, int mv, const double *X, const double *Z, const int32_t *nbr,
                const double *y, const or_theta *th, double *grad, double *parts, int64_t *bad_row) {
  *bad_row = -1;
  const int d = th->d, P = d + 2;
  if (n < 1 || m < 0 || mv < 0 || d < 1 || d > 16) return OR_INVALID;
  const int m1 = m > 0 ? m : 1, s_max = mv + 1;
  double *Lm = NULL, *U = NULL, *dU = NULL, *Phi = NULL, *dKm = NULL;
  double *A = (double *)malloc(sizeof(double) * (size_t)n * (mv > 0 ? mv : 1));
  double *W = (double *)malloc(sizeof(double) * (size_t)n * m1);
  or_rowinfo *info = (or_rowinfo *)malloc(sizeof(or_rowinfo) * (size_t)n);
  if (!A || !W || !info) { free(A); free(W); free(info); return OR_NOMEM; }
  int status = OR_OK;
  if (m > 0) {
    Lm = (double *)malloc(sizeof(double) * (size_t)m * m);
    U = (double *)malloc(sizeof(double) * (size_t)n * m);
    dU = (double *)malloc(sizeof(double) * (size_t)n * m);
    Phi = (double *)malloc(sizeof(double) * (size_t)m * m);
    dKm = (double *)malloc(sizeof(double) * (size_t)m * m);
    if (!Lm || !U || !dU || !Phi || !dKm) { status = OR_NOMEM; goto done; }
    if (or_build_Lm(th, Z, m, Lm) != OR_OK) { status = OR_NOT_PD; goto done; }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) or_u_row(th, Z, m, Lm, X + i * d, U + i * (size_t)m);
  }
  /* ---- pass 0: A_i, D_i, w_i, r_i (steps 3-4 of the factor) and M_w, v ---- */
  {
    int64_t badr = -1;
#pragma omp parallel
    {
      int32_t *S = (int32_t *)malloc(sizeof(int32_t) * s_max);
      double *uS = (double *)malloc(sizeof(double) * (size_t)s_max * m1);
      double *work = (double *)malloc(sizeof(double) * (size_t)s_max * s_max);
#pragma omp for schedule(static)
      for (int64_t i = 0; i < n; ++i) {
        const int32_t *row = nbr + i * mv;
        int q = or_count_nbrs(row, mv), s = q + 1;
        for (int p = 0; p < q; ++p) S[p] = row[p];
        S[q] = (int32_t)i;
        for (int p = 0; p < s; ++p)
          for (int k = 0; k < m; ++k) uS[(size_t)p * m + k] = U[(size_t)S[p] * m + k];
        double Di, *a = A + i * mv;
        int b = or_vecchia_row(th, X, S, s, uS, m, work, a, &Di);
        if (b >= 0 || !(Di > 0.0)) {
#pragma omp critical
          { if (badr < 0 || i < badr) badr = i; }
          continue;
        }
        double r = y[i];
        for (int p = 0; p < q; ++p) r -= a[p] * y[S[p]];
        for (int k = 0; k < m; ++k) {
          double t = uS[(size_t)q * m + k];
          for (int p = 0; p < q; ++p) t -= a[p] * uS[(size_t)p * m + k];
          W[i * (size_t)m + k] = t;
        }
        info[i].q = q;
        info[i].D = Di;
        info[i].r = r;
      }
      free(S); free(uS); free(work);
    }
    if (badr >= 0) { *bad_row = badr; status = OR_NOT_PD; goto done; }
  }
  /* M_w, v (serial, row order), Minv = M_w^{-1}, z = M_w^{-1} v */
  double *M = (double *)calloc((size_t)m1 * m1 * 2 + 2 * m1, sizeof(double));
  double *Minv = M + (size_t)m1 * m1, *v = Minv + (size_t)m1 * m1, *z = v + m1;
  for (int64_t i = 0; i < n; ++i) {
    const double *w = W + i * (size_t)m;
    for (int k = 0; k < m; ++k) {
      for (int l = 0; l < m; ++l) M[(size_t)k * m + l] += w[k] * w[l] / info[i].D;
      v[k] += w[k] * info[i].r / info[i].D;
    }
  }
  if (m > 0) {
    for (int k = 0; k < m; ++k) M[(size_t)k * m + k] += 1.0;
    if (or_chol(M, m, m) >= 0) { free(M); status = OR_NOT_PD; goto done; }
    for (int c = 0; c < m; ++c) { /* column c of M^{-1}: L L^T x = e_c */
      double *e = (double *)calloc(m, sizeof(double));
      e[c] = 1.0;
      or_fwd(M, m, m, e);
      or_bwd(M, m, m, e);
      for (int k = 0; k < m; ++k) Minv[(size_t)k * m + c] = e[k];
      free(e);
    }
    for (int k = 0; k < m; ++k) z[k] = v[k];
    or_fwd(M, m, m, z);
    or_bwd(M, m, m, z);
  }
  /* ---- one pass per parameter ---- */
  for (int p = 0; p < P; ++p) {
    const int is_nugget = p == d + 1;
    if (m > 0) {
      if (is_nugget) {
        memset(dU, 0, sizeof(double) * (size_t)n * m);
      } else {
        /* dK_m and Phi = L^{-1} dK_m L^{-T} (column solves; dK_m symmetric) */
        double dk[1 + 16 + 1];
        for (int a = 0; a < m; ++a)
          for (int b = 0; b < m; ++b) {
            or_dcov(th, Z + (size_t)a * d, Z + (size_t)b * d, dk);
            dKm[(size_t)a * m + b] = dk[p];
          }
        double *col = (double *)malloc(sizeof(double) * m);
        for (int c = 0; c < m; ++c) { /* T = L^{-1} dK_m, column c; stored transposed in Phi */
          for (int k = 0; k < m; ++k) col[k] = dKm[(size_t)k * m + c];
          or_fwd(Lm, m, m, col);
          for (int k = 0; k < m; ++k) Phi[(size_t)c * m + k] = col[k]; /* Phi = T^T = dK L^{-T} */
        }
        double *T2 = (double *)malloc(sizeof(double) * (size_t)m * m);
        for (int c = 0; c < m; ++c) { /* L^{-1} (dK L^{-T}), column c */
          for (int k = 0; k < m; ++k) col[k] = Phi[(size_t)k * m + c];
          or_fwd(Lm, m, m, col);
          for (int k = 0; k < m; ++k) T2[(size_t)k * m + c] = col[k];
        }
        for (int a = 0; a < m; ++a)
          for (int b = 0; b < m; ++b)
            Phi[(size_t)a * m + b] = b < a ? T2[(size_t)a * m + b] : (b == a ? 0.5 * T2[(size_t)a * m + a] : 0.0);
        free(T2);
        free(col);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
          double dkk[1 + 16 + 1], *du = dU + i * (size_t)m;
          for (int a = 0; a < m; ++a) {
            or_dcov(th, Z + (size_t)a * d, X + i * d, dkk);
            du[a] = dkk[p];
          }
          or_fwd(Lm, m, m, du);
          const double *u = U + i * (size_t)m;
          for (int a = 0; a < m; ++a) {
            double t = 0.0;
            for (int b = 0; b <= a; ++b) t += Phi[(size_t)a * m + b] * u[b];
            du[a] -= t;
          }
        }
      }
    }
    /* row pass: dD, dw, dr -> dM, dv, scalars; per-thread partials merged in thread order */
    int nthreads = 1;
#ifdef _OPENMP
    nthreads = omp_get_max_threads();
#endif
    const size_t stride = (size_t)m1 * m1 + m1 + 2;
    double *part = (double *)calloc((size_t)nthreads * stride, sizeof(double));
#pragma omp parallel num_threads(nthreads)
    {
      int tid = 0;
#ifdef _OPENMP
      tid = omp_get_thread_num();
#endif
      double *dM = part + (size_t)tid * stride, *dv = dM + (size_t)m1 * m1, *sc = dv + m1;
      int32_t *S = (int32_t *)malloc(sizeof(int32_t) * s_max);
      double *C = (double *)malloc(sizeof(double) * (size_t)s_max * s_max);
      double *dC = (double *)malloc(sizeof(double) * (size_t)s_max * s_max);
      double *da = (double *)malloc(sizeof(double) * s_max);
      double *dw = (double *)malloc(sizeof(double) * m1);
#pragma omp for schedule(static)
      for (int64_t i = 0; i < n; ++i) {
        const int q = info[i].q, s = q + 1;
        const int32_t *row = nbr + i * mv;
        for (int k = 0; k < q; ++k) S[k] = row[k];
        S[q] = (int32_t)i;
        const double *a = A + i * mv;
        const double Di = info[i].D, ri = info[i].r;
        /* C and dC on S (App. A brackets) */
        for (int u1 = 0; u1 < s; ++u1)
          for (int u2 = 0; u2 < s; ++u2) {
            const double *xa = X + (size_t)S[u1] * d, *xb = X + (size_t)S[u2] * d;
            double dk[1 + 16 + 1];
            or_dcov(th, xa, xb, dk);
            double c = or_cov(th, xa, xb), dc = is_nugget ? 0.0 : dk[p];
            for (int k = 0; k < m; ++k) {
              const double ua = U[(size_t)S[u1] * m + k], ub = U[(size_t)S[u2] * m + k];
              c -= ua * ub;
              dc -= dU[(size_t)S[u1] * m + k] * ub + ua * dU[(size_t)S[u2] * m + k];
            }
            if (u1 == u2) { c += th->nugget; if (is_nugget) dc += 1.0; }
            C[(size_t)u1 * s + u2] = c;
            dC[(size_t)u1 * s + u2] = dc;
          }
        /* dA = C_NN^{-1} (dC_Ni - dC_NN a),  dD */
        double dD = dC[(size_t)q * s + q];
        for (int k = 0; k < q; ++k) {
          double t = dC[(size_t)k * s + q];
          for (int l = 0; l < q; ++l) t -= dC[(size_t)k * s + l] * a[l];
          da[k] = t;
          dD -= 2.0 * a[k] * dC[(size_t)k * s + q];
          for (int l = 0; l < q; ++l) dD += a[k] * dC[(size_t)k * s + l] * a[l];
        }
        if (q > 0) {
          or_chol(C, q, s); /* succeeded in pass 0 */
          or_fwd(C, q, s, da);
          or_bwd(C, q, s, da);
        }
        /* dw, dr */
        double dr = 0.0;
        for (int k = 0; k < q; ++k) dr -= da[k] * y[S[k]];
        for (int c = 0; c < m; ++c) {
          double t = dU[(size_t)i * m + c];
          for (int k = 0; k < q; ++k) t -= da[k] * U[(size_t)S[k] * m + c] + a[k] * dU[(size_t)S[k] * m + c];
          dw[c] = t;
        }
        const double *w = W + i * (size_t)m;
        const double iD = 1.0 / Di, iD2 = dD / (Di * Di);
        for (int k = 0; k < m; ++k) {
          for (int l = 0; l < m; ++l) dM[(size_t)k * m + l] += (dw[k] * w[l] + w[k] * dw[l]) * iD - w[k] * w[l] * iD2;
          dv[k] += (dw[k] * ri + w[k] * dr) * iD - w[k] * ri * iD2;
        }
        sc[0] += dD * iD;                               /* dlogdetD */
        sc[1] += 2.0 * ri * dr * iD - ri * ri * iD2;    /* d sum r^2/D */
      }
      free(S); free(C); free(dC); free(da); free(dw);
    }
    double *acc = (double *)calloc(stride, sizeof(double));
    for (int t = 0; t < nthreads; ++t)
      for (size_t k = 0; k < stride; ++k) acc[k] += part[(size_t)t * stride + k];
    double *dM = acc, *dv = acc + (size_t)m1 * m1, *sc = dv + m1;
    double dlogdetM = 0.0, dquad = sc[1];
    for (int k = 0; k < m; ++k) {
      for (int l = 0; l < m; ++l) {
        dlogdetM += Minv[(size_t)k * m + l] * dM[(size_t)l * m + k];
        dquad += z[k] * dM[(size_t)k * m + l] * z[l];
      }
      dquad -= 2.0 * z[k] * dv[k];
    }
    grad[p] = 0.5 * (sc[0] + dlogdetM + dquad);
    if (parts) {
      parts[3 * p + 0] = sc[0];
      parts[3 * p + 1] = dlogdetM;
      parts[3 * p + 2] = dquad;
    }
    free(acc);
    free(part);
  }
  free(M);
done:
  free(A); free(W); free(info); free(Lm); free(U); free(dU); free(Phi); free(dKm);
  return status;
}

/* =====================================================================================
 * Predictive means (Proposition 1), reading p1: every prediction point conditions on
 * m_v training points only (B_p = I, B_po row p = -A_p), so with the training factor's
 * z = M_w^{-1} v (step 6):
 *   mu_p = u_p . z + A_p (y_N(p) - U_N(p) z),  u_p = L_m^{-1} k(Z, x_p),
 *   A_p = C_{p,N} C_{N,N}^{-1},  D_p = C_pp - A_p C_{N,p},
 *   C(a,b) = k - u_a.u_b + sigma^2 [a = b] on training pairs, C(p,a) = k(x_p,x_a) - u_p.u_a,
 *   C_pp = sigma_1^2 + sigma^2 - u_p.u_p  (the response y_p),
 *   var_p = D_p + e_p^T M_w^{-1} e_p,  e_p = u_p - sum_k A_pk u_N(p)_k   (App. C.1).
 * Derivation from Prop. 1 / App. C.1 with whitening in DESIGN.md section 11; pinned in tests/test_oracle_pred.py
 * against the exact GP (all training points as neighbours) and the paper's dense formula P:143-144.
 * ===================================================================================== */
int oracle_predict(int64_t n, int m, int mv, const double *X, const double *Z, const int32_t *nbr, const double *y,
                   const or_theta *th, int64_t np, const double *Xp, const int32_t *nbrp, double *mu, double *var,
                   double *Dp, double *Bp, int64_t *bad_row) {
  *bad_row = -1;
  const int d = th->d, m1 = m > 0 ? m : 1, s_max = mv + 1;
  double *Lm = NULL, *U = NULL;
  double *A = (double *)malloc(sizeof(double) * (size_t)n * (mv > 0 ? mv : 1));
  double *W = (double *)malloc(sizeof(double) * (size_t)n * m1);
  or_rowinfo *info = (or_rowinfo *)malloc(sizeof(or_rowinfo) * (size_t)n);
  double *M = (double *)calloc((size_t)m1 * m1 + 2 * m1, sizeof(double));
  double *v = M + (size_t)m1 * m1, *z = v + m1;
  int status = OR_OK;
  if (!A || !W || !info || !M) { status = OR_NOMEM; goto done; }
  if (m > 0) {
    Lm = (double *)malloc(sizeof(double) * (size_t)m * m);
    U = (double *)malloc(sizeof(double) * (size_t)n * m);
    if (!Lm || !U) { status = OR_NOMEM; goto done; }
    if (or_build_Lm(th, Z, m, Lm) != OR_OK) { status = OR_NOT_PD; goto done; }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) or_u_row(th, Z, m, Lm, X + i * d, U + i * (size_t)m);
  }
  /* training factor: A_i, D_i, w_i, r_i -> M_w, v, z (steps 3-6) */
  {
    int64_t badr = -1;
#pragma omp parallel
    {
      int32_t *S = (int32_t *)malloc(sizeof(int32_t) * s_max);
      double *uS = (double *)malloc(sizeof(double) * (size_t)s_max * m1);
      double *work = (double *)malloc(sizeof(double) * (size_t)s_max * s_max);
#pragma omp for schedule(static)
      for (int64_t i = 0; i < n; ++i) {
        const int32_t *row = nbr + i * mv;
        int q = or_count_nbrs(row, mv), s = q + 1;
        for (int k = 0; k < q; ++k) S[k] = row[k];
        S[q] = (int32_t)i;
        for (int k = 0; k < s; ++k)
          for (int c = 0; c < m; ++c) uS[(size_t)k * m + c] = U[(size_t)S[k] * m + c];
        double Di, *a = A + i * mv;
        int b = or_vecchia_row(th, X, S, s, uS, m, work, a, &Di);
        if (b >= 0 || !(Di > 0.0)) {
#pragma omp critical
          { if (badr < 0 || i < badr) badr = i; }
          continue;
        }
        double r = y[i];
        for (int k = 0; k < q; ++k) r -= a[k] * y[S[k]];
        for (int c = 0; c < m; ++c) {
          double t = uS[(size_t)q * m + c];
          for (int k = 0; k < q; ++k) t -= a[k] * uS[(size_t)k * m + c];
          W[i * (size_t)m + c] = t;
        }
        info[i].q = q; info[i].D = Di; info[i].r = r;
      }
      free(S); free(uS); free(work);
    }
    if (badr >= 0) { *bad_row = badr; status = OR_NOT_PD; goto done; }
  }
  for (int64_t i = 0; i < n; ++i) {
    const double *w = W + i * (size_t)m;
    for (int k = 0; k < m; ++k) {
      for (int l = 0; l < m; ++l) M[(size_t)k * m + l] += w[k] * w[l] / info[i].D;
      v[k] += w[k] * info[i].r / info[i].D;
    }
  }
  if (m > 0) {
    for (int k = 0; k < m; ++k) M[(size_t)k * m + k] += 1.0;
    if (or_chol(M, m, m) >= 0) { status = OR_NOT_PD; goto done; }
    for (int k = 0; k < m; ++k) z[k] = v[k];
    or_fwd(M, m, m, z);
    or_bwd(M, m, m, z);
  }
  /* prediction points */
  {
    int64_t badp = -1;
#pragma omp parallel
    {
      double *up = (double *)malloc(sizeof(double) * m1);
      double *C = (double *)malloc(sizeof(double) * (size_t)s_max * s_max);
      double *c = (double *)malloc(sizeof(double) * s_max);
#pragma omp for schedule(static)
      for (int64_t t = 0; t < np; ++t) {
        const double *xp = Xp + t * d;
        if (m > 0) or_u_row(th, Z, m, Lm, xp, up);
        const int32_t *row = nbrp + t * mv;
        const int q = or_count_nbrs(row, mv);
        for (int a = 0; a < q; ++a) {
          const double *xa = X + (size_t)row[a] * d;
          for (int b = 0; b < q; ++b) {
            double cc = or_cov(th, xa, X + (size_t)row[b] * d);
            for (int k = 0; k < m; ++k) cc -= U[(size_t)row[a] * m + k] * U[(size_t)row[b] * m + k];
            if (a == b) cc += th->nugget;
            C[(size_t)a * q + b] = cc;
          }
          double cp = or_cov(th, xa, xp);
          for (int k = 0; k < m; ++k) cp -= U[(size_t)row[a] * m + k] * up[k];
          c[a] = cp;
        }
        double Cpp = th->sigma2 + th->nugget;
        for (int k = 0; k < m; ++k) Cpp -= up[k] * up[k];
        /* A_p = C_NN^{-1} c */
        double *ap = c + 0;
        double *cN = (double *)malloc(sizeof(double) * (q > 0 ? q : 1));
        for (int a = 0; a < q; ++a) cN[a] = c[a];
        if (q > 0) {
          if (or_chol(C, q, q) >= 0) {
#pragma omp critical
            { if (badp < 0 || t < badp) badp = t; }
            free(cN);
            continue;
          }
          or_fwd(C, q, q, ap);
          or_bwd(C, q, q, ap);
        }
        double D = Cpp, mean = 0.0;
        for (int a = 0; a < q; ++a) D -= ap[a] * cN[a];
        for (int k = 0; k < m; ++k) mean += up[k] * z[k];
        for (int a = 0; a < q; ++a) {
          double uz = 0.0;
          for (int k = 0; k < m; ++k) uz += U[(size_t)row[a] * m + k] * z[k];
          mean += ap[a] * (y[row[a]] - uz);
        }
        mu[t] = mean;
        if (var) {
          /* e_p M_w^{-1} e_p = |L_M^{-1} e_p|^2 (M holds L_M after step 6) */
          double *e = (double *)malloc(sizeof(double) * m1), vv = D;
          for (int k = 0; k < m; ++k) {
            double t2 = up[k];
            for (int a = 0; a < q; ++a) t2 -= ap[a] * U[(size_t)row[a] * m + k];
            e[k] = t2;
          }
          if (m > 0) or_fwd(M, m, m, e);
          for (int k = 0; k < m; ++k) vv += e[k] * e[k];
          var[t] = vv;
          free(e);
        }
        if (Dp) Dp[t] = D;
        if (Bp)
          for (int a = 0; a < mv; ++a) Bp[t * mv + a] = a < q ? -ap[a] : 0.0;
        free(cN);
      }
      free(up); free(C); free(c);
    }
    if (badp >= 0) { *bad_row = badp; status = OR_NOT_PD; }
  }
done:
  free(A); free(W); free(info); free(M); free(Lm); free(U);
  return status;
}

/* =====================================================================================
 * Correlation-distance neighbour sets, exact brute force.
 *   rho_c(i,j) = k(x_i,x_j) - u_i.u_j   (residual process without the nugget)
 *   d_c(i,j) = sqrt(1 - |rho_c(i,j)| / sqrt(rho_c(i,i) rho_c(j,j)))
 * N(i) = the m_v predecessors j < i with the smallest d_c, ranked by (d_c, index) (reading c6);
 * i <= m_v: all predecessors (reading c5).  Reading c7: a candidate whose residual variance
 * rho_c(j,j) < 1e-7 sigma_1^2 gets d_c = 1; a query with such a variance ranks its predecessors by the
 * length-scale-scaled Euclidean distance.  The paper's cover tree (Alg. 3-4) returns the same sets.
 * Scores compared: |corr| descending (= d_c ascending), or -dist^2 for degenerate queries.
 * ===================================================================================== */
int oracle_dc_neighbors(int64_t n, int m, int mv, const double *X, const double *Z, const or_theta *th,
                        int32_t *nbr_out, double *score_out) {
  const int d = th->d;
  double *Lm = NULL, *U = NULL, *rd = NULL;
  int status = OR_OK;
  rd = (double *)malloc(sizeof(double) * (size_t)n);
  if (!rd) return OR_NOMEM;
  if (m > 0) {
    Lm = (double *)malloc(sizeof(double) * (size_t)m * m);
    U = (double *)malloc(sizeof(double) * (size_t)n * m);
    if (!Lm || !U) { status = OR_NOMEM; goto done; }
    if (or_build_Lm(th, Z, m, Lm) != OR_OK) { status = OR_NOT_PD; goto done; }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) or_u_row(th, Z, m, Lm, X + i * d, U + i * (size_t)m);
  }
  for (int64_t i = 0; i < n; ++i) {
    double v = th->sigma2;
    for (int k = 0; k < m; ++k) v -= U[i * (size_t)m + k] * U[i * (size_t)m + k];
    rd[i] = v;
  }
  {
    const double tau = 1e-7 * th->sigma2;
#pragma omp parallel
    {
      double *bv = (double *)malloc(sizeof(double) * (mv > 0 ? mv : 1));
      int32_t *bi = (int32_t *)malloc(sizeof(int32_t) * (mv > 0 ? mv : 1));
#pragma omp for schedule(dynamic, 64)
      for (int64_t i = 0; i < n; ++i) {
        int cnt = 0;
        const int qdeg = rd[i] < tau;
        for (int64_t j = 0; j < i; ++j) {
          double sc;
          if (qdeg) {
            double d2 = 0.0;
            for (int k = 0; k < d; ++k) {
              double t = (X[i * d + k] - X[j * d + k]) / th->lengthscale[k];
              d2 += t * t;
            }
            sc = -d2;
          } else if (rd[j] < tau) {
            sc = 0.0; /* d_c = 1 */
          } else {
            double c = or_cov(th, X + i * d, X + j * d);
            for (int k = 0; k < m; ++k) c -= U[i * (size_t)m + k] * U[j * (size_t)m + k];
            sc = fabs(c) / sqrt(rd[i] * rd[j]);
          }
          /* insert (sc desc, j asc); j increases, so equal scores keep earlier indices first */
          if (cnt < mv || sc > bv[cnt - 1]) {
            int pos = cnt < mv ? cnt : mv - 1;
            while (pos > 0 && sc > bv[pos - 1]) {
              bv[pos] = bv[pos - 1];
              bi[pos] = bi[pos - 1];
              --pos;
            }
            bv[pos] = sc;
            bi[pos] = (int32_t)j;
            if (cnt < mv) ++cnt;
          }
        }
        for (int k = 0; k < mv; ++k) {
          nbr_out[i * mv + k] = k < cnt ? bi[k] : -1;
          if (score_out) score_out[i * mv + k] = k < cnt ? bv[k] : -INFINITY;
        }
      }
      free(bv);
      free(bi);
    }
  }
done:
  free(Lm); free(U); free(rd);
  return status;
}

/* score of given (i, j) pairs under the same rules (for validity checks of other implementations) */
int oracle_dc_scores(int64_t n, int m, const double *X, const double *Z, const or_theta *th, int64_t npairs,
                     const int64_t *qi, const int64_t *cj, double *score) {
  const int d = th->d;
  double *Lm = NULL;
  if (m > 0) {
    Lm = (double *)malloc(sizeof(double) * (size_t)m * m);
    if (or_build_Lm(th, Z, m, Lm) != OR_OK) { free(Lm); return OR_NOT_PD; }
  }
  const double tau = 1e-7 * th->sigma2;
#pragma omp parallel
  {
    double *ui = (double *)malloc(sizeof(double) * (m > 0 ? m : 1));
    double *uj = (double *)malloc(sizeof(double) * (m > 0 ? m : 1));
#pragma omp for schedule(static)
    for (int64_t t = 0; t < npairs; ++t) {
      const int64_t i = qi[t], j = cj[t];
      if (m > 0) {
        or_u_row(th, Z, m, Lm, X + i * d, ui);
        or_u_row(th, Z, m, Lm, X + j * d, uj);
      }
      double ri = th->sigma2, rj = th->sigma2, c = or_cov(th, X + i * d, X + j * d);
      for (int k = 0; k < m; ++k) { ri -= ui[k] * ui[k]; rj -= uj[k] * uj[k]; c -= ui[k] * uj[k]; }
      if (ri < tau) {
        double d2 = 0.0;
        for (int k = 0; k < d; ++k) {
          double q = (X[i * d + k] - X[j * d + k]) / th->lengthscale[k];
          d2 += q * q;
        }
        score[t] = -d2;
      } else if (rj < tau) {
        score[t] = 0.0;
      } else {
        score[t] = fabs(c) / sqrt(ri * rj);
      }
    }
    free(ui); free(uj);
  }
  free(Lm);
  return OR_OK;
}
