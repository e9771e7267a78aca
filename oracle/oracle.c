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
