// k_laplace.cu -- kernels of the VIF-Laplace iterative path (Sect. 3).
//
// Vectors are row-major n x ncol (ncol = 1 for the Newton solves, ell for the SLQ probes), rows by
// point index (the Vecchia order).  The latent factor B (unit lower triangular, B[i, N(i)] = -A_i),
// D and the whitened U come from the VIF factor with the error variance removed.
//
//   la_trsv_fwd   x = B^{-1} (s o v)        sync-free forward substitution: a warp takes the next
//                                           row from a ticket counter, waits (acquire) on the
//                                           ready flags of its m_v neighbours, gathers them, and
//                                           publishes its row with a release store of the flag;
//   la_trsv_bwd   y = B^{-T} u              the same on the transposed structure (children lists),
//                                           rows taken in decreasing order;
//   la_tsgemm     C = U^T diag(rs) V        tall-skinny split-row contraction (m x ncol), two-stage
//                                           deterministic reduction;
//   la_coldot ... per-column dot products (two-stage, fixed order), CG vector updates, FITC rows,
//                 the Newton step and the SLQ quadrature e_1^T log(T) e_1 (implicit QL on T).
//
// Tickets make the schedule deadlock-free: a warp only waits on rows with smaller tickets, which
// were claimed by warps that are already running.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace vif {

namespace {

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int LA_THREADS = 256;
constexpr int LA_WARPS = LA_THREADS / 32;

// ------------------------------------------------------------------ transposed structure of B
__global__ void la_count_kernel(const int32_t* __restrict__ nbr, int64_t n, int mv, int* __restrict__ cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * mv; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = nbr[e];
    if (j >= 0) atomicAdd(cnt + j, 1);
  }
}

// exclusive scan of cnt (n) into ptr (n + 1); one block of 1024 threads, contiguous chunks
__global__ void __launch_bounds__(1024) la_scan_kernel(const int* __restrict__ cnt, int64_t n, int* __restrict__ ptr) {
  __shared__ int part[1024];
  const int t = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t b0 = t * per, b1 = b0 + per < n ? b0 + per : n;
  int s = 0;
  for (int64_t i = b0; i < b1; ++i) s += cnt[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int acc = 0;
    for (int k = 0; k < 1024; ++k) {
      const int v = part[k];
      part[k] = acc;
      acc += v;
    }
    ptr[n] = acc;
  }
  __syncthreads();
  int acc = part[t];
  for (int64_t i = b0; i < b1; ++i) {
    ptr[i] = acc;
    acc += cnt[i];
  }
}

__global__ void la_fill_kernel(const int32_t* __restrict__ nbr, int64_t n, int mv, const int* __restrict__ ptr,
                               int* __restrict__ cursor, int* __restrict__ tpos) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * mv; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = nbr[e];
    if (j >= 0) tpos[ptr[j] + atomicAdd(cursor + j, 1)] = (int)e;
  }
}

// sort each children list by entry index (= by child row): a deterministic gather order
__global__ void la_sort_kernel(int64_t n, const int* __restrict__ ptr, int* __restrict__ tpos) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int a = ptr[j], b = ptr[j + 1];
    for (int k = a + 1; k < b; ++k) {
      const int v = tpos[k];
      int q = k - 1;
      while (q >= a && tpos[q] > v) {
        tpos[q + 1] = tpos[q];
        --q;
      }
      tpos[q + 1] = v;
    }
  }
}

// ------------------------------------------------------------------ sync-free triangular solves
// x_i = s_i v_i - sum_p B[i,p] x_{N(i)_p}   (B x = s o v, B unit lower triangular)
// optional out2_i = x_i + w2_i * v2_i (the W^{-1} p term of (W^{-1} + Sigma_dagger) p is added there)
__global__ void __launch_bounds__(LA_THREADS) la_trsv_fwd_kernel(
    const int32_t* __restrict__ nbr, const double* __restrict__ Bc, int mv, int64_t n, int ncol,
    const double* __restrict__ v, const double* __restrict__ s, double* x, const double* __restrict__ v2,
    const double* __restrict__ w2, double* __restrict__ out2, int* flags, int epoch,
    unsigned long long* ticket) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if ((int64_t)t >= n) break;
    const int64_t i = (int64_t)t;
    const int32_t* nb = nbr + i * mv;
    const double* bi = Bc + i * mv;
    for (int p = lane; p < mv; p += 32) {
      const int j = nb[p];
      if (j >= 0)
        while (ld_acquire(flags + j) != epoch) {
        }
    }
    __syncwarp();
    const double si = s ? s[i] : 1.0;
    if (ncol == 1) {
      double acc = 0.0;
      for (int p = lane; p < mv; p += 32) {
        const int j = nb[p];
        if (j >= 0) acc = fma(bi[p], __ldcg(x + j), acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        const double xi = si * v[i] - acc;
        __stcg(x + i, xi);
        if (out2) out2[i] = xi + w2[i] * v2[i];
      }
    } else {
      for (int c = lane; c < ncol; c += 32) {
        double acc = 0.0;
        for (int p = 0; p < mv; ++p) {
          const int j = nb[p];
          if (j >= 0) acc = fma(bi[p], __ldcg(x + (int64_t)j * ncol + c), acc);
        }
        const double xi = si * v[i * ncol + c] - acc;
        __stcg(x + i * ncol + c, xi);
        if (out2) out2[i * ncol + c] = xi + w2[i] * v2[i * ncol + c];
      }
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(flags + i, epoch);
  }
}

// y_j = u_j - sum_{(i,p): N(i)_p = j} B[i,p] y_i   (B^T y = u), rows in decreasing order
__global__ void __launch_bounds__(LA_THREADS) la_trsv_bwd_kernel(
    const int* __restrict__ tptr, const int* __restrict__ tpos, const double* __restrict__ Bc, int mv, int64_t n,
    int ncol, const double* __restrict__ u, double* y, int* flags, int epoch, unsigned long long* ticket) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if ((int64_t)t >= n) break;
    const int64_t j = n - 1 - (int64_t)t;
    const int a = tptr[j], b = tptr[j + 1];
    for (int k = a + lane; k < b; k += 32) {
      const int i = tpos[k] / mv;
      while (ld_acquire(flags + i) != epoch) {
      }
    }
    __syncwarp();
    if (ncol == 1) {
      double acc = 0.0;
      for (int k = a + lane; k < b; k += 32) {
        const int e = tpos[k];
        acc = fma(Bc[e], __ldcg(y + e / mv), acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) __stcg(y + j, u[j] - acc);
    } else {
      for (int c = lane; c < ncol; c += 32) {
        double acc = 0.0;
        for (int k = a; k < b; ++k) {
          const int e = tpos[k];
          acc = fma(Bc[e], __ldcg(y + (int64_t)(e / mv) * ncol + c), acc);
        }
        __stcg(y + j * ncol + c, u[j * ncol + c] - acc);
      }
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(flags + j, epoch);
  }
}

// ------------------------------------------------------------------ C = U^T diag(rs) V (split rows)
// grid (nsplit, ceil(mk / 64)); thread (kk = t % 64, g = t / 64): k = k0 + kk, rows r = r0 + g + 4 q;
// part[split][c][k] (ncol x mk per split)
constexpr int TS_K = 64, TS_R = 32;
template <int NC>
__global__ void __launch_bounds__(256) la_tsgemm_kernel(const double* __restrict__ U, int64_t ldu, int mk, int64_t n,
                                                        const double* __restrict__ V, int ncol,
                                                        const int64_t* __restrict__ vrow,
                                                        const double* __restrict__ rs, int64_t rows_per,
                                                        double* __restrict__ part) {
  __shared__ double vs[TS_R][NC + 1];
  constexpr int CH = NC > 8 ? 8 : NC;  // columns per reduction round
  __shared__ double red[4][TS_K][CH + 1];
  const int t = threadIdx.x, kk = t & (TS_K - 1), g = t >> 6;
  const int k = blockIdx.y * TS_K + kk;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < n ? r0 + rows_per : n;
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  for (int64_t rb = r0; rb < r1; rb += TS_R) {
    __syncthreads();
    for (int e = t; e < TS_R * NC; e += 256) {
      const int rr = e / NC, c = e % NC;
      const int64_t r = rb + rr;
      double val = 0.0;
      if (r < r1 && c < ncol) {
        const int64_t src = vrow ? vrow[r] : r;
        val = V[src * ncol + c];
        if (rs) val *= rs[src];
      }
      vs[rr][c] = val;
    }
    __syncthreads();
    if (k < mk) {
      for (int rr = g; rr < TS_R && rb + rr < r1; rr += 4) {
        const double u = U[(rb + rr) * ldu + k];
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] = fma(u, vs[rr][c], acc[c]);
      }
    }
  }
  // reduce over the 4 row groups, CH columns at a time
#pragma unroll
  for (int c0 = 0; c0 < NC; c0 += CH) {
    __syncthreads();
#pragma unroll
    for (int c = 0; c < CH; ++c) red[g][kk][c] = acc[c0 + c];
    __syncthreads();
    for (int e = t; e < TS_K * CH; e += 256) {
      const int k2 = e % TS_K, c = e / TS_K;
      const int kg = blockIdx.y * TS_K + k2;
      if (kg < mk && c0 + c < ncol) {
        const double sum = red[0][k2][c] + red[1][k2][c] + red[2][k2][c] + red[3][k2][c];
        part[((size_t)blockIdx.x * ncol + c0 + c) * mk + kg] = sum;
      }
    }
  }
}

// Ct[c][k] = sum_s part[s][c][k] (+ Ct when accum)
__global__ void la_tsreduce_kernel(const double* __restrict__ part, int nsplit, int ncol, int mk, double* __restrict__ Ct,
                                   double alpha) {
  const int64_t tot = (int64_t)ncol * mk;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nsplit; ++q) s += part[(size_t)q * tot + e];
    Ct[e] = alpha * s;
  }
}

// ------------------------------------------------------------------ reductions
// OP 0: sum_i a[i,c] b[i,c] (per column c);  OP 1: sum_i y_i b_i - log(1 + e^{b_i}) (ncol = 1, a = y, b = b);
// OP 2: sum_i log a_i (ncol = 1)
template <int OP>
__global__ void __launch_bounds__(256) la_reduce_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                        int64_t n, int ncol, int64_t rows_per,
                                                        double* __restrict__ part) {
  __shared__ double sm[256];
  const int t = threadIdx.x;
  const int used = (256 / ncol) * ncol;  // threads in use: thread t always sees column t % ncol
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < n ? r0 + rows_per : n;
  double s = 0.0;
  if (t < used) {
    const int64_t e0 = r0 * ncol, e1 = r1 * ncol;
    for (int64_t e = e0 + t; e < e1; e += used) {
      if (OP == 0) {
        s = fma(a[e], b[e], s);
      } else if (OP == 1) {
        const double bb = b[e];
        s += a[e] * bb - (fmax(bb, 0.0) + log1p(exp(-fabs(bb))));
      } else {
        s += log(a[e]);
      }
    }
  }
  sm[t] = s;
  __syncthreads();
  if (t < ncol) {
    double acc = 0.0;
    for (int q = t; q < used; q += ncol) acc += sm[q];
    part[(size_t)blockIdx.x * ncol + t] = acc;
  }
}

__global__ void la_reduce_final_kernel(const double* __restrict__ part, int nsplit, int ncol, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  double s = 0.0;
  for (int q = 0; q < nsplit; ++q) s += part[(size_t)q * ncol + c];
  out[c] = s;
}

// ------------------------------------------------------------------ elementwise
// Newton step inputs at b: pi = sigma(b), W = pi (1 - pi), winv = 1/W, v = W b + (y - pi)
__global__ void la_newton_prep_kernel(const double* __restrict__ y, const double* __restrict__ b, int64_t n,
                                      double* __restrict__ W, double* __restrict__ winv, double* __restrict__ v,
                                      double* __restrict__ x0) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double bi = b[i];
    const double pi = 1.0 / (1.0 + exp(-bi));
    const double w = pi * (1.0 - pi);
    W[i] = w;
    winv[i] = 1.0 / w;
    v[i] = w * bi + (y[i] - pi);
    if (x0) x0[i] = w * bi;
  }
}

// after the solve: b = x / W = winv x, a = v - x   (P:265 via pcls2)
__global__ void la_newton_update_kernel(const double* __restrict__ x, const double* __restrict__ v,
                                        const double* __restrict__ winv, int64_t n, double* __restrict__ b,
                                        double* __restrict__ a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    b[i] = winv[i] * x[i];
    a[i] = v[i] - x[i];
  }
}

// FITC rows: DV_i = sigma_1^2 - ||u_i||^2 + 1/W_i, dvinv = 1/DV, S_i = u_i / sqrt(DV_i) (App. FITC)
__global__ void la_fitc_rows_kernel(const double* __restrict__ U, int64_t ldu, int mk, int ld, int64_t n,
                                    const double* __restrict__ unorm2, double sigma2, const double* __restrict__ winv,
                                    double* __restrict__ DV, double* __restrict__ dvinv, double* __restrict__ S) {
  const int64_t i = blockIdx.x;
  if (i >= n) return;
  const double dv = sigma2 - unorm2[i] + winv[i];
  const double r = 1.0 / sqrt(dv);
  if (threadIdx.x == 0) {
    DV[i] = dv;
    dvinv[i] = 1.0 / dv;
  }
  for (int k = threadIdx.x; k < ld; k += blockDim.x) S[i * ld + k] = k < mk ? U[i * ldu + k] * r : 0.0;
}

__global__ void la_rownorm2_kernel(const double* __restrict__ U, int64_t ldu, int mk, int64_t n,
                                   double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  double s = 0.0;
  for (int k = lane; k < mk; k += 32) {
    const double u = U[i * ldu + k];
    s = fma(u, u, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[i] = s;
}

// out[i,c] = alpha_row(i) * in[i,c]  (alpha_row = r[i] or sqrt(r[i]))
__global__ void la_rowscale_kernel(const double* __restrict__ in, const double* __restrict__ r, int use_sqrt,
                                   int64_t n, int ncol, double* __restrict__ out) {
  const int64_t tot = n * ncol;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const double s = r[e / ncol];
    out[e] = (use_sqrt ? sqrt(s) : s) * in[e];
  }
}

// out = (a - b) * r_row  (FITC solve tail: P^{-1} w = D_V^{-1} (w - U M_V^{-1} U^T D_V^{-1} w))
__global__ void la_sub_rowscale_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                       const double* __restrict__ r, int64_t n, int ncol, double* __restrict__ out) {
  const int64_t tot = n * ncol;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = (a[e] - b[e]) * r[e / ncol];
}

// CG: r = b - r (in place: r holds A x0), used for a warm start
__global__ void la_residual_kernel(const double* __restrict__ b, int64_t tot, double* __restrict__ r) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x)
    r[e] = b[e] - r[e];
}

// CG step 1: alpha_c = rz_c / pq_c on active columns (0 otherwise), recorded in hist_a[it][c]
__global__ void la_cg_alpha_kernel(const double* __restrict__ rz, const double* __restrict__ pq,
                                   const int* __restrict__ active, int ncol, double* __restrict__ alpha,
                                   double* __restrict__ hist_a) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const double a = active[c] ? rz[c] / pq[c] : 0.0;
  alpha[c] = a;
  if (hist_a) hist_a[c] = a;
}

// CG step 2: x += alpha p, r -= alpha q
__global__ void la_cg_xr_kernel(const double* __restrict__ alpha, const double* __restrict__ p,
                                const double* __restrict__ q, int64_t n, int ncol, double* __restrict__ x,
                                double* __restrict__ r) {
  const int64_t tot = n * ncol;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const double a = alpha[e % ncol];
    x[e] = fma(a, p[e], x[e]);
    r[e] = fma(-a, q[e], r[e]);
  }
}

// CG step 3: beta_c = rz_new_c / rz_c (active), rz = rz_new; recorded in hist_b[it][c]
__global__ void la_cg_beta_kernel(const double* __restrict__ rz_new, double* __restrict__ rz,
                                  const int* __restrict__ active, int ncol, double* __restrict__ beta,
                                  double* __restrict__ hist_b) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const double b = active[c] ? rz_new[c] / rz[c] : 0.0;
  beta[c] = b;
  if (hist_b) hist_b[c] = b;
  if (active[c]) rz[c] = rz_new[c];
}

// CG step 4: p = z + beta p on active columns
__global__ void la_cg_p_kernel(const double* __restrict__ beta, const int* __restrict__ active,
                               const double* __restrict__ z, int64_t n, int ncol, double* __restrict__ p) {
  const int64_t tot = n * ncol;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % ncol);
    if (active[c]) p[e] = fma(beta[c], p[e], z[e]);
  }
}

__global__ void la_transpose_kernel(const double* __restrict__ in, int rows, int cols, int ldin,
                                    double* __restrict__ out, int ldout) {
  const int64_t tot = (int64_t)rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / cols), c = (int)(e % cols);
    out[(int64_t)c * ldout + r] = in[(int64_t)r * ldin + c];
  }
}

// sum_j log L_jj of an in-place Cholesky factor (lower part of A)
__global__ void la_logdiag_kernel(const double* __restrict__ A, int m, int lda, double* __restrict__ out) {
  __shared__ double sm[256];
  double s = 0.0;
  for (int j = threadIdx.x; j < m; j += blockDim.x) s += log(A[(size_t)j * lda + j]);
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = 2.0 * sm[0];
}

// s_i = (b_i + sum_p B[i,p] b_{N(i)_p}) / sqrt(D_i)  (D^{-1/2} B b, for b^T Sigma_dagger^{-1} b)
__global__ void la_bapply_kernel(const int32_t* __restrict__ nbr, const double* __restrict__ Bc, int mv, int64_t n,
                                 const double* __restrict__ D, const double* __restrict__ b, double* __restrict__ s) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = b[i];
    for (int p = 0; p < mv; ++p) {
      const int j = nbr[i * mv + p];
      if (j >= 0) acc = fma(Bc[i * mv + p], b[j], acc);
    }
    s[i] = acc / sqrt(D[i]);
  }
}

// fin[0] = log p(y|b~), fin[1] = s.s, fin[2] = z.z, fin[3] = log det W, fin[4] = sum log D_V,
// fin[5] = log det M_V; slq[c] = e1^T log(T_c) e1.  out = (nll, -log p, quad, logdet, logdet_W, logdet_P)
// with L = -log p + quad / 2 + logdet / 2 and logdet from slq_v2
__global__ void la_finish_kernel(const double* __restrict__ fin, const double* __restrict__ slq, int64_t n, int ell,
                                 double* __restrict__ out) {
  const double quad = fin[1] - fin[2];
  const double ldP = fin[4] + fin[5];
  double ssum = 0.0;
  for (int c = 0; c < ell; ++c) ssum += slq[c];
  const double logdet = ell > 0 ? fin[3] + (double)n / ell * ssum + ldP : 0.0;
  out[0] = -fin[0] + 0.5 * quad + 0.5 * logdet;
  out[1] = -fin[0];
  out[2] = quad;
  out[3] = logdet;
  out[4] = fin[3];
  out[5] = ldP;
}

// ------------------------------------------------------------------ SLQ quadrature
// One thread per probe c: T (k x k tridiagonal) from the CG coefficients:
//   T_jj = 1/alpha_j + beta_{j-1}/alpha_{j-1},  T_{j,j+1} = sqrt(beta_j)/alpha_j
// eigen-decomposition by the implicit QL iteration with Wilkinson shifts, tracking only the first
// row of the eigenvector matrix; e_1^T log(T) e_1 = sum_k q_{1k}^2 log(lambda_k).
// d, e, q: per-probe scratch of kmax doubles each.
__global__ void la_slq_kernel(const double* __restrict__ hist_a, const double* __restrict__ hist_b,
                              const int* __restrict__ iters, int ncol, int kmax, double* __restrict__ scratch,
                              double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const int k = iters[c];
  double* d = scratch + (size_t)c * 3 * kmax;
  double* e = d + kmax;
  double* q = e + kmax;
  for (int j = 0; j < k; ++j) {
    const double aj = hist_a[(size_t)j * ncol + c];
    d[j] = 1.0 / aj + (j > 0 ? hist_b[(size_t)(j - 1) * ncol + c] / hist_a[(size_t)(j - 1) * ncol + c] : 0.0);
    e[j] = j + 1 < k ? sqrt(hist_b[(size_t)j * ncol + c]) / aj : 0.0;
    q[j] = j == 0 ? 1.0 : 0.0;
  }
  // implicit QL (symmetric tridiagonal): e[j] couples d[j], d[j+1]
  for (int l = 0; l < k; ++l) {
    for (int it = 0; it < 60; ++it) {
      int mm = l;
      for (; mm < k - 1; ++mm) {
        const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(e[mm]) <= 1e-16 * dd) break;
      }
      if (mm == l) break;
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = hypot(g, 1.0);
      g = d[mm] - d[l] + e[l] / (g + (g >= 0.0 ? r : -r));
      double s = 1.0, cc = 1.0, p = 0.0;
      int i = mm - 1;
      bool early = false;
      for (; i >= l; --i) {
        double f = s * e[i];
        const double b = cc * e[i];
        r = hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= p;
          e[mm] = 0.0;
          early = true;
          break;
        }
        s = f / r;
        cc = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0 * cc * b;
        p = s * r;
        d[i + 1] = g + p;
        g = cc * r - b;
        // first-row rotation of the eigenvector matrix (columns i, i+1)
        f = q[i + 1];
        q[i + 1] = s * q[i] + cc * f;
        q[i] = cc * q[i] - s * f;
      }
      if (early) continue;
      d[l] -= p;
      e[l] = g;
      e[mm] = 0.0;
    }
  }
  double sum = 0.0;
  for (int j = 0; j < k; ++j) sum += q[j] * q[j] * log(d[j]);
  out[c] = sum;
}

}  // namespace

// ============================================================================ launchers
static unsigned grid_for(int64_t work, int per = 256) {
  int64_t g = (work + per - 1) / per;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (unsigned)g;
}

cudaError_t launch_la_transpose_struct(const int32_t* nbr, int64_t n, int mv, int* cnt, int* cursor, int* tptr,
                                       int* tpos, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(cnt, 0, (size_t)n * sizeof(int), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(cursor, 0, (size_t)n * sizeof(int), s);
  if (e != cudaSuccess) return e;
  if (mv > 0) la_count_kernel<<<grid_for(n * mv), 256, 0, s>>>(nbr, n, mv, cnt);
  la_scan_kernel<<<1, 1024, 0, s>>>(cnt, n, tptr);
  if (mv > 0) {
    la_fill_kernel<<<grid_for(n * mv), 256, 0, s>>>(nbr, n, mv, tptr, cursor, tpos);
    la_sort_kernel<<<grid_for(n), 256, 0, s>>>(n, tptr, tpos);
  }
  return cudaGetLastError();
}

static int la_trsv_blocks(const void* fn) {
  static int cached[2] = {0, 0};
  int idx = fn == (const void*)la_trsv_fwd_kernel ? 0 : 1;
  if (!cached[idx]) {
    int per_sm = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, LA_THREADS, 0);
    cached[idx] = sms * (per_sm > 0 ? per_sm : 1);
  }
  return cached[idx];
}

cudaError_t launch_la_trsv_fwd(const int32_t* nbr, const double* Bc, int mv, int64_t n, int ncol, const double* v,
                               const double* scale, double* x, const double* v2, const double* w2, double* out2,
                               int* flags, int epoch, unsigned long long* ticket, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(ticket, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  int64_t blocks = la_trsv_blocks((const void*)la_trsv_fwd_kernel);
  const int64_t need = (n + LA_WARPS - 1) / LA_WARPS;
  if (blocks > need) blocks = need;
  la_trsv_fwd_kernel<<<(unsigned)blocks, LA_THREADS, 0, s>>>(nbr, Bc, mv, n, ncol, v, scale, x, v2, w2, out2, flags,
                                                              epoch, ticket);
  return cudaGetLastError();
}

cudaError_t launch_la_trsv_bwd(const int* tptr, const int* tpos, const double* Bc, int mv, int64_t n, int ncol,
                               const double* u, double* y, int* flags, int epoch, unsigned long long* ticket,
                               cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(ticket, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  int64_t blocks = la_trsv_blocks((const void*)la_trsv_bwd_kernel);
  const int64_t need = (n + LA_WARPS - 1) / LA_WARPS;
  if (blocks > need) blocks = need;
  la_trsv_bwd_kernel<<<(unsigned)blocks, LA_THREADS, 0, s>>>(tptr, tpos, Bc, mv > 0 ? mv : 1, n, ncol, u, y, flags,
                                                              epoch, ticket);
  return cudaGetLastError();
}

int la_ts_nsplit(int64_t n) {
  int64_t ns = (n + 4095) / 4096;
  if (ns > 296) ns = 296;
  if (ns < 1) ns = 1;
  return (int)ns;
}

cudaError_t launch_la_tsgemm(const double* U, int64_t ldu, int mk, int64_t n, const double* V, int ncol,
                             const int64_t* vrow, const double* rs, double* part, double* Ct, double alpha,
                             cudaStream_t s) {
  if (mk == 0) return cudaSuccess;
  const int ns = la_ts_nsplit(n);
  const int64_t rows_per = (n + ns - 1) / ns;
  dim3 grid(ns, (mk + TS_K - 1) / TS_K);
  if (ncol <= 1)
    la_tsgemm_kernel<1><<<grid, 256, 0, s>>>(U, ldu, mk, n, V, ncol, vrow, rs, rows_per, part);
  else if (ncol <= 8)
    la_tsgemm_kernel<8><<<grid, 256, 0, s>>>(U, ldu, mk, n, V, ncol, vrow, rs, rows_per, part);
  else if (ncol <= 16)
    la_tsgemm_kernel<16><<<grid, 256, 0, s>>>(U, ldu, mk, n, V, ncol, vrow, rs, rows_per, part);
  else if (ncol <= 32)
    la_tsgemm_kernel<32><<<grid, 256, 0, s>>>(U, ldu, mk, n, V, ncol, vrow, rs, rows_per, part);
  else if (ncol <= 64)
    la_tsgemm_kernel<64><<<grid, 256, 0, s>>>(U, ldu, mk, n, V, ncol, vrow, rs, rows_per, part);
  else
    return cudaErrorInvalidValue;
  la_tsreduce_kernel<<<grid_for((int64_t)ncol * mk), 256, 0, s>>>(part, ns, ncol, mk, Ct, alpha);
  return cudaGetLastError();
}

int la_red_nsplit(int64_t n) {
  int64_t ns = (n + 8191) / 8192;
  if (ns > 592) ns = 592;
  if (ns < 1) ns = 1;
  return (int)ns;
}

cudaError_t launch_la_reduce(int op, const double* a, const double* b, int64_t n, int ncol, double* part,
                             double* out, cudaStream_t s) {
  if (ncol < 1 || ncol > 256) return cudaErrorInvalidValue;
  const int ns = la_red_nsplit(n);
  const int64_t rows_per = (n + ns - 1) / ns;
  switch (op) {
    case 0: la_reduce_kernel<0><<<ns, 256, 0, s>>>(a, b, n, ncol, rows_per, part); break;
    case 1: la_reduce_kernel<1><<<ns, 256, 0, s>>>(a, b, n, 1, rows_per, part); break;
    default: la_reduce_kernel<2><<<ns, 256, 0, s>>>(a, b, n, 1, rows_per, part); break;
  }
  la_reduce_final_kernel<<<(ncol + 255) / 256, 256, 0, s>>>(part, ns, op == 0 ? ncol : 1, out);
  return cudaGetLastError();
}

cudaError_t launch_la_newton_prep(const double* y, const double* b, int64_t n, double* W, double* winv, double* v,
                                  double* x0, cudaStream_t s) {
  la_newton_prep_kernel<<<grid_for(n), 256, 0, s>>>(y, b, n, W, winv, v, x0);
  return cudaGetLastError();
}

cudaError_t launch_la_newton_update(const double* x, const double* v, const double* winv, int64_t n, double* b,
                                    double* a, cudaStream_t s) {
  la_newton_update_kernel<<<grid_for(n), 256, 0, s>>>(x, v, winv, n, b, a);
  return cudaGetLastError();
}

cudaError_t launch_la_fitc_rows(const double* U, int64_t ldu, int mk, int ld, int64_t n, const double* unorm2,
                                double sigma2, const double* winv, double* DV, double* dvinv, double* S,
                                cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  la_fitc_rows_kernel<<<(unsigned)n, 128, 0, s>>>(U, ldu, mk, ld, n, unorm2, sigma2, winv, DV, dvinv, S);
  return cudaGetLastError();
}

cudaError_t launch_la_rownorm2(const double* U, int64_t ldu, int mk, int64_t n, double* out, cudaStream_t s) {
  la_rownorm2_kernel<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(U, ldu, mk, n, out);
  return cudaGetLastError();
}

cudaError_t launch_la_rowscale(const double* in, const double* r, int use_sqrt, int64_t n, int ncol, double* out,
                               cudaStream_t s) {
  la_rowscale_kernel<<<grid_for(n * ncol), 256, 0, s>>>(in, r, use_sqrt, n, ncol, out);
  return cudaGetLastError();
}

cudaError_t launch_la_sub_rowscale(const double* a, const double* b, const double* r, int64_t n, int ncol, double* out,
                                   cudaStream_t s) {
  la_sub_rowscale_kernel<<<grid_for(n * ncol), 256, 0, s>>>(a, b, r, n, ncol, out);
  return cudaGetLastError();
}

cudaError_t launch_la_residual(const double* b, int64_t tot, double* r, cudaStream_t s) {
  la_residual_kernel<<<grid_for(tot), 256, 0, s>>>(b, tot, r);
  return cudaGetLastError();
}

cudaError_t launch_la_cg_alpha(const double* rz, const double* pq, const int* active, int ncol, double* alpha,
                               double* hist_a, cudaStream_t s) {
  la_cg_alpha_kernel<<<(ncol + 127) / 128, 128, 0, s>>>(rz, pq, active, ncol, alpha, hist_a);
  return cudaGetLastError();
}

cudaError_t launch_la_cg_xr(const double* alpha, const double* p, const double* q, int64_t n, int ncol, double* x,
                            double* r, cudaStream_t s) {
  la_cg_xr_kernel<<<grid_for(n * ncol), 256, 0, s>>>(alpha, p, q, n, ncol, x, r);
  return cudaGetLastError();
}

cudaError_t launch_la_cg_beta(const double* rz_new, double* rz, const int* active, int ncol, double* beta,
                              double* hist_b, cudaStream_t s) {
  la_cg_beta_kernel<<<(ncol + 127) / 128, 128, 0, s>>>(rz_new, rz, active, ncol, beta, hist_b);
  return cudaGetLastError();
}

cudaError_t launch_la_cg_p(const double* beta, const int* active, const double* z, int64_t n, int ncol, double* p,
                           cudaStream_t s) {
  la_cg_p_kernel<<<grid_for(n * ncol), 256, 0, s>>>(beta, active, z, n, ncol, p);
  return cudaGetLastError();
}

cudaError_t launch_la_transpose(const double* in, int rows, int cols, int ldin, double* out, int ldout, cudaStream_t s) {
  la_transpose_kernel<<<grid_for((int64_t)rows * cols), 256, 0, s>>>(in, rows, cols, ldin, out, ldout);
  return cudaGetLastError();
}

cudaError_t launch_la_logdiag(const double* A, int m, int lda, double* out, cudaStream_t s) {
  la_logdiag_kernel<<<1, 256, 0, s>>>(A, m, lda, out);
  return cudaGetLastError();
}

cudaError_t launch_la_slq(const double* hist_a, const double* hist_b, const int* iters, int ncol, int kmax,
                          double* scratch, double* out, cudaStream_t s) {
  la_slq_kernel<<<(ncol + 31) / 32, 32, 0, s>>>(hist_a, hist_b, iters, ncol, kmax, scratch, out);
  return cudaGetLastError();
}

cudaError_t launch_la_bapply(const int32_t* nbr, const double* Bc, int mv, int64_t n, const double* D, const double* b,
                             double* s, cudaStream_t st) {
  la_bapply_kernel<<<grid_for(n), 256, 0, st>>>(nbr, Bc, mv, n, D, b, s);
  return cudaGetLastError();
}

cudaError_t launch_la_finish(const double* fin, const double* slq, int64_t n, int ell, double* out, cudaStream_t s) {
  la_finish_kernel<<<1, 1, 0, s>>>(fin, slq, n, ell, out);
  return cudaGetLastError();
}

}  // namespace vif
