// k_dense.cu -- K0 / K5: the two m x m dense factorizations of the path, and the NLL finish.
//
//   K0: K_m = K(Z,Z) + eps I (reading c3); L_m = chol(K_m); L_m^{-1}  (for U = K L_m^{-T})
//   K5: M_w = I + G_WW;  L_M = chol(M_w);  z = L_M^{-1} G_Wr;  quad = G_rr - z.z;
//       logdet M_w = 2 sum log (L_M)_jj;  NLL = n/2 log 2pi + (sum log D + logdet M_w + quad)/2
//
//
// chol_inv_kernel: one cooperative persistent kernel (grid = SMs), 32 x 32 tiles, right-looking:
//   per panel k: (A) one warp factors the diagonal tile in registers (row per lane, column
//   broadcast through shared memory, inline rsqrt) and inverts it (column-oriented substitution);
//   (B) L_ik = A_ik inv(L_kk)^T for i > k; (C) trailing update A_ij -= L_ik L_jk^T; grid sync between.
//   If the inverse is wanted (K0 only), it is completed by recursive doubling over the tile grid:
//   inv([[P,0],[C,Q]]) = [[P^-1, 0], [-Q^-1 C P^-1, Q^-1]] with block sizes 1, 2, 4, ... tiles,
//   two fully parallel GEMM steps per level (log2(m/32) levels) instead of a sequential wavefront.
// K5 needs only the diagonal-tile inverses (they drive the blocked forward solve in finish_kernel).
// These are O(m^3/3) once per evaluation: 4e7 flops at m = 500.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace vif {

namespace {

constexpr int TB = 32;  // tile size

__device__ __forceinline__ void load_tile(double (*T)[TB + 1], const double* A, int lda, int lim, int ti, int tj) {
  for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
    const int r = e / TB, c = e % TB;
    const int gr = ti * TB + r, gc = tj * TB + c;
    T[r][c] = (gr < lim && gc < lim) ? __ldcg(A + (size_t)gr * lda + gc) : 0.0;
  }
}

__device__ __forceinline__ void store_tile(const double (*T)[TB + 1], double* A, int lda, int lim, int ti, int tj) {
  for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
    const int r = e / TB, c = e % TB;
    const int gr = ti * TB + r, gc = tj * TB + c;
    if (gr < lim && gc < lim) __stcg(A + (size_t)gr * lda + gc, T[r][c]);
  }
}

struct Smem {
  double T[TB][TB + 1];
  double P[TB][TB + 1];
  double Q[TB][TB + 1];
  double R[TB][TB + 1];
  double cb[2][TB];
};

// acc[j] (rows r0 + 8j, column c) += sign * P Q^T  (TRANSB) or P Q
template <bool TRANSB>
__device__ __forceinline__ void tile_mac(const Smem& sm, double acc[4], int r0, int c) {
#pragma unroll 8
  for (int t = 0; t < TB; ++t) {
    const double q = TRANSB ? sm.Q[c][t] : sm.Q[t][c];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j] = fma(sm.P[r0 + 8 * j][t], q, acc[j]);
  }
}

// warp 0: factor sm.T (lower, SPD) in place and write inv(L) into sm.P
__device__ void factor_diag_tile(Smem& sm, int* fail) {
  const int lane = threadIdx.x & 31;
  double crow[TB];
#pragma unroll
  for (int c = 0; c < TB; ++c) crow[c] = c <= lane ? sm.T[lane][c] : 0.0;
  bool ok = true;
  double myinv = 1.0;
#pragma unroll
  for (int j = 0; j < TB; ++j) {
    const double djj = __shfl_sync(0xffffffffu, crow[j], j);
    ok = ok && (djj > 0.0);
    const double y = rsqrt_nr(djj);
    const double lrj = crow[j] * y;
    crow[j] = lrj;
    if (lane == j) myinv = y;
    if (j + 1 < TB) {
      sm.cb[j & 1][lane] = lrj;
      __syncwarp();
#pragma unroll
      for (int c = j + 1; c < TB; ++c) crow[c] = fma(-lrj, sm.cb[j & 1][c], crow[c]);
    }
  }
  if (!ok && lane == 0) atomicExch(fail, 1);
#pragma unroll
  for (int c = 0; c < TB; ++c) sm.T[lane][c] = c <= lane ? crow[c] : 0.0;
  __syncwarp();
  // inverse: lane = column c of X with L X = I; column-oriented forward substitution
  double x[TB];
#pragma unroll
  for (int r = 0; r < TB; ++r) x[r] = r == lane ? 1.0 : 0.0;
#pragma unroll
  for (int q = 0; q < TB; ++q) {
    const double inv_qq = __shfl_sync(0xffffffffu, myinv, q);
    x[q] *= inv_qq;
#pragma unroll
    for (int r = q + 1; r < TB; ++r) x[r] = fma(-sm.T[r][q], x[q], x[r]);
  }
#pragma unroll
  for (int r = 0; r < TB; ++r) sm.P[r][lane] = x[r];
  __syncwarp();
}

}  // namespace

// In-place Cholesky of the m x m symmetric matrix A (+ diag_add * I), lower part (the upper part is
// scratch afterwards).  Linv (lim_inv x lim_inv, ld ldi, pre-zeroed by the caller) receives the
// inverses of the diagonal tiles, and the full lower inverse when full_inverse != 0.
// fail: set to 1 on a non-positive pivot.
__global__ void __launch_bounds__(256) chol_inv_kernel(double* A, int m, int lda, double diag_add, double* Linv,
                                                       int ldi, int lim_inv, int full_inverse, double* Tscr,
                                                       int* fail) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Smem sm;
  const int nt = (m + TB - 1) / TB;
  const int tid = threadIdx.x;
  const int c = tid & 31, r0 = tid >> 5;  // thread -> (rows r0 + 8j, col c)

  for (int k = 0; k < nt; ++k) {
    // ---- A: factor + invert the diagonal tile ----
    if (blockIdx.x == 0) {
      for (int e = tid; e < TB * TB; e += blockDim.x) {
        const int r = e / TB, cc = e % TB;
        const int gr = k * TB + r, gc = k * TB + cc;
        double v;
        if (gr < m && gc < m) v = cc <= r ? __ldcg(A + (size_t)gr * lda + gc) + (r == cc ? diag_add : 0.0) : 0.0;
        else v = r == cc ? 1.0 : 0.0;  // identity padding beyond m
        sm.T[r][cc] = v;
      }
      __syncthreads();
      if (tid < 32) factor_diag_tile(sm, fail);
      __syncthreads();
      store_tile(sm.T, A, lda, m, k, k);
      store_tile(sm.P, Linv, ldi, lim_inv, k, k);
    }
    grid.sync();
    // ---- B: L_ik = A_ik inv(L_kk)^T ----
    for (int i = k + 1 + blockIdx.x; i < nt; i += gridDim.x) {
      load_tile(sm.P, A, lda, m, i, k);
      load_tile(sm.Q, Linv, ldi, lim_inv, k, k);
      __syncthreads();
      double acc[4] = {0, 0, 0, 0};
      tile_mac<true>(sm, acc, r0, c);
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 4; ++j) sm.P[r0 + 8 * j][c] = acc[j];
      __syncthreads();
      store_tile(sm.P, A, lda, m, i, k);
      __syncthreads();
    }
    grid.sync();
    // ---- C: trailing update A_ij -= L_ik L_jk^T, k < j <= i ----
    const int ntr = nt - k - 1;
    const int cnt = ntr * (ntr + 1) / 2;
    for (int t = blockIdx.x; t < cnt; t += gridDim.x) {
      int ii = 0;
      while ((ii + 1) * (ii + 2) / 2 <= t) ++ii;
      const int jj = t - ii * (ii + 1) / 2;
      const int i = k + 1 + ii, j = k + 1 + jj;
      load_tile(sm.P, A, lda, m, i, k);
      load_tile(sm.Q, A, lda, m, j, k);
      load_tile(sm.R, A, lda, m, i, j);
      __syncthreads();
      double acc[4] = {0, 0, 0, 0};
      tile_mac<true>(sm, acc, r0, c);
#pragma unroll
      for (int jx = 0; jx < 4; ++jx) sm.R[r0 + 8 * jx][c] -= acc[jx];
      __syncthreads();
      store_tile(sm.R, A, lda, m, i, j);
      __syncthreads();
    }
    grid.sync();
  }
  if (!full_inverse) return;
  // ---- recursive doubling: blocks of 2h tiles starting at b = 2h * blk ----
  // T = C inv(P) goes to the scratch Tscr (same shape as Linv) at tile (r, c).
  for (int h = 1; h < nt; h *= 2) {
    const int nblk = (nt + 2 * h - 1) / (2 * h);
    // step 1: T_rc = sum_{q in [b, b+h)} L_rq Linv_qc   for r in [b+h, b+2h), c in [b, b+h)
    for (int w = blockIdx.x; w < nblk * h * h; w += gridDim.x) {
      const int blk = w / (h * h), rc = w % (h * h);
      const int b = blk * 2 * h;
      const int r = b + h + rc / h, cc = b + rc % h;
      if (r >= nt) continue;
      double acc[4] = {0, 0, 0, 0};
      for (int q = cc; q < b + h; ++q) {  // Linv_qc = 0 for q < c
        load_tile(sm.P, A, lda, m, r, q);
        load_tile(sm.Q, Linv, ldi, lim_inv, q, cc);
        __syncthreads();
        tile_mac<false>(sm, acc, r0, c);
        __syncthreads();
      }
#pragma unroll
      for (int jx = 0; jx < 4; ++jx) sm.R[r0 + 8 * jx][c] = acc[jx];
      __syncthreads();
      store_tile(sm.R, Tscr, ldi, lim_inv, r, cc);
      __syncthreads();
    }
    grid.sync();
    // step 2: Linv_rc = - sum_{q in [b+h, r]} Linv_rq T_qc
    for (int w = blockIdx.x; w < nblk * h * h; w += gridDim.x) {
      const int blk = w / (h * h), rc = w % (h * h);
      const int b = blk * 2 * h;
      const int r = b + h + rc / h, cc = b + rc % h;
      if (r >= nt) continue;
      double acc[4] = {0, 0, 0, 0};
      for (int q = b + h; q <= r; ++q) {
        load_tile(sm.P, Linv, ldi, lim_inv, r, q);
        load_tile(sm.Q, Tscr, ldi, lim_inv, q, cc);
        __syncthreads();
        tile_mac<false>(sm, acc, r0, c);
        __syncthreads();
      }
#pragma unroll
      for (int jx = 0; jx < 4; ++jx) sm.R[r0 + 8 * jx][c] = -acc[jx];
      __syncthreads();
      store_tile(sm.R, Linv, ldi, lim_inv, r, cc);
      __syncthreads();
    }
    grid.sync();
  }
}

// K_m[a][b] = k(z_a, z_b) + eps [a == b]  (reading c3)
template <int FAM>
__global__ void build_km_kernel(const double* __restrict__ Z, int m, CovParams p, double* __restrict__ Km) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)m * m) return;
  const int a = (int)(e / m), b = (int)(e % m);
  double v = cov<FAM>(Z + (size_t)a * p.d, Z + (size_t)b * p.d, p);
  if (a == b) v += p.jitter;
  Km[e] = v;
}

// Deterministic two-stage sum of log D over the owned points (sum_i log D_i).
__global__ void __launch_bounds__(256) logd_partial_kernel(const double* __restrict__ Dpos, int64_t npts,
                                                           double* __restrict__ partials) {
  __shared__ double red[256];
  const int64_t per = (npts + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = (int64_t)blockIdx.x * per;
  const int64_t b1 = b0 + per < npts ? b0 + per : npts;
  double s = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) s += log(Dpos[i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}

__global__ void sum_partials_kernel(const double* __restrict__ partials, int np, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < np; ++i) s += partials[i];
    *out = s;
  }
}

// Finish (after the all-reduce and the Cholesky of M_w), one CTA:
//   z = L_M^{-1} g by blocked forward substitution (g = G_Wr = row ycol of G; the diagonal-tile
//   inverses come from chol_inv_kernel), quad = G_rr - z.z, logdet M_w = 2 sum log L_jj, NLL.
// terms[0..3] = nll, logdetD, logdetM, quad.
__global__ void __launch_bounds__(1024) finish_kernel(const double* __restrict__ G, int ld, int m, int ycol,
                                                      const double* __restrict__ Dinv, int ldi,
                                                      const double* __restrict__ logdetD_dev, int64_t n,
                                                      double* __restrict__ terms) {
  __shared__ double z[2048];
  __shared__ double rhs[TB];
  __shared__ double part[32];
  __shared__ double red[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nt = (m + TB - 1) / TB;
  for (int k = 0; k < nt; ++k) {
    // rhs_r = g_r - sum_{c < 32k} L[r][c] z_c : warp w takes row r = 32k + w, lanes over c (coalesced)
    const int r = k * TB + warp;
    double s = 0.0;
    if (r < m)
      for (int cc = lane; cc < k * TB; cc += 32) s = fma(G[(size_t)r * ld + cc], z[cc], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) rhs[warp] = r < m ? G[(size_t)ycol * ld + r] - s : 0.0;
    __syncthreads();
    if (warp == 0) {
      // z_block = inv(L_kk) rhs  (diagonal-tile inverse stored at Dinv tile (k, k))
      const int rr = k * TB + lane;
      double zz = 0.0;
      if (rr < m)
        for (int cc = 0; cc <= lane; ++cc) zz = fma(Dinv[(size_t)rr * ldi + k * TB + cc], rhs[cc], zz);
      if (rr < m) z[rr] = zz;
    }
    __syncthreads();
  }
  double zs = 0.0, ls = 0.0;
  for (int a = tid; a < m; a += blockDim.x) {
    zs += z[a] * z[a];
    ls += 2.0 * log(G[(size_t)a * ld + a]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    zs += __shfl_xor_sync(0xffffffffu, zs, o);
    ls += __shfl_xor_sync(0xffffffffu, ls, o);
  }
  if (lane == 0) {
    part[warp] = zs;
    red[warp] = ls;
  }
  __syncthreads();
  if (tid == 0) {
    double z2 = 0.0, lm = 0.0;
    for (int w = 0; w < 32; ++w) {
      z2 += part[w];
      lm += red[w];
    }
    const double lD = *logdetD_dev;
    const double quad = G[(size_t)ycol * ld + ycol] - z2;
    terms[0] = 0.5 * (double)n * 1.8378770664093453 + 0.5 * (lD + lm) + 0.5 * quad;  // log(2 pi)
    terms[1] = lD;
    terms[2] = lm;
    terms[3] = quad;
  }
}

// ----------------------------------------------------------------------------- launchers
cudaError_t launch_build_km(const double* Z, int m, const CovParams& p, double* Km, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const int64_t tot = (int64_t)m * m;
  const int blocks = (int)((tot + 255) / 256);
  switch (p.family) {
    case FAM_M12: build_km_kernel<FAM_M12><<<blocks, 256, 0, s>>>(Z, m, p, Km); break;
    case FAM_M32: build_km_kernel<FAM_M32><<<blocks, 256, 0, s>>>(Z, m, p, Km); break;
    case FAM_M52: build_km_kernel<FAM_M52><<<blocks, 256, 0, s>>>(Z, m, p, Km); break;
    default: build_km_kernel<FAM_GAUSS><<<blocks, 256, 0, s>>>(Z, m, p, Km); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_chol_inv(double* A, int m, int lda, double diag_add, double* Linv, int ldi, int lim_inv,
                            int full_inverse, double* Tscr, int* fail, int num_sms, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  int blocks_per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, chol_inv_kernel, 256, 0);
  if (e != cudaSuccess) return e;
  if (blocks_per_sm < 1) return cudaErrorLaunchOutOfResources;
  const int nt = (m + TB - 1) / TB;
  int grid = num_sms;
  const int need = nt * nt;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  void* args[] = {&A, &m, &lda, &diag_add, &Linv, &ldi, &lim_inv, &full_inverse, &Tscr, &fail};
  return cudaLaunchCooperativeKernel((void*)chol_inv_kernel, dim3(grid), dim3(256), args, 0, s);
}

cudaError_t launch_logd_sum(const double* Dpos, int64_t npts, double* partials, int np, double* out,
                            cudaStream_t s) {
  logd_partial_kernel<<<np, 256, 0, s>>>(Dpos, npts, partials);
  sum_partials_kernel<<<1, 32, 0, s>>>(partials, np, out);
  return cudaGetLastError();
}

cudaError_t launch_finish(const double* G, int ld, int m, int ycol, const double* Dinv, int ldi,
                          const double* logdetD_dev, int64_t n, double* terms, cudaStream_t s) {
  if (m > 2048) return cudaErrorInvalidValue;
  finish_kernel<<<1, 1024, 0, s>>>(G, ld, m, ycol, Dinv, ldi, logdetD_dev, n, terms);
  return cudaGetLastError();
}

}  // namespace vif
