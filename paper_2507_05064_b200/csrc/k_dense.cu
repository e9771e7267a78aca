// k_dense.cu -- K0 / K5: the two m x m dense factorizations of the path, and the NLL finish.
//
//   K0: K_m = K(Z,Z) + eps I (reading c3); L_m = chol(K_m); L_m^{-1}  (for U = K L_m^{-T})
//   K5: M_w = I + G_WW;  L_M = chol(M_w);  z = L_M^{-1} G_Wr;  quad = G_rr - z.z;
//       logdet M_w = 2 sum log (L_M)_jj;  NLL = n/2 log 2pi + (sum log D + logdet M_w + quad)/2
//
//
// Both factorizations use one cooperative persistent kernel (one CTA per SM, grid-wide sync
// between the phases of a right-looking blocked Cholesky with 32x32 tiles, then a wavefront
// over the tile diagonals for the triangular inverse).  These are O(m^3/3) once per
// evaluation: 4e7 flops at m = 500, 1.1e9 at m = 1500 -- < 1% of the O(n m^2) work.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace vif {

namespace {

constexpr int TB = 32;  // tile size

// element (r, c) of the symmetric input (lower part stored), identity beyond m
__device__ __forceinline__ double ld_sym(const double* A, int lda, int m, int r, int c, double diag_add) {
  if (r < m && c < m) return __ldcg(A + (size_t)r * lda + c) + (r == c ? diag_add : 0.0);
  return r == c ? 1.0 : 0.0;
}

// load tile (ti, tj) of a lower-stored matrix into smem, zero beyond `lim`
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
    if (gr < lim && gc < lim) A[(size_t)gr * lda + gc] = T[r][c];
  }
}

struct Smem {
  double T[TB][TB + 1];
  double P[TB][TB + 1];
  double Q[TB][TB + 1];
  double R[TB][TB + 1];
};

}  // namespace

// In-place Cholesky of the m x m symmetric matrix A (+ diag_add * I), lower part; writes the lower
// triangular inverse to Linv (lim_inv x lim_inv, ld ldi, upper part left untouched: caller zeroes).
// fail: set to 1 on a non-positive pivot.
__global__ void __launch_bounds__(256) chol_inv_kernel(double* A, int m, int lda, double diag_add, double* Linv,
                                                       int ldi, int lim_inv, int* fail) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Smem sm;
  const int nt = (m + TB - 1) / TB;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int c = tid & 31, r0 = tid >> 5;  // thread -> (rows r0 + 8j, col c)

  for (int k = 0; k < nt; ++k) {
    // ---- phase A: factor the diagonal tile and invert it (block 0) ----
    if (blockIdx.x == 0) {
      for (int e = tid; e < TB * TB; e += blockDim.x) {
        const int r = e / TB, cc = e % TB;
        sm.T[r][cc] = cc <= r ? ld_sym(A, lda, m, k * TB + r, k * TB + cc, diag_add) : 0.0;
      }
      __syncthreads();
      if (tid < 32) {
        for (int j = 0; j < TB; ++j) {
          const double djj = sm.T[j][j];
          if (!(djj > 0.0) && lane == 0) atomicExch(fail, 1);
          const double ljj = sqrt(djj);
          __syncwarp();
          if (lane > j) sm.T[lane][j] /= ljj;
          __syncwarp();
          if (lane == j) sm.T[j][j] = ljj;
          if (lane > j) {
            const double lrj = sm.T[lane][j];
            for (int cc = j + 1; cc <= lane; ++cc) sm.T[lane][cc] -= lrj * sm.T[cc][j];
          }
          __syncwarp();
        }
        // inverse of the lower-triangular tile, lane = column
        for (int r = 0; r < TB; ++r) {
          double v;
          if (r < lane) {
            v = 0.0;
          } else if (r == lane) {
            v = 1.0 / sm.T[r][r];
          } else {
            double s = 0.0;
            for (int q = lane; q < r; ++q) s += sm.T[r][q] * sm.P[q][lane];
            v = -s / sm.T[r][r];
          }
          sm.P[r][lane] = v;
        }
      }
      __syncthreads();
      store_tile(sm.T, A, lda, m, k, k);
      store_tile(sm.P, Linv, ldi, lim_inv, k, k);
      // identity padding of Linv beyond m inside the diagonal tile is stored when lim_inv > m
    }
    grid.sync();
    // ---- phase B: L_ik = A_ik L_kk^{-T} for i > k ----
    for (int i = k + 1 + blockIdx.x; i < nt; i += gridDim.x) {
      load_tile(sm.P, A, lda, m, i, k);
      load_tile(sm.Q, Linv, ldi, lim_inv, k, k);
      __syncthreads();
      double acc[4] = {0, 0, 0, 0};
#pragma unroll 8
      for (int t = 0; t < TB; ++t) {
        const double q = sm.Q[c][t];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] += sm.P[r0 + 8 * j][t] * q;
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 4; ++j) sm.P[r0 + 8 * j][c] = acc[j];
      __syncthreads();
      store_tile(sm.P, A, lda, m, i, k);
      __syncthreads();
    }
    grid.sync();
    // ---- phase C: trailing update A_ij -= L_ik L_jk^T, k < j <= i ----
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
#pragma unroll 8
      for (int q = 0; q < TB; ++q) {
        const double b = sm.Q[c][q];
#pragma unroll
        for (int jx = 0; jx < 4; ++jx) acc[jx] += sm.P[r0 + 8 * jx][q] * b;
      }
#pragma unroll
      for (int jx = 0; jx < 4; ++jx) sm.R[r0 + 8 * jx][c] -= acc[jx];
      __syncthreads();
      store_tile(sm.R, A, lda, m, i, j);
      __syncthreads();
    }
    grid.sync();
  }
  // ---- triangular inverse, wavefront over tile diagonals t = i - j ----
  for (int t = 1; t < nt; ++t) {
    for (int j = blockIdx.x; j + t < nt; j += gridDim.x) {
      const int i = j + t;
      double acc[4] = {0, 0, 0, 0};
      for (int k = j; k < i; ++k) {
        load_tile(sm.P, A, lda, m, i, k);          // L_ik
        load_tile(sm.Q, Linv, ldi, lim_inv, k, j);  // Linv_kj
        __syncthreads();
#pragma unroll 8
        for (int q = 0; q < TB; ++q) {
          const double b = sm.Q[q][c];
#pragma unroll
          for (int jx = 0; jx < 4; ++jx) acc[jx] += sm.P[r0 + 8 * jx][q] * b;
        }
        __syncthreads();
      }
#pragma unroll
      for (int jx = 0; jx < 4; ++jx) sm.R[r0 + 8 * jx][c] = acc[jx];
      load_tile(sm.P, Linv, ldi, lim_inv, i, i);  // Linv_ii
      __syncthreads();
      double out[4] = {0, 0, 0, 0};
#pragma unroll 8
      for (int q = 0; q < TB; ++q) {
        const double b = sm.R[q][c];
#pragma unroll
        for (int jx = 0; jx < 4; ++jx) out[jx] -= sm.P[r0 + 8 * jx][q] * b;
      }
      __syncthreads();
#pragma unroll
      for (int jx = 0; jx < 4; ++jx) sm.R[r0 + 8 * jx][c] = out[jx];
      __syncthreads();
      store_tile(sm.R, Linv, ldi, lim_inv, i, j);
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

// Finish (after the all-reduce and the Cholesky of M_w): terms[0..3] = nll, logdetD, logdetM, quad.
// G: lower (ld x ld) Gram with rows/cols [0,m) overwritten by L_M; row ycol holds G_Wr, G_rr.
__global__ void __launch_bounds__(1024) finish_kernel(const double* __restrict__ G, int ld, int m, int ycol,
                                                      const double* __restrict__ LinvM, int ldi, double logdetD,
                                                      const double* __restrict__ logdetD_dev, int64_t n,
                                                      double* __restrict__ terms) {
  __shared__ double zsq[32];
  __shared__ double ldm[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double zs = 0.0, ls = 0.0;
  for (int a = warp; a < m; a += 32) {
    double acc = 0.0;
    for (int b = lane; b <= a; b += 32) acc += LinvM[(size_t)a * ldi + b] * G[(size_t)ycol * ld + b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    zs += acc * acc;
    if (lane == 0) ls += 2.0 * log(G[(size_t)a * ld + a]);
  }
  if (lane == 0) {
    zsq[warp] = zs;
    ldm[warp] = ls;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double z2 = 0.0, lm = 0.0;
    for (int w = 0; w < 32; ++w) {
      z2 += zsq[w];
      lm += ldm[w];
    }
    const double lD = logdetD_dev ? *logdetD_dev : logdetD;
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
                            int* fail, int num_sms, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  int blocks_per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, chol_inv_kernel, 256, 0);
  if (e != cudaSuccess) return e;
  if (blocks_per_sm < 1) return cudaErrorLaunchOutOfResources;
  const int nt = (m + TB - 1) / TB;
  int grid = num_sms;
  const int need = nt * (nt + 1) / 2;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  void* args[] = {&A, &m, &lda, &diag_add, &Linv, &ldi, &lim_inv, &fail};
  return cudaLaunchCooperativeKernel((void*)chol_inv_kernel, dim3(grid), dim3(256), args, 0, s);
}

cudaError_t launch_logd_sum(const double* Dpos, int64_t npts, double* partials, int np, double* out,
                            cudaStream_t s) {
  logd_partial_kernel<<<np, 256, 0, s>>>(Dpos, npts, partials);
  sum_partials_kernel<<<1, 32, 0, s>>>(partials, np, out);
  return cudaGetLastError();
}

cudaError_t launch_finish(const double* G, int ld, int m, int ycol, const double* LinvM, int ldi,
                          const double* logdetD_dev, int64_t n, double* terms, cudaStream_t s) {
  finish_kernel<<<1, 1024, 0, s>>>(G, ld, m, ycol, LinvM, ldi, 0.0, logdetD_dev, n, terms);
  return cudaGetLastError();
}

}  // namespace vif
