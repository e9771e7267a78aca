// k_grad.cu -- gradient of the VIF Gaussian NLL with respect to
// theta = (sigma_1^2, lambda_1..lambda_d, sigma^2)   (Appendix A).
//
// Differentiating NLL = n/2 log 2pi + 1/2 sum log D_i + NLL_G(G), G = sum_i a_i a_i^T,
// a_i = [w_i, r_i] = sum_k c_ik U_aug[S_k] (c_i = [-A_i, 1] / sqrt(D_i), reading c4):
//   dNLL_G = tr(Q dG) = sum_i g_i . da_i,   g_i = 2 Q a_i,
//   Q = [[ (M_w^{-1} + z z^T)/2, -z/2 ], [ -z^T/2, 1/2 ]],  z = M_w^{-1} G_Wr   (reading g1),
//   da_i = sum_k dc_ik U_aug[S_k] + c_ik dU_aug[S_k],
//   dU = dK(X,Z) L_m^{-T} - U Phi_low^T,  Phi_low = tril(L_m^{-1} dK_m L_m^{-T}), halved diagonal,
//   dc_i from dA_i = C_NN^{-1} (dC_Ni - dC_NN A_i^T), dD_i = dC_ii - 2 A_i.dC_Ni + A_i dC_NN A_i^T,
//   dC_S = dK_SS + [p = nugget] I - (dU_S U_S^T + U_S dU_S^T)           (Appendix A brackets).
// Once: grad_state_kernel (one warp per point): Gram on DMMA and the dots g_i . U_aug[S_k] in one pass
// over the gathered rows, C_S, register Cholesky, A_i, D_i -> a per-point state (L packed, A_i,
// 1/L_jj, dots, D_i).  Per parameter p: dK_m -> Phi (two DMMA GEMMs) -> Phi_low;  dK(X,Z)
// (kx_deriv_kernel) -> dU (two triangular DMMA GEMMs, gemm_tn);  grad_param_kernel: the cross product
// X = dU_S U_S^T (all RB^2 tiles; dG = X + X^T) and the dots g_i . dU_aug[S_k] in one pass, dC_S, then
// with the state dA_i, dD_i (two triangular solves) and the point's contribution
// 1/2 dD_i/D_i + sum_k dc_ik (g_i.U_S_k) + c_ik (g_i.dU_S_k); block partials, fixed-order reduction.
// The nugget's pass has dU = 0 and dC_S = I: no gathers.
#include "common.cuh"
#include "kernels.h"

namespace vif {

namespace {

// dk(a,b)/dtheta_p for p = 0 (sigma_1^2) and p = 1..d (lambda_{p-1}); exact libdevice arithmetic.
// k = sigma_1^2 f(r): dk/dsigma_1^2 = f(r), dk/dlambda_j = sigma_1^2 h(r) Delta_j^2 / lambda_j^3 with
// h = -f'(r)/r: M12 e^{-r}/r, M32 3 e^{-sqrt3 r}, M52 5/3 (1 + sqrt5 r) e^{-sqrt5 r}, Gaussian 2 e^{-r^2}.
template <int FAM>
__device__ __forceinline__ double dcov(const double* __restrict__ a, const double* __restrict__ b, int pidx,
                                       const CovParams& p) {
  double r2 = 0.0;
  for (int k = 0; k < p.d; ++k) {
    const double t = (a[k] - b[k]) * p.inv_ls[k];
    r2 = fma(t, t, r2);
  }
  const double r = sqrt(r2);
  if (pidx == 0) {
    if (FAM == FAM_M12) return exp(-r);
    if (FAM == FAM_M32) return (1.0 + 1.7320508075688772 * r) * exp(-1.7320508075688772 * r);
    if (FAM == FAM_M52) return (1.0 + 2.23606797749979 * r + (5.0 / 3.0) * r2) * exp(-2.23606797749979 * r);
    return exp(-r2);
  }
  double h;
  if (FAM == FAM_M12) h = r > 0.0 ? exp(-r) / r : 0.0;
  else if (FAM == FAM_M32) h = 3.0 * exp(-1.7320508075688772 * r);
  else if (FAM == FAM_M52) h = (5.0 / 3.0) * (1.0 + 2.23606797749979 * r) * exp(-2.23606797749979 * r);
  else h = 2.0 * exp(-r2);
  const int j = pidx - 1;
  const double il = p.inv_ls[j], dj = a[j] - b[j];
  return p.sigma2 * h * dj * dj * il * il * il;
}

// dk/dtheta_p from pre-scaled coordinates (a~ = fam_scale a / lambda) and the exp table (cov_fast):
// with Delta~_j = a~_j - b~_j and E = sigma_1^2 e^{-t}:  dk/dsigma_1^2 = k / sigma_1^2;
// dk/dlambda_j = E Delta~_j^2 / lambda_j x {1/t (M12), 1 (M32), (1+t)/3 (M52), 2 (Gaussian, t = r^2)}.
template <int FAM>
__global__ void dkm_kernel(const double* __restrict__ Z, int m, int mk, int pidx, CovParams p,
                           double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)mk * mk) return;
  const int a = (int)(e / mk), b = (int)(e % mk);
  out[e] = (a < m && b < m) ? dcov<FAM>(Z + (size_t)a * p.d, Z + (size_t)b * p.d, pidx, p) : 0.0;
}

// Phi_low = tril(Phi) with halved diagonal, zero above (so the triangular GEMM may read whole blocks)
__global__ void phi_low_kernel(const double* __restrict__ Phi, int mk, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)mk * mk) return;
  const int a = (int)(e / mk), b = (int)(e % mk);
  out[e] = b < a ? Phi[e] : (b == a ? 0.5 * Phi[e] : 0.0);
}

// zh = Linv g (g = G[ycol][0..m)), Linv lower (ld ldi)
__global__ void zhalf_kernel(const double* __restrict__ Linv, int ldi, const double* __restrict__ G, int ldg,
                             int ycol, int m, double* __restrict__ zh) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  double s = 0.0;
  for (int j = 0; j <= k; ++j) s = fma(Linv[(size_t)k * ldi + j], G[(size_t)ycol * ldg + j], s);
  zh[k] = s;
}

// z = Linv^T zh  (z = M_w^{-1} G_Wr)
__global__ void zfull_kernel(const double* __restrict__ Linv, int ldi, const double* __restrict__ zh, int m,
                             double* __restrict__ z) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  double s = 0.0;
  for (int k = a; k < m; ++k) s = fma(Linv[(size_t)k * ldi + a], zh[k], s);
  z[a] = s;
}

// Q2 = 2 Q (ld x ld): [[M^{-1} + z z^T, -z], [-z^T, 1]] on the W columns [0, m) and the y column;
// M^{-1} = Linv^T Linv
__global__ void q_kernel(const double* __restrict__ Linv, int ldi, const double* __restrict__ z, int m, int ycol,
                         int ld, double* __restrict__ Q2) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)ld * ld) return;
  const int a = (int)(e / ld), b = (int)(e % ld);
  double v = 0.0;
  if (a < m && b < m) {
    const int k0 = a > b ? a : b;
    for (int k = k0; k < m; ++k) v = fma(Linv[(size_t)k * ldi + a], Linv[(size_t)k * ldi + b], v);
    v = fma(z[a], z[b], v);
  } else if (a < m && b == ycol) {
    v = -z[a];
  } else if (a == ycol && b < m) {
    v = -z[b];
  } else if (a == ycol && b == ycol) {
    v = 1.0;
  }
  Q2[e] = v;
}

__global__ void grad_reduce_kernel(const double* __restrict__ part, int64_t nparts, double* __restrict__ out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int64_t k = threadIdx.x; k < nparts; k += blockDim.x) s += part[k];  // fixed assignment and order
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

constexpr int GW = 4;  // warps (points) per block

template <int RB>
__host__ __device__ constexpr int grad_warp_doubles(int d) {
  return 2 * (RB * 8) * (RB * 8 + 1) + 3 * (RB * 8) + RB * 8 * d;  // C, dC (or X), abuf, gam, gamd, xs
}
// per-point state of pass 0, by position: L (packed lower, SP rows incl. the identity padding), A_i,
// 1/L_jj, g_i . U_aug[S_k], D_i, ok
template <int RB>
__host__ __device__ constexpr int state_doubles() {
  return vif_state_doubles<RB>();
}

// per-warp setup shared by both passes: S, its (unscaled) coordinates, row pointers
#define GRAD_WARP_SETUP                                                                          \
  constexpr int SP = RB * 8;                                                                     \
  constexpr int CS = SP + 1;                                                                     \
  extern __shared__ __align__(16) double gsm_[];                                                 \
  __shared__ int Sidx_all[GW][SP];                                                               \
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;                                    \
  double* C = gsm_ + warp * grad_warp_doubles<RB>(p.d);                                          \
  double* dC = C + SP * CS;                                                                      \
  double* abuf = dC + SP * CS;                                                                   \
  double* gam_s = abuf + SP;                                                                     \
  double* gamd_s = gam_s + SP;                                                                   \
  double* xs = gamd_s + SP;                                                                      \
  int* Sidx = Sidx_all[warp];                                                                    \
  const int64_t pos = (int64_t)blockIdx.x * GW + warp;

// ---- pass 0 (once): Gram, g_i dots, C_S, Cholesky, A_i, D_i -> state[pos] ----
template <int FAM, int RB>
__global__ void __launch_bounds__(GW * 32, 4) grad_state_kernel(
    const double* __restrict__ U, const double* __restrict__ Gam, int64_t ldu, int mk, int ld,
    const double* __restrict__ X, const int32_t* __restrict__ nbr, int mv, const int64_t* __restrict__ order,
    int64_t npts, CovParams p, double* __restrict__ state) {
  GRAD_WARP_SETUP
  constexpr int NT = RB * (RB + 1) / 2;
  constexpr int LP = SP * (SP + 1) / 2;
  static_assert(SP <= 32, "gradient kernels need s <= 32");
  __shared__ double tbl[64];
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  __syncthreads();
  if (pos >= npts) return;
  const int64_t i = order[pos];
  const int nb0 = lane < mv ? nbr[i * mv + lane] : -1;
  const int q = __popc(__ballot_sync(0xffffffffu, nb0 >= 0));
  const int s = q + 1;
  const int myidx = lane < q ? nb0 : (lane == q ? (int)i : -1);
  if (lane < SP) Sidx[lane] = myidx;
  if (lane < s)
    for (int k = 0; k < p.d; ++k) xs[lane * p.d + k] = X[(int64_t)myidx * p.d + k] * (fam_scale<FAM>() * p.inv_ls[k]);
  __syncwarp();
  double acc[NT][2], gm[RB];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
  for (int R = 0; R < RB; ++R) gm[R] = 0.0;
  const double* rp[RB];
#pragma unroll
  for (int R = 0; R < RB; ++R) {
    const int gi = Sidx[R * 8 + (lane >> 2)];
    rp[R] = gi >= 0 ? U + (int64_t)gi * ldu + 2 * (lane & 3) : nullptr;
  }
  const double* grow = Gam + pos * (int64_t)ld + 2 * (lane & 3);
  for (int k0 = 0; k0 < ld; k0 += 8) {
    const double2 g2 = __ldg(reinterpret_cast<const double2*>(grow + k0));
    double2 f[RB];
#pragma unroll
    for (int R = 0; R < RB; ++R)
      f[R] = rp[R] ? __ldg(reinterpret_cast<const double2*>(rp[R] + k0)) : make_double2(0.0, 0.0);
#pragma unroll
    for (int R = 0; R < RB; ++R) gm[R] = fma(f[R].x, g2.x, fma(f[R].y, g2.y, gm[R]));
    if (k0 < mk) {
      int t = 0;
#pragma unroll
      for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
        for (int R2 = 0; R2 <= R1; ++R2, ++t) {
          dmma884(acc[t][0], acc[t][1], f[R1].x, f[R2].x);
          dmma884(acc[t][0], acc[t][1], f[R1].y, f[R2].y);
        }
    }
  }
#pragma unroll
  for (int R = 0; R < RB; ++R) {
    gm[R] += __shfl_xor_sync(0xffffffffu, gm[R], 1);
    gm[R] += __shfl_xor_sync(0xffffffffu, gm[R], 2);
    if ((lane & 3) == 0) gam_s[R * 8 + (lane >> 2)] = gm[R];
  }
  {
    int t = 0;
#pragma unroll
    for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
      for (int R2 = 0; R2 <= R1; ++R2, ++t) {
        const int r = R1 * 8 + (lane >> 2), c = R2 * 8 + 2 * (lane & 3);
        C[r * CS + c] = acc[t][0];
        C[r * CS + c + 1] = acc[t][1];
      }
  }
  __syncwarp();
  const int ne = s * (s + 1) / 2;
  for (int e = lane; e < ne; e += 32) {
    int r = (int)((sqrtf_fast(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
    if ((r + 1) * (r + 2) / 2 <= e) ++r;
    if (r * (r + 1) / 2 > e) --r;
    const int c = e - r * (r + 1) / 2;
    double v = cov_fast<FAM>(xs + r * p.d, xs + c * p.d, p.d, tbl) - C[r * CS + c];
    if (r == c) v += p.nugget;
    C[r * CS + c] = v;
  }
  __syncwarp();
  double crow[SP];
#pragma unroll
  for (int c = 0; c < SP; ++c) {
    double v = 0.0;
    if (lane < s) {
      if (c <= lane) v = C[lane * CS + c];
    } else if (c == lane) {
      v = 1.0;
    }
    crow[c] = v;
  }
  bool ok = true;
  double Di = 0.0, myinv = 1.0;
  double* colbuf = abuf;
#pragma unroll
  for (int j = 0; j < SP; ++j) {
    const double djj = __shfl_sync(0xffffffffu, crow[j], j);
    if (j < s) {
      ok = ok && (djj > 0.0);
      if (j == s - 1) Di = djj;
    }
    const double y = rsqrt_nr(djj);
    const double lrj = crow[j] * y;
    crow[j] = lrj;
    if (lane == j) myinv = y;
    if (j + 1 < SP) {
      __syncwarp();
      if (lane < SP) colbuf[lane] = lrj;
      __syncwarp();
#pragma unroll
      for (int c = j + 1; c < SP; ++c) crow[c] = fma(-lrj, colbuf[c], crow[c]);
    }
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < SP; ++c)
    if (lane < SP) C[lane * CS + c] = crow[c];
  __syncwarp();
  double a = lane < q ? C[q * CS + lane] : 0.0;
  for (int j = q - 1; j >= 0; --j) {
    const double xj = __shfl_sync(0xffffffffu, a * myinv, j);
    if (lane == j) a = xj;
    else if (lane < j) a = fma(-C[j * CS + lane], xj, a);
  }
  if (lane >= q) a = 0.0;
  double* st = state + pos * (int64_t)state_doubles<RB>();
  // L rows (packed lower), lane r writes row r
  if (lane < SP) {
    double* row = st + lane * (lane + 1) / 2;
#pragma unroll
    for (int c = 0; c < SP; ++c)
      if (c <= lane) row[c] = crow[c];
    st[LP + lane] = a;
    st[LP + SP + lane] = myinv;
    st[LP + 2 * SP + lane] = gam_s[lane];
  }
  if (lane == 0) {
    st[LP + 3 * SP] = Di;
    st[LP + 3 * SP + 1] = ok ? 1.0 : 0.0;
  }
}

// S of point i: q valid neighbours (a prefix of its row, m_v <= 48: two loads per lane), then i itself
__device__ __forceinline__ int grad_load_S(const int32_t* __restrict__ nbr, int mv, int64_t i, int lane, int SP,
                                           int* __restrict__ Sidx) {
  const int v0 = lane < mv ? nbr[i * mv + lane] : -1;
  const int v1 = lane + 32 < mv ? nbr[i * mv + lane + 32] : -1;
  const int q = __popc(__ballot_sync(0xffffffffu, v0 >= 0)) + __popc(__ballot_sync(0xffffffffu, v1 >= 0));
  for (int t = lane; t < SP; t += 32) {
    const int v = t < 32 ? v0 : v1;
    Sidx[t] = t < q ? v : (t == q ? (int)i : -1);
  }
  return q;
}

// ---- pass 0 for s > 32 (m_v <= 47): the same Gram / dots on DMMA, the Cholesky of C_S in shared
// memory (right-looking, the warp over the trailing triangle), A_i by substitution with dot products
// over the lanes; the same state layout (padding rows of L are identity rows) ----
template <int RB>
__host__ __device__ constexpr int big_warp_doubles(int d) {
  return (RB * 8) * (RB * 8 + 1) + 3 * (RB * 8) + RB * 8 * d;  // C, gam, inv, a, xs
}

template <int FAM, int RB>
__global__ void __launch_bounds__(GW * 32) grad_state_big_kernel(
    const double* __restrict__ U, const double* __restrict__ Gam, int64_t ldu, int mk, int ld,
    const double* __restrict__ X, const int32_t* __restrict__ nbr, int mv, const int64_t* __restrict__ order,
    int64_t npts, CovParams p, double* __restrict__ state) {
  constexpr int SP = RB * 8;
  constexpr int CS = SP + 1;
  constexpr int NT = RB * (RB + 1) / 2;
  constexpr int LP = SP * (SP + 1) / 2;
  extern __shared__ __align__(16) double gsm_[];
  __shared__ int Sidx_all[GW][SP];
  __shared__ double tbl[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* C = gsm_ + warp * big_warp_doubles<RB>(p.d);
  double* gam_s = C + SP * CS;
  double* inv_s = gam_s + SP;
  double* a_s = inv_s + SP;
  double* xs = a_s + SP;
  int* Sidx = Sidx_all[warp];
  const int64_t pos = (int64_t)blockIdx.x * GW + warp;
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  __syncthreads();
  if (pos >= npts) return;
  const int64_t i = order[pos];
  const int q = grad_load_S(nbr, mv, i, lane, SP, Sidx);
  const int s = q + 1;
  __syncwarp();
  for (int t = lane; t < s; t += 32)
    for (int k = 0; k < p.d; ++k) xs[t * p.d + k] = X[(int64_t)Sidx[t] * p.d + k] * (fam_scale<FAM>() * p.inv_ls[k]);
  // Gram (lower tiles) and the dots g_i . U_aug[S_k] (as grad_state_kernel)
  double acc[NT][2], gm[RB];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
  for (int R = 0; R < RB; ++R) gm[R] = 0.0;
  const double* rp[RB];
#pragma unroll
  for (int R = 0; R < RB; ++R) {
    const int gi = Sidx[R * 8 + (lane >> 2)];
    rp[R] = gi >= 0 ? U + (int64_t)gi * ldu + 2 * (lane & 3) : nullptr;
  }
  const double* grow = Gam + pos * (int64_t)ld + 2 * (lane & 3);
  for (int k0 = 0; k0 < ld; k0 += 8) {
    const double2 g2 = __ldg(reinterpret_cast<const double2*>(grow + k0));
    double2 f[RB];
#pragma unroll
    for (int R = 0; R < RB; ++R)
      f[R] = rp[R] ? __ldg(reinterpret_cast<const double2*>(rp[R] + k0)) : make_double2(0.0, 0.0);
#pragma unroll
    for (int R = 0; R < RB; ++R) gm[R] = fma(f[R].x, g2.x, fma(f[R].y, g2.y, gm[R]));
    if (k0 < mk) {
      int t = 0;
#pragma unroll
      for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
        for (int R2 = 0; R2 <= R1; ++R2, ++t) {
          dmma884(acc[t][0], acc[t][1], f[R1].x, f[R2].x);
          dmma884(acc[t][0], acc[t][1], f[R1].y, f[R2].y);
        }
    }
  }
#pragma unroll
  for (int R = 0; R < RB; ++R) {
    gm[R] += __shfl_xor_sync(0xffffffffu, gm[R], 1);
    gm[R] += __shfl_xor_sync(0xffffffffu, gm[R], 2);
    if ((lane & 3) == 0) gam_s[R * 8 + (lane >> 2)] = gm[R];
  }
  {
    int t = 0;
#pragma unroll
    for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
      for (int R2 = 0; R2 <= R1; ++R2, ++t) {
        const int r = R1 * 8 + (lane >> 2), c = R2 * 8 + 2 * (lane & 3);
        C[r * CS + c] = acc[t][0];
        C[r * CS + c + 1] = acc[t][1];
      }
  }
  __syncwarp();
  const int ne = s * (s + 1) / 2;
  for (int e = lane; e < ne; e += 32) {
    int r = (int)((sqrtf_fast(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
    if ((r + 1) * (r + 2) / 2 <= e) ++r;
    if (r * (r + 1) / 2 > e) --r;
    const int c = e - r * (r + 1) / 2;
    double v = cov_fast<FAM>(xs + r * p.d, xs + c * p.d, p.d, tbl) - C[r * CS + c];
    if (r == c) v += p.nugget;
    C[r * CS + c] = v;
  }
  __syncwarp();
  // right-looking Cholesky of the s x s lower triangle
  bool ok = true;
  double Di = 0.0;
  for (int j = 0; j < s; ++j) {
    const double djj = C[j * CS + j];
    ok = ok && (djj > 0.0);
    if (j == s - 1) Di = djj;
    const double y = rsqrt_nr(djj);
    for (int r = j + 1 + lane; r < s; r += 32) C[r * CS + j] *= y;
    __syncwarp();
    if (lane == 0) {
      C[j * CS + j] = djj * y;
      inv_s[j] = y;
    }
    const int w = s - j - 1;  // trailing triangle of order w
    const int nt = w * (w + 1) / 2;
    for (int e = lane; e < nt; e += 32) {
      int r = (int)((sqrtf_fast(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
      if ((r + 1) * (r + 2) / 2 <= e) ++r;
      if (r * (r + 1) / 2 > e) --r;
      const int c = e - r * (r + 1) / 2;
      const int rr = j + 1 + r, cc = j + 1 + c;
      C[rr * CS + cc] = fma(-C[rr * CS + j], C[cc * CS + j], C[rr * CS + cc]);
    }
    __syncwarp();
  }
  // A_i = L_NN^{-T} l, l = row q of L (k < q)
  for (int j = q - 1; j >= 0; --j) {
    double sm = 0.0;
    for (int k = j + 1 + lane; k < q; k += 32) sm = fma(C[k * CS + j], a_s[k], sm);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
    if (lane == 0) a_s[j] = (C[q * CS + j] - sm) * inv_s[j];
    __syncwarp();
  }
  double* st = state + pos * (int64_t)state_doubles<RB>();
  for (int e = lane; e < LP; e += 32) {
    int r = (int)((sqrtf_fast(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
    if ((r + 1) * (r + 2) / 2 <= e) ++r;
    if (r * (r + 1) / 2 > e) --r;
    const int c = e - r * (r + 1) / 2;
    st[e] = r < s ? C[r * CS + c] : (r == c ? 1.0 : 0.0);
  }
  for (int t = lane; t < SP; t += 32) {
    st[LP + t] = t < q ? a_s[t] : 0.0;
    st[LP + SP + t] = t < s ? inv_s[t] : 1.0;
    st[LP + 2 * SP + t] = t < s ? gam_s[t] : 0.0;
  }
  if (lane == 0) {
    st[LP + 3 * SP] = Di;
    st[LP + 3 * SP + 1] = ok ? 1.0 : 0.0;
  }
}

// ---- adjoint form of the per-parameter pass ----
// Every term of a point's contribution is linear in (dC_S, dU_S) with parameter-independent coefficients
// (from L, A_i, D_i, gam of the state).  With a~ = (-A_i, 1) over S = (N(i), i), gam_k = g_i . U_aug[S_k],
// beta~ = (C_NN^{-1} gam_N, 0), Dm = D_i^{-1/2}:
//   dD_i = a~^T dC a~,  dA_i = C_NN^{-1} [dC a~]_N,  so (1/2) dD/D + sum_k dc_k gam_k = tr(M dC) with
//   M = mu a~ a~^T - Dm (beta~ a~^T + a~ beta~^T) / 2,  mu = 1/(2 D) - Dm^3 (a~ . gam) / 2;
//   with dC = dK_S (+ I for the nugget) - (dU_S U_S^T + U_S dU_S^T) and the term Dm a~_k g_i . dU_S_k:
//   contribution = sum_{a,b} w_a a~_b dK_ab + rho . (sum_b a~_b dU_b) + sig . (sum_b beta~_b dU_b),
//   w = mu a~ - Dm beta~,  rho = -2 mu p + Dm (q + g_i),  sig = Dm p,  p = sum_b a~_b U_b,  q = sum_b beta~_b U_b.
// The cross-Gram (s^2 m DMMA work per parameter) becomes two gathered sums (2 s m).
constexpr int ADJ_STRIDE = 56;  // per point: mu, Dm, beta~[0..SP), SP <= 48

template <int RB>
__global__ void __launch_bounds__(GW * 32) grad_adjoint_kernel(const double* __restrict__ U,
                                                                const double* __restrict__ Gam, int64_t ldu, int mk,
                                                                int ld, const int32_t* __restrict__ nbr, int mv,
                                                                const int64_t* __restrict__ order, int64_t npts,
                                                                const double* __restrict__ state,
                                                                double* __restrict__ rho, double* __restrict__ sig,
                                                                double* __restrict__ adj) {
  constexpr int SP = RB * 8;
  constexpr int LP = SP * (SP + 1) / 2;
  __shared__ int Sidx_all[GW][SP];
  __shared__ double at_all[GW][SP], bt_all[GW][SP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pos = (int64_t)blockIdx.x * GW + warp;
  if (pos >= npts) return;
  const int64_t i = order[pos];
  int* Sidx = Sidx_all[warp];
  double* at = at_all[warp];
  double* bt = bt_all[warp];
  const int q = grad_load_S(nbr, mv, i, lane, SP, Sidx);
  const double* st = state + pos * (int64_t)state_doubles<RB>();
  const double Di = st[LP + 3 * SP];
  double ag = 0.0;
  for (int t = lane; t < SP; t += 32) {
    const double atl = t < q ? -st[LP + t] : (t == q ? 1.0 : 0.0);
    at[t] = atl;
    ag = fma(atl, st[LP + 2 * SP + t], ag);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ag += __shfl_xor_sync(0xffffffffu, ag, o);
  const double Dm = rsqrt_nr(Di);
  const double mu = 0.5 / Di - 0.5 * Dm * Dm * Dm * ag;
  // beta = C_NN^{-1} gam_N = L_NN^{-T} L_NN^{-1} gam_N (rows of L packed in the state)
  if constexpr (SP <= 32) {
    const double myinv = lane < SP ? st[LP + SP + lane] : 1.0;
    double y = lane < q ? st[LP + 2 * SP + lane] : 0.0;
    for (int j = 0; j < q; ++j) {
      const double yj = __shfl_sync(0xffffffffu, y * myinv, j);
      if (lane == j) y = yj;
      else if (lane > j && lane < q) y = fma(-st[lane * (lane + 1) / 2 + j], yj, y);
    }
    for (int j = q - 1; j >= 0; --j) {
      const double xj = __shfl_sync(0xffffffffu, y * myinv, j);
      if (lane == j) y = xj;
      else if (lane < j) y = fma(-st[j * (j + 1) / 2 + lane], xj, y);
    }
    if (lane < SP) bt[lane] = lane < q ? y : 0.0;
  } else {
    // s > 32: substitutions one unknown at a time, the dot products over the lanes
    for (int t = lane; t < SP; t += 32) bt[t] = 0.0;
    __syncwarp();
    for (int j = 0; j < q; ++j) {
      double sm = 0.0;
      for (int k = lane; k < j; k += 32) sm = fma(st[j * (j + 1) / 2 + k], bt[k], sm);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
      if (lane == 0) bt[j] = (st[LP + 2 * SP + j] - sm) * st[LP + SP + j];
      __syncwarp();
    }
    for (int j = q - 1; j >= 0; --j) {
      double sm = 0.0;
      for (int k = j + 1 + lane; k < q; k += 32) sm = fma(st[k * (k + 1) / 2 + j], bt[k], sm);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
      if (lane == 0) bt[j] = (bt[j] - sm) * st[LP + SP + j];
      __syncwarp();
    }
  }
  __syncwarp();
  double* ad = adj + pos * (int64_t)ADJ_STRIDE;
  for (int t = lane; t < SP; t += 32) ad[2 + t] = bt[t];
  if (lane == 0) {
    ad[0] = mu;
    ad[1] = Dm;
  }
  const int s = q + 1;
  const double* grow = Gam + pos * (int64_t)ld;
  double* rrow = rho + pos * (int64_t)mk;
  double* srow = sig + pos * (int64_t)mk;
  for (int k = lane; k < mk; k += 32) {
    double pk = 0.0, qk = 0.0;
    for (int b = 0; b < s; ++b) {
      const double u = __ldg(U + (int64_t)Sidx[b] * ldu + k);
      pk = fma(at[b], u, pk);
      qk = fma(bt[b], u, qk);
    }
    rrow[k] = fma(-2.0 * mu, pk, Dm * (qk + __ldg(grow + k)));
    srow[k] = Dm * pk;
  }
}

// The same point terms for EVERY parameter in one pass (the default; no dU): per pair (r, c) of the lower
// triangle the distance, the table exponential (cov_fast's) and the family factor are formed once and feed the
// derivatives dk/dsigma_1^2 = k / sigma_1^2, dk/dlambda_j = E Delta~_j^2 / lambda_j x {1/t, 1, (1+t)/3, 2}
// (Matern 1/2, 3/2, 5/2, Gaussian) and dk/dsigma^2 = I (one pass per parameter before round 2: the sums are
// bit-identical, the pass 3x cheaper).  part[pi * nblocks + block]: block partials.
template <int FAM, int RB>
__global__ void __launch_bounds__(GW * 32) grad_param_adj_all_kernel(
    const double* __restrict__ X, const int32_t* __restrict__ nbr, int mv, const int64_t* __restrict__ order,
    int64_t npts, CovParams p, const double* __restrict__ state, const double* __restrict__ adj,
    double* __restrict__ part, int64_t nblocks) {
  constexpr int SP = RB * 8;
  constexpr int LP = SP * (SP + 1) / 2;
  constexpr int NPM = VIF_MAX_D + 2;
  __shared__ int Sidx_all[GW][SP];
  __shared__ double at_all[GW][SP], w_all[GW][SP];
  __shared__ double xs_all[GW][SP * VIF_MAX_D];
  __shared__ double wsum[GW][NPM];
  __shared__ double tbl[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pos = (int64_t)blockIdx.x * GW + warp;
  const int d = p.d;
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  __syncthreads();
  double acc[NPM];
#pragma unroll
  for (int k = 0; k < NPM; ++k) acc[k] = 0.0;
  bool ok = true;
  if (pos < npts) {
    const int64_t i = order[pos];
    int* Sidx = Sidx_all[warp];
    double* at = at_all[warp];
    double* wv = w_all[warp];
    double* xs = xs_all[warp];
    const int q = grad_load_S(nbr, mv, i, lane, SP, Sidx);
    const int s = q + 1;
    __syncwarp();
    for (int t = lane; t < s; t += 32)
      for (int k = 0; k < d; ++k) xs[t * d + k] = X[(int64_t)Sidx[t] * d + k] * (fam_scale<FAM>() * p.inv_ls[k]);
    const double* st = state + pos * (int64_t)state_doubles<RB>();
    ok = st[LP + 3 * SP + 1] != 0.0;
    const double* ad = adj + pos * (int64_t)ADJ_STRIDE;
    const double mu = ad[0], Dm = ad[1];
    for (int t = lane; t < SP; t += 32) {
      const double atl = t < q ? -st[LP + t] : (t == q ? 1.0 : 0.0);
      at[t] = atl;
      wv[t] = fma(mu, atl, -Dm * ad[2 + t]);
    }
    __syncwarp();
    const int ne = s * (s + 1) / 2;
    for (int e = lane; e < ne; e += 32) {
      int r = (int)((sqrtf_fast(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
      if ((r + 1) * (r + 2) / 2 <= e) ++r;
      if (r * (r + 1) / 2 > e) --r;
      const int c = e - r * (r + 1) / 2;
      const double coef = r == c ? wv[r] * at[r] : fma(wv[r], at[c], wv[c] * at[r]);
      const double* xa = xs + r * d;
      const double* xb = xs + c * d;
      double t2 = 0.0;
      for (int k = 0; k < d; ++k) {
        const double dk = xa[k] - xb[k];
        t2 = fma(dk, dk, t2);
      }
      const double t = FAM == FAM_GAUSS ? t2 : sqrt_fast(t2);
      const double E = sig2_exp_neg(t, tbl);
      const double f = FAM == FAM_M12 || FAM == FAM_GAUSS ? E : (FAM == FAM_M32 ? fma(E, t, E) : fma(E, fma(t2, 1.0 / 3.0, t), E));
      acc[0] = fma(coef, f / p.sigma2, acc[0]);
#pragma unroll
      for (int j = 0; j < VIF_MAX_D; ++j) {
        if (j < d) {
          const double dj = xa[j] - xb[j];
          const double g = E * dj * dj * p.inv_ls[j];
          double dkj;
          if (FAM == FAM_M12) dkj = t > 0.0 ? g / t : 0.0;
          else if (FAM == FAM_M32) dkj = g;
          else if (FAM == FAM_M52) dkj = fma(g, t, g) * (1.0 / 3.0);
          else dkj = 2.0 * g;
          acc[1 + j] = fma(coef, dkj, acc[1 + j]);
        }
      }
      acc[NPM - 1] = fma(coef, r == c ? 1.0 : 0.0, acc[NPM - 1]);  // nugget: dK = I
    }
  }
#pragma unroll
  for (int k = 0; k < NPM; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    acc[k] = ok ? v : __longlong_as_double(0x7ff8000000000000LL);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NPM; ++k) wsum[warp][k] = acc[k];
  }
  __syncthreads();
  const int np = d + 2;
  if ((int)threadIdx.x < np) {
    const int k = (int)threadIdx.x == np - 1 ? NPM - 1 : (int)threadIdx.x;  // the nugget sits in the last slot
    double sum = 0.0;
    for (int w = 0; w < GW; ++w) sum += wsum[w][k];
    part[(int64_t)threadIdx.x * nblocks + blockIdx.x] = sum;
  }
}

template <int FAM, int RB>
cudaError_t launch_param_adj_all_rb(const GradPointArgs& a, cudaStream_t s) {
  const unsigned blocks = (unsigned)((a.npts + GW - 1) / GW);
  grad_param_adj_all_kernel<FAM, RB><<<blocks, GW * 32, 0, s>>>(a.X, a.nbr, a.mv, a.order, a.npts, a.p, a.state,
                                                                a.adj, a.part, (int64_t)blocks);
  return cudaGetLastError();
}

template <int FAM>
cudaError_t launch_param_adj_all_fam(const GradPointArgs& a, cudaStream_t s) {
  switch ((a.mv + 1 + 7) / 8) {
    case 1: return launch_param_adj_all_rb<FAM, 1>(a, s);
    case 2: return launch_param_adj_all_rb<FAM, 2>(a, s);
    case 3: return launch_param_adj_all_rb<FAM, 3>(a, s);
    case 4: return launch_param_adj_all_rb<FAM, 4>(a, s);
    case 5: return launch_param_adj_all_rb<FAM, 5>(a, s);
    default: return launch_param_adj_all_rb<FAM, 6>(a, s);
  }
}

template <int RB>
cudaError_t launch_adj_rb(const GradPointArgs& a, cudaStream_t s) {
  const unsigned blocks = (unsigned)((a.npts + GW - 1) / GW);
  grad_adjoint_kernel<RB><<<blocks, GW * 32, 0, s>>>(a.U, a.Gam, a.ldu, a.mk, a.ld, a.nbr, a.mv, a.order, a.npts,
                                                     a.state, a.rho, a.sig, a.adj);
  return cudaGetLastError();
}

// ---- no dU at all: <R, dU> = <R L_m^{-1}, dK(X,Z)> - <R^T U, Phi_low>, R = sum over the points of the
// adjoint rows scattered to their conditioning sets (a deterministic gather over children lists) ----
// children of point j: entries e = pos * 64 + b with S_{order[pos]}[b] = j (b = q: the point itself)
__global__ void gchild_count_kernel(const int32_t* __restrict__ nbr, int mv, const int64_t* __restrict__ order,
                                    int64_t npts, int* __restrict__ cnt) {
  for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < npts; pos += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = order[pos];
    for (int b = 0; b < mv; ++b) {
      const int j = nbr[i * mv + b];
      if (j < 0) break;
      atomicAdd(cnt + j, 1);
    }
    atomicAdd(cnt + i, 1);
  }
}

__global__ void gchild_fill_kernel(const int32_t* __restrict__ nbr, int mv, const int64_t* __restrict__ order,
                                   int64_t npts, const int* __restrict__ ptr, int* __restrict__ cursor,
                                   int* __restrict__ ent) {
  for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < npts; pos += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = order[pos];
    int b = 0;
    for (; b < mv; ++b) {
      const int j = nbr[i * mv + b];
      if (j < 0) break;
      ent[ptr[j] + atomicAdd(cursor + j, 1)] = (int)(pos * 64 + b);
    }
    ent[ptr[i] + atomicAdd(cursor + i, 1)] = (int)(pos * 64 + b);
  }
}

__global__ void __launch_bounds__(1024) gchild_scan_kernel(const int* __restrict__ cnt, int64_t n, int* __restrict__ ptr) {
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

// sort each children list (deterministic order): a warp per list, every element's rank = the number of
// smaller entries (entries are distinct), elements scattered to their ranks through the second buffer
__global__ void gchild_sort_kernel(int64_t n, const int* __restrict__ ptr, const int* __restrict__ ent_in,
                                   int* __restrict__ ent_out) {
  const int lane = threadIdx.x & 31;
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); j < n;
       j += (int64_t)gridDim.x * (blockDim.x / 32)) {
    const int a = ptr[j], b = ptr[j + 1];
    for (int k = a + lane; k < b; k += 32) {
      const int v = ent_in[k];
      int r = 0;
      for (int q = a; q < b; ++q) r += ent_in[q] < v;
      ent_out[a + r] = v;
    }
  }
}

// R[j][k] = sum_{entries (pos, b) of j} a~_{pos,b} rho[pos][k] + beta~_{pos,b} sig[pos][k]; warp per j,
// j in index order (jorder: an optional visiting order)
// CPL as a template parameter: nvcc then issues all 2 CPL row loads of an entry before its FMAs (140
// registers, one 8-warp block per SM: 148 vs 159 ms per gradient at config 3 against 72 registers and
// 24 warps with the loads interleaved; 64-register / 4-block variants 151-152 ms)
template <int RB, int CPL = 16, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) gR_kernel(const int* __restrict__ ptr, const int* __restrict__ ent,
                                                 const int64_t* __restrict__ order, const int64_t* __restrict__ jorder,
                                                 int64_t n, int mk, const double* __restrict__ state,
                                                 const double* __restrict__ adj, const double* __restrict__ rho,
                                                 const double* __restrict__ sig, double* __restrict__ R,
                                                 unsigned long long* __restrict__ next) {
  constexpr int SP = RB * 8;
  constexpr int LP = SP * (SP + 1) / 2;
  // 16 columns per lane per pass (mk <= 512: one pass); the entries' metadata (position, a~, beta~) is
  // loaded by the lanes in parallel, 32 entries at a time, and broadcast by shuffles, so the row loads
  // of consecutive entries carry no dependent-load chain
  const int lane = threadIdx.x & 31;
  // rows are handed out by a counter (not grid-strided): warps with long children lists would otherwise
  // drift apart and the window of rows in flight -- whose adjoint rows should stay in L2 -- would spread
  for (;;) {
    unsigned long long tt = 0;
    if (lane == 0) tt = atomicAdd(next, 1ull);
    const int64_t t = (int64_t)__shfl_sync(0xffffffffu, tt, 0);
    if (t >= n) break;
    const int64_t j = jorder ? jorder[t] : t;
    const int a = ptr[j], b = ptr[j + 1];
    for (int k0 = 0; k0 < mk; k0 += 32 * CPL) {
      double acc[CPL];
#pragma unroll
      for (int u = 0; u < CPL; ++u) acc[u] = 0.0;
      for (int e0 = a; e0 < b; e0 += 32) {
        int64_t mypos = 0;
        double myal = 0.0, mybe = 0.0;
        if (e0 + lane < b) {
          const int en = ent[e0 + lane];
          mypos = en >> 6;
          const int bb = en & 63;
          const bool self = order[mypos] == j;
          myal = self ? 1.0 : -state[mypos * (int64_t)state_doubles<RB>() + LP + bb];
          mybe = self ? 0.0 : adj[mypos * (int64_t)ADJ_STRIDE + 2 + bb];
        }
        const int ne = min(32, b - e0);
        for (int q = 0; q < ne; ++q) {
          const int64_t pos = __shfl_sync(0xffffffffu, mypos, q);
          const double al = __shfl_sync(0xffffffffu, myal, q);
          const double be = __shfl_sync(0xffffffffu, mybe, q);
          const double* rr = rho + pos * (int64_t)mk + k0 + lane;
          const double* ss = sig + pos * (int64_t)mk + k0 + lane;
          double rv[CPL], sv[CPL];
#pragma unroll
          for (int u = 0; u < CPL; ++u) {
            const bool in = k0 + lane + 32 * u < mk;
            rv[u] = in ? __ldg(rr + 32 * u) : 0.0;
            sv[u] = in ? __ldg(ss + 32 * u) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < CPL; ++u) acc[u] = fma(al, rv[u], fma(be, sv[u], acc[u]));
        }
      }
#pragma unroll
      for (int u = 0; u < CPL; ++u) {
        const int k = k0 + lane + 32 * u;
        if (k < mk) R[j * (int64_t)mk + (mk - 1 - k)] = acc[u];  // columns reversed (see launch_gR)
      }
    }
  }
}

// sum_{p, k < m} T[p][k] dk(x_p, z_k)/dtheta_q for q = 0 (sigma_1^2), 1..d (lambda): one exp per pair,
// block partials part[block][q] (fixed order)
template <int FAM, int D>
__global__ void __launch_bounds__(256) gTdK_kernel(const double* __restrict__ X, const double* __restrict__ Z,
                                                   int64_t n, int m, int mk, CovParams p,
                                                   const double* __restrict__ T, double* __restrict__ part) {
  extern __shared__ double zs[];  // m x d, pre-scaled
  __shared__ double tbl[64];
  __shared__ double red[8][VIF_MAX_D + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int DM = D > 0 ? D : VIF_MAX_D;  // D > 0: compile-time dimension (registers, no local memory)
  const int dd = D > 0 ? D : p.d;
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  for (int e = threadIdx.x; e < m * dd; e += blockDim.x) zs[e] = Z[e] * (fam_scale<FAM>() * p.inv_ls[e % dd]);
  __syncthreads();
  double acc[DM + 1];
#pragma unroll
  for (int q = 0; q <= DM; ++q) acc[q] = 0.0;
  double xr[DM];
  for (int64_t r = (int64_t)blockIdx.x * 8 + warp; r < n; r += (int64_t)gridDim.x * 8) {
#pragma unroll
    for (int k = 0; k < DM; ++k)
      if (k < dd) xr[k] = X[r * dd + k] * (fam_scale<FAM>() * p.inv_ls[k]);
    const double* trow = T + r * (int64_t)mk;
    for (int b = lane; b < m; b += 32) {
      const double t_ = __ldg(trow + (mk - 1 - b));  // T stored with reversed columns
      const double* z = zs + b * dd;
      double t2 = 0.0;
#pragma unroll
      for (int k = 0; k < DM; ++k)
        if (k < dd) {
          const double dk = xr[k] - z[k];
          t2 = fma(dk, dk, t2);
        }
      const double t = FAM == FAM_GAUSS ? t2 : sqrt_fast(t2);
      const double E = sig2_exp_neg(t, tbl);
      const double f = FAM == FAM_M12 || FAM == FAM_GAUSS ? E
                     : (FAM == FAM_M32 ? fma(E, t, E) : fma(E, fma(t2, 1.0 / 3.0, t), E));
      acc[0] = fma(t_, f / p.sigma2, acc[0]);
      // dk/dlambda_j = E Delta~_j^2 / lambda_j x {1/t, 1, (1+t)/3, 2} (as grad_param_adj_all_kernel)
      double g;
      if (FAM == FAM_M12) g = t > 0.0 ? 1.0 / t : 0.0;
      else if (FAM == FAM_M32) g = 1.0;
      else if (FAM == FAM_M52) g = (1.0 + t) * (1.0 / 3.0);
      else g = 2.0;
      const double Eg = E * g * t_;
#pragma unroll
      for (int k = 0; k < DM; ++k)
        if (k < dd) {
          const double dk = xr[k] - z[k];
          acc[1 + k] = fma(Eg * dk * dk, p.inv_ls[k], acc[1 + k]);
        }
    }
  }
#pragma unroll
  for (int q = 0; q <= DM; ++q) {
    if (q > dd) break;
    double v = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x <= p.d) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
    part[(size_t)blockIdx.x * (p.d + 1) + threadIdx.x] = v;
  }
}

// Bp[k'][c'] = Linv[mk-1-c'][mk-1-k']: with R's columns reversed, T = R L_m^{-1} becomes a product with a
// lower-triangular right operand (T'[p][k'] = sum_{c' <= k'} R'[p][c'] Bp[k'][c'], T' = T with reversed
// columns), so the triangular GEMM skips half the work
__global__ void grev_linv_kernel(const double* __restrict__ Linv, int mk, double* __restrict__ Bp) {
  const int64_t tot = (int64_t)mk * mk;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int kp = (int)(e / mk), cp = (int)(e % mk);
    Bp[e] = Linv[(int64_t)(mk - 1 - cp) * mk + (mk - 1 - kp)];
  }
}

// out[q] = sum_blocks part[block][q]
__global__ void gTdK_reduce_kernel(const double* __restrict__ part, int nblocks, int nq, double* __restrict__ out) {
  const int q = threadIdx.x;
  if (q >= nq) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += part[(size_t)b * nq + q];
  out[q] = s;
}

// out[pi] += tdk[q] - sum G2 o Phi_low (one block)
__global__ void __launch_bounds__(1024) gfinal_kernel(double* __restrict__ out, const double* __restrict__ tdk, int q,
                                                      const double* __restrict__ G2, const double* __restrict__ Phil,
                                                      int mk) {
  __shared__ double red[1024];
  double s = 0.0;
  const int64_t tot = (int64_t)mk * mk;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    const int64_t c = e / mk, k = e % mk;  // G2 stored with reversed rows (R's reversed columns)
    s = fma(G2[(mk - 1 - c) * mk + k], Phil[e], s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out += tdk[q] - red[0];
}

template <int FAM, int RB>
cudaError_t launch_grad_rb(const GradPointArgs& a, cudaStream_t s) {
  const size_t smem = (size_t)GW * grad_warp_doubles<RB>(a.p.d) * sizeof(double);
  const unsigned blocks = (unsigned)((a.npts + GW - 1) / GW);
  {
    cudaError_t e = smem_optin(grad_state_kernel<FAM, RB>, smem);  // + the kernel's static shared memory
    if (e != cudaSuccess) return e;
  }
  grad_state_kernel<FAM, RB><<<blocks, GW * 32, smem, s>>>(a.U, a.Gam, a.ldu, a.mk, a.ld, a.X, a.nbr, a.mv,
                                                           a.order, a.npts, a.p, a.state);
  return cudaGetLastError();
}

template <int FAM>
cudaError_t launch_grad_fam(const GradPointArgs& a, cudaStream_t s) {
  switch ((a.mv + 1 + 7) / 8) {
    case 1: return launch_grad_rb<FAM, 1>(a, s);
    case 2: return launch_grad_rb<FAM, 2>(a, s);
    case 3: return launch_grad_rb<FAM, 3>(a, s);
    default: return launch_grad_rb<FAM, 4>(a, s);
  }
}

cudaError_t launch_grad_any(const GradPointArgs& a, cudaStream_t s) {
  switch (a.p.family) {
    case FAM_M12: return launch_grad_fam<FAM_M12>(a, s);
    case FAM_M32: return launch_grad_fam<FAM_M32>(a, s);
    case FAM_M52: return launch_grad_fam<FAM_M52>(a, s);
    default: return launch_grad_fam<FAM_GAUSS>(a, s);
  }
}

}  // namespace

// g_i . U_aug[S_k] (k < s) into a state whose L, A_i, 1/L_jj, D_i the factor wrote: warp per point,
// lanes over columns (each load instruction reads 512 contiguous bytes of one row), one partial sum
// per row in registers, then a transposing butterfly (31 shuffles) leaves the sum for row k in lane k
// (s > 32: rows 32.. in a second pass over the columns)
template <int RB>
__global__ void __launch_bounds__(GW * 32) grad_gam_kernel(const double* __restrict__ U, const double* __restrict__ Gam,
                                                          int64_t ldu, int ld, const int32_t* __restrict__ nbr,
                                                          int mv, const int64_t* __restrict__ order, int64_t npts,
                                                          double* __restrict__ state) {
  constexpr int SP = RB * 8;
  constexpr int LP = SP * (SP + 1) / 2;
  constexpr int NH = (SP + 31) / 32;  // halves of 32 rows (s > 32: two passes over the columns)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pos = (int64_t)blockIdx.x * GW + warp;
  if (pos >= npts) return;
  const int64_t i = order[pos];
  const int nb0 = lane < mv ? nbr[i * mv + lane] : -1;
  const int nb1 = lane + 32 < mv ? nbr[i * mv + lane + 32] : -1;
  const int q = __popc(__ballot_sync(0xffffffffu, nb0 >= 0)) + __popc(__ballot_sync(0xffffffffu, nb1 >= 0));
  const double* grow = Gam + pos * (int64_t)ld;
  double* st = state + pos * (int64_t)vif_state_doubles<RB>();
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    constexpr int HR = SP < 32 ? SP : 32;  // rows per half
    const int row = 32 * h + lane;
    const int nb = h == 0 ? nb0 : nb1;
    const int64_t myrow = row < q ? (int64_t)nb : (row == q ? i : 0);  // rows past s: never loaded
    double v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = 0.0;
    for (int c0 = 0; c0 < ld; c0 += 64) {  // warp-uniform trip count (the shuffles below need all lanes)
      const int c = c0 + 2 * lane;
      const bool in = c < ld;
      const double2 g2 = in ? __ldg(reinterpret_cast<const double2*>(grow + c)) : make_double2(0.0, 0.0);
#pragma unroll
      for (int kb = 0; kb < HR; kb += 16) {  // 16 rows' loads in flight per lane
        double2 u[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int64_t r = __shfl_sync(0xffffffffu, myrow, (kb + k) & 31);
          const int kr = 32 * h + kb + k;
          u[k] = (in && kb + k < HR && kr < SP && kr <= q) ? __ldg(reinterpret_cast<const double2*>(U + r * ldu + c))
                                                          : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (kb + k < HR) v[kb + k] = fma(u[k].x, g2.x, fma(u[k].y, g2.y, v[kb + k]));
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int k = 0; k < o; ++k) {
        const double send = upper ? v[k] : v[k + o];
        const double keep = upper ? v[k + o] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    if (row < SP) st[LP + 2 * SP + row] = v[0];
  }
}

cudaError_t launch_grad_gam(const GradPointArgs& a, cudaStream_t s) {
  if (a.npts <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((a.npts + GW - 1) / GW);
  switch ((a.mv + 1 + 7) / 8) {
    case 1: grad_gam_kernel<1><<<blocks, GW * 32, 0, s>>>(a.U, a.Gam, a.ldu, a.ld, a.nbr, a.mv, a.order, a.npts, a.state); break;
    case 2: grad_gam_kernel<2><<<blocks, GW * 32, 0, s>>>(a.U, a.Gam, a.ldu, a.ld, a.nbr, a.mv, a.order, a.npts, a.state); break;
    case 3: grad_gam_kernel<3><<<blocks, GW * 32, 0, s>>>(a.U, a.Gam, a.ldu, a.ld, a.nbr, a.mv, a.order, a.npts, a.state); break;
    case 4: grad_gam_kernel<4><<<blocks, GW * 32, 0, s>>>(a.U, a.Gam, a.ldu, a.ld, a.nbr, a.mv, a.order, a.npts, a.state); break;
    case 5: grad_gam_kernel<5><<<blocks, GW * 32, 0, s>>>(a.U, a.Gam, a.ldu, a.ld, a.nbr, a.mv, a.order, a.npts, a.state); break;
    case 6: grad_gam_kernel<6><<<blocks, GW * 32, 0, s>>>(a.U, a.Gam, a.ldu, a.ld, a.nbr, a.mv, a.order, a.npts, a.state); break;
    default: return cudaErrorInvalidValue;  // m_v <= 47
  }
  return cudaGetLastError();
}

int64_t grad_point_nparts(int64_t npts) { return (npts + GW - 1) / GW; }

size_t grad_state_doubles(int mv) {
  switch ((mv + 1 + 7) / 8) {
    case 1: return state_doubles<1>();
    case 2: return state_doubles<2>();
    case 3: return state_doubles<3>();
    case 4: return state_doubles<4>();
    case 5: return state_doubles<5>();
    default: return state_doubles<6>();
  }
}

template <int FAM, int RB>
cudaError_t launch_state_big_rb(const GradPointArgs& a, cudaStream_t s) {
  const size_t smem = (size_t)GW * big_warp_doubles<RB>(a.p.d) * sizeof(double);
  if (smem > 40 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(grad_state_big_kernel<FAM, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  const unsigned blocks = (unsigned)((a.npts + GW - 1) / GW);
  grad_state_big_kernel<FAM, RB><<<blocks, GW * 32, smem, s>>>(a.U, a.Gam, a.ldu, a.mk, a.ld, a.X, a.nbr, a.mv,
                                                              a.order, a.npts, a.p, a.state);
  return cudaGetLastError();
}

template <int FAM>
cudaError_t launch_state_big_fam(const GradPointArgs& a, cudaStream_t s) {
  return (a.mv + 1 + 7) / 8 == 5 ? launch_state_big_rb<FAM, 5>(a, s) : launch_state_big_rb<FAM, 6>(a, s);
}

cudaError_t launch_grad_state(const GradPointArgs& a, cudaStream_t s) {
  if (a.npts > 0 && a.mv > 31 && a.mv <= 47) {
    switch (a.p.family) {
      case FAM_M12: return launch_state_big_fam<FAM_M12>(a, s);
      case FAM_M32: return launch_state_big_fam<FAM_M32>(a, s);
      case FAM_M52: return launch_state_big_fam<FAM_M52>(a, s);
      default: return launch_state_big_fam<FAM_GAUSS>(a, s);
    }
  }
  if (a.mv > 47) return cudaErrorNotSupported;
  return a.npts > 0 ? launch_grad_any(a, s) : cudaSuccess;
}

size_t grad_adj_doubles() { return ADJ_STRIDE; }

cudaError_t launch_grad_adjoint(const GradPointArgs& a, cudaStream_t s) {
  if (a.mv > 47) return cudaErrorNotSupported;
  if (a.npts == 0) return cudaSuccess;
  switch ((a.mv + 1 + 7) / 8) {
    case 1: return launch_adj_rb<1>(a, s);
    case 2: return launch_adj_rb<2>(a, s);
    case 3: return launch_adj_rb<3>(a, s);
    case 4: return launch_adj_rb<4>(a, s);
    case 5: return launch_adj_rb<5>(a, s);
    default: return launch_adj_rb<6>(a, s);
  }
}

// every parameter's point terms in one pass (no dU): out[0 .. d+1]; a.part holds (d + 2) x grad_point_nparts(npts)
cudaError_t launch_grad_points_adj_all(const GradPointArgs& a, double* out, cudaStream_t s) {
  if (a.mv > 47 || a.dU) return cudaErrorNotSupported;
  const int64_t nb = grad_point_nparts(a.npts);
  if (a.npts > 0) {
    cudaError_t e;
    switch (a.p.family) {
      case FAM_M12: e = launch_param_adj_all_fam<FAM_M12>(a, s); break;
      case FAM_M32: e = launch_param_adj_all_fam<FAM_M32>(a, s); break;
      case FAM_M52: e = launch_param_adj_all_fam<FAM_M52>(a, s); break;
      default: e = launch_param_adj_all_fam<FAM_GAUSS>(a, s); break;
    }
    if (e != cudaSuccess) return e;
  }
  for (int pi = 0; pi < a.p.d + 2; ++pi) grad_reduce_kernel<<<1, 1024, 0, s>>>(a.part + pi * nb, nb, out + pi);
  return cudaGetLastError();
}

cudaError_t launch_gchild(const int32_t* nbr, int mv, const int64_t* order, int64_t npts, int64_t n, int* cnt,
                          int* cursor, int* ptr, int* ent, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(cnt, 0, (size_t)n * sizeof(int), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(cursor, 0, (size_t)n * sizeof(int), s);
  if (e != cudaSuccess) return e;
  const unsigned g1 = (unsigned)((npts + 255) / 256 > 4096 ? 4096 : (npts + 255) / 256 + 1);
  gchild_count_kernel<<<g1, 256, 0, s>>>(nbr, mv, order, npts, cnt);
  gchild_scan_kernel<<<1, 1024, 0, s>>>(cnt, n, ptr);
  gchild_fill_kernel<<<g1, 256, 0, s>>>(nbr, mv, order, npts, ptr, cursor, ent + n * (int64_t)(mv + 1));
  // fill into the scratch half, rank-sort into ent (the caller's ent has room for 2 n (m_v + 1) entries)
  const unsigned g2 = (unsigned)((n + 7) / 8 > 148 * 16 ? 148 * 16 : (n + 7) / 8);
  gchild_sort_kernel<<<g2, 256, 0, s>>>(n, ptr, ent + n * (int64_t)(mv + 1), ent);
  return cudaGetLastError();
}

cudaError_t launch_gR(const int* ptr, const int* ent, const int64_t* order, const int64_t* jorder, int64_t n, int mk,
                      int mv, const double* state, const double* adj, const double* rho, const double* sig, double* R,
                      unsigned long long* next, cudaStream_t s) {
  cudaError_t e0 = cudaMemsetAsync(next, 0, sizeof(unsigned long long), s);
  if (e0 != cudaSuccess) return e0;
  if (mv > 47) return cudaErrorNotSupported;
  // a resident-sized grid: the warps advance through the visiting order together, so the rows they read
  // (the adjoint rows of nearby points) stay within a window that fits L2; VIF_GR_BLOCKS overrides
  static const char* gb_env = getenv("VIF_GR_BLOCKS");
  const int64_t cap = gb_env ? atoll(gb_env) : 148 * 8;
  const unsigned blocks = (unsigned)((n + 7) / 8 > cap ? cap : (n + 7) / 8);
  switch ((mv + 1 + 7) / 8) {
    case 1: gR_kernel<1><<<blocks, 256, 0, s>>>(ptr, ent, order, jorder, n, mk, state, adj, rho, sig, R, next); break;
    case 2: gR_kernel<2><<<blocks, 256, 0, s>>>(ptr, ent, order, jorder, n, mk, state, adj, rho, sig, R, next); break;
    case 3: gR_kernel<3><<<blocks, 256, 0, s>>>(ptr, ent, order, jorder, n, mk, state, adj, rho, sig, R, next); break;
    case 4: gR_kernel<4><<<blocks, 256, 0, s>>>(ptr, ent, order, jorder, n, mk, state, adj, rho, sig, R, next); break;
    case 5: gR_kernel<5><<<blocks, 256, 0, s>>>(ptr, ent, order, jorder, n, mk, state, adj, rho, sig, R, next); break;
    default: gR_kernel<6><<<blocks, 256, 0, s>>>(ptr, ent, order, jorder, n, mk, state, adj, rho, sig, R, next); break;
  }
  return cudaGetLastError();
}

int gTdK_blocks() { return 148 * 4; }

cudaError_t launch_gTdK(const double* X, const double* Z, int64_t n, int m, int mk, const CovParams& p,
                        const double* T, double* part, double* out, cudaStream_t s) {
  const int blocks = gTdK_blocks();
  const size_t zb = (size_t)m * p.d * sizeof(double);
  auto go = [&](auto kern) -> cudaError_t {
    {
      cudaError_t e = smem_optin(kern, zb);  // static shared memory comes on top
      if (e != cudaSuccess) return e;
    }
    kern<<<blocks, 256, zb, s>>>(X, Z, n, m, mk, p, T, part);
    return cudaSuccess;
  };
  cudaError_t e;
  if (p.d == 2) {
    switch (p.family) {
      case FAM_M12: e = go(gTdK_kernel<FAM_M12, 2>); break;
      case FAM_M32: e = go(gTdK_kernel<FAM_M32, 2>); break;
      case FAM_M52: e = go(gTdK_kernel<FAM_M52, 2>); break;
      default: e = go(gTdK_kernel<FAM_GAUSS, 2>); break;
    }
  } else {
    switch (p.family) {
      case FAM_M12: e = go(gTdK_kernel<FAM_M12, 0>); break;
      case FAM_M32: e = go(gTdK_kernel<FAM_M32, 0>); break;
      case FAM_M52: e = go(gTdK_kernel<FAM_M52, 0>); break;
      default: e = go(gTdK_kernel<FAM_GAUSS, 0>); break;
    }
  }
  if (e != cudaSuccess) return e;
  gTdK_reduce_kernel<<<1, 32, 0, s>>>(part, blocks, p.d + 1, out);
  return cudaGetLastError();
}

cudaError_t launch_grev_linv(const double* Linv, int mk, double* Bp, cudaStream_t s) {
  const int64_t tot = (int64_t)mk * mk;
  grev_linv_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(Linv, mk, Bp);
  return cudaGetLastError();
}

cudaError_t launch_gfinal(double* out, const double* tdk, int q, const double* G2, const double* Phil, int mk,
                          cudaStream_t s) {
  gfinal_kernel<<<1, 1024, 0, s>>>(out, tdk, q, G2, Phil, mk);
  return cudaGetLastError();
}

cudaError_t launch_dkm(const double* Z, int m, int mk, int pidx, const CovParams& p, double* out, cudaStream_t s) {
  const int64_t tot = (int64_t)mk * mk;
  const unsigned blocks = (unsigned)((tot + 255) / 256);
  switch (p.family) {
    case FAM_M12: dkm_kernel<FAM_M12><<<blocks, 256, 0, s>>>(Z, m, mk, pidx, p, out); break;
    case FAM_M32: dkm_kernel<FAM_M32><<<blocks, 256, 0, s>>>(Z, m, mk, pidx, p, out); break;
    case FAM_M52: dkm_kernel<FAM_M52><<<blocks, 256, 0, s>>>(Z, m, mk, pidx, p, out); break;
    default: dkm_kernel<FAM_GAUSS><<<blocks, 256, 0, s>>>(Z, m, mk, pidx, p, out); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_phi_low(const double* Phi, int mk, double* out, cudaStream_t s) {
  const int64_t tot = (int64_t)mk * mk;
  phi_low_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(Phi, mk, out);
  return cudaGetLastError();
}

// Prediction (Prop. 1; App. C.1): for the prediction row [w_p, r_p] (computed with y_p = 0,
// w_p = e_p / sqrt(D_p)):  mu_p = sqrt(D_p) (w_p . z - r_p) = u_p . z + A_p (y_N - U_N z),
// var_p = D_p (1 + |T_p|^2), T = W L_M^{-T} (so D_p |T_p|^2 = e_p^T M_w^{-1} e_p).  One warp per point.
__global__ void pred_mean_kernel(const double* __restrict__ Wp, int ld, int m, int ycol, const double* __restrict__ z,
                                 const double* __restrict__ Dpos, const int64_t* __restrict__ order, int64_t np,
                                 double* __restrict__ mu, const double* __restrict__ T, int ldt,
                                 double* __restrict__ var) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pos = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (pos >= np) return;
  const double* w = Wp + pos * (int64_t)ld;
  double s = 0.0, t2 = 0.0;
  for (int a = lane; a < m; a += 32) s = fma(w[a], z[a], s);
  if (T)
    for (int a = lane; a < m; a += 32) {
      const double t = T[pos * (int64_t)ldt + a];
      t2 = fma(t, t, t2);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    t2 += __shfl_xor_sync(0xffffffffu, t2, o);
  }
  if (lane == 0) {
    const double D = Dpos[pos];
    const int64_t i = order[pos];
    mu[i] = sqrt(D) * (s - w[ycol]);
    if (var) var[i] = D * (1.0 + t2);
  }
}

cudaError_t launch_pred_mean(const double* Wp, int ld, int m, int ycol, const double* z, const double* Dpos,
                             const int64_t* order, int64_t np, double* mu, const double* T, int ldt, double* var,
                             cudaStream_t s) {
  if (np == 0) return cudaSuccess;
  pred_mean_kernel<<<(unsigned)((np + 7) / 8), 256, 0, s>>>(Wp, ld, m, ycol, z, Dpos, order, np, mu, T, ldt, var);
  return cudaGetLastError();
}

cudaError_t launch_zvec(const double* LinvM, int ldi, const double* G, int ldg, int ycol, int m, double* zh,
                        double* z, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  zhalf_kernel<<<(m + 127) / 128, 128, 0, s>>>(LinvM, ldi, G, ldg, ycol, m, zh);
  zfull_kernel<<<(m + 127) / 128, 128, 0, s>>>(LinvM, ldi, zh, m, z);
  return cudaGetLastError();
}

cudaError_t launch_grad_q(const double* LinvM, int ldi, const double* G, int ldg, int ycol, int m, int ld,
                          double* zh, double* z, double* Q2, cudaStream_t s) {
  if (m > 0) {
    zhalf_kernel<<<(m + 127) / 128, 128, 0, s>>>(LinvM, ldi, G, ldg, ycol, m, zh);
    zfull_kernel<<<(m + 127) / 128, 128, 0, s>>>(LinvM, ldi, zh, m, z);
  }
  const int64_t tot = (int64_t)ld * ld;
  q_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(LinvM, ldi, z, m, ycol, ld, Q2);
  return cudaGetLastError();
}

}  // namespace vif
