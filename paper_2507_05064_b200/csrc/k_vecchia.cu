// k_vecchia.cu -- K2 + K3 fused: the batched residual-process Vecchia factor and the
// whitened Woodbury rows w_i, r_i.
//
// One warp per point i, conditioning set S = (N(i)..., i), s = |N(i)| + 1 <= 8 * RB:
//   1. Gram  G_S = U_S U_S^T over k in [0, mk) on the FP64 tensor core: the s rows of U are
//      gathered straight from L2/HBM into registers (16 B per lane per 8 k, NB chunks in flight);
//      lane l carries k = k0 + 2(l%4) + {0,1} of row l/4 of each 8-row block, which is both the A
//      and the B fragment of mma.m8n8k4 (a consistent k permutation on both operands), so only the
//      RB (RB+1)/2 lower 8x8 tiles are issued.
//   2. C_S = K(X_S, X_S) - G_S + sigma^2 I (nugget by index identity, reading c2) into shared memory.
//   3. Right-looking Cholesky of C_S with i last, lane-per-row (rows lane, lane + 32):
//      pivot s-1 is D_i = C_ii - C_iN C_NN^{-1} C_Ni, row s-1 is l = L_NN^{-1} C_Ni (Eq. D_A_Vecchia).
//   4. A_i^T = L_NN^{-T} l by back substitution.
//   5. w_i = (u_i - sum_k A_ik u_{N(i)_k}) / sqrt(D_i) over all ld columns of U_aug; the y column
//      (index mk) of U_aug makes the same pass produce r_i / sqrt(D_i).
// Outputs: W row at the processing position, D at the position (for sum log D), and optionally
// B_out[i] = -A_i (reading c16) and D_out[i].
#include "common.cuh"
#include "kernels.h"

namespace vif {

constexpr int VW = 4;  // warps per block

template <int RB>
__host__ __device__ constexpr int vecchia_warp_doubles() {
  return RB * 8 * (RB * 8 + 1) + RB * 8;  // C (SP x (SP+1)) + coef (SP)
}

template <int FAM, int RB, int NB>
__global__ void __launch_bounds__(VW * 32) vecchia_kernel(
    const double* __restrict__ U, int64_t ldu, int mk, int ld, const double* __restrict__ X,
    const int32_t* __restrict__ nbr, int mv, const int64_t* __restrict__ order, int64_t npts, CovParams p,
    double* __restrict__ W, int64_t ldw, double* __restrict__ Dpos, double* __restrict__ B_out,
    double* __restrict__ D_out, DevStatus* __restrict__ st) {
  constexpr int SP = RB * 8;
  constexpr int CS = SP + 1;
  constexpr int NT = RB * (RB + 1) / 2;
  extern __shared__ __align__(16) double vsm[];
  __shared__ int Sidx_all[VW][SP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* C = vsm + warp * vecchia_warp_doubles<RB>();
  double* coef = C + SP * CS;
  int* Sidx = Sidx_all[warp];
  const int64_t pos = (int64_t)blockIdx.x * VW + warp;
  if (pos >= npts) return;
  const int64_t i = order[pos];

  // ---- conditioning set ----
  const int nb0 = lane < mv ? nbr[i * mv + lane] : -1;
  const int nb1 = lane + 32 < mv ? nbr[i * mv + lane + 32] : -1;
  const int q = __popc(__ballot_sync(0xffffffffu, nb0 >= 0)) + __popc(__ballot_sync(0xffffffffu, nb1 >= 0));
  const int s = q + 1;
  if (lane < SP) Sidx[lane] = lane < q ? nb0 : (lane == q ? (int)i : -1);
  if (lane + 32 < SP) Sidx[lane + 32] = lane + 32 < q ? nb1 : (lane + 32 == q ? (int)i : -1);
  __syncwarp();

  // ---- 1. Gram on DMMA ----
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  const double* rp[RB];
#pragma unroll
  for (int R = 0; R < RB; ++R) {
    const int gi = Sidx[R * 8 + (lane >> 2)];
    rp[R] = gi >= 0 ? U + (int64_t)gi * ldu + 2 * (lane & 3) : nullptr;
  }
  double2 f[NB][RB];
  auto load = [&](int k0) {
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int R = 0; R < RB; ++R) {
        const int k = k0 + b * 8;
        f[b][R] = (rp[R] != nullptr && k < mk) ? __ldg(reinterpret_cast<const double2*>(rp[R] + k))
                                               : make_double2(0.0, 0.0);
      }
  };
  if (mk > 0) load(0);
  for (int k0 = 0; k0 < mk; k0 += 8 * NB) {
    double2 g[NB][RB];
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int R = 0; R < RB; ++R) g[b][R] = f[b][R];
    if (k0 + 8 * NB < mk) load(k0 + 8 * NB);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      int t = 0;
#pragma unroll
      for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
        for (int R2 = 0; R2 <= R1; ++R2, ++t) dmma884(acc[t][0], acc[t][1], g[b][R1].x, g[b][R2].x);
      t = 0;
#pragma unroll
      for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
        for (int R2 = 0; R2 <= R1; ++R2, ++t) dmma884(acc[t][0], acc[t][1], g[b][R1].y, g[b][R2].y);
    }
  }

  // ---- 2. residual covariance block into shared memory (lower part) ----
  {
    int t = 0;
#pragma unroll
    for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
      for (int R2 = 0; R2 <= R1; ++R2, ++t) {
        const int r = R1 * 8 + (lane >> 2);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int c = R2 * 8 + 2 * (lane & 3) + j;
          if (c <= r) {
            double v;
            if (r < s) {
              const int gr = Sidx[r], gc = Sidx[c];
              v = cov<FAM>(X + (int64_t)gr * p.d, X + (int64_t)gc * p.d, p) - acc[t][j];
              if (r == c) v += p.nugget;
            } else {
              v = r == c ? 1.0 : 0.0;
            }
            C[r * CS + c] = v;
          }
        }
      }
  }
  __syncwarp();

  // ---- 3. Cholesky of C_S (i last) ----
  bool ok = true;
  double Di = 0.0;
  for (int j = 0; j < s; ++j) {
    const double djj = C[j * CS + j];
    if (!(djj > 0.0)) {
      ok = false;
      break;
    }
    Di = djj;
    const double ljj = sqrt(djj);
    __syncwarp();
    for (int r = lane; r < s; r += 32)
      if (r > j) C[r * CS + j] /= ljj;
    if (lane == 0) C[j * CS + j] = ljj;
    __syncwarp();
    for (int r = lane; r < s; r += 32)
      if (r > j) {
        const double lrj = C[r * CS + j];
        for (int c = j + 1; c <= r; ++c) C[r * CS + c] -= lrj * C[c * CS + j];
      }
    __syncwarp();
  }
  if (!ok) {
    if (lane == 0) atomicMin(&st->bad_row, (unsigned long long)i);
    for (int c = 2 * lane; c < ld; c += 64) *reinterpret_cast<double2*>(W + pos * ldw + c) = make_double2(0.0, 0.0);
    if (lane == 0) {
      Dpos[pos] = 1.0;
      if (D_out) D_out[i] = __longlong_as_double(0x7ff8000000000000LL);
    }
    return;
  }

  // ---- 4. A_i^T = L_NN^{-T} l,  l = row s-1 of L ----
  {
    double a0 = lane < q ? C[q * CS + lane] : 0.0;
    double a1 = lane + 32 < q ? C[q * CS + lane + 32] : 0.0;
    for (int j = q - 1; j >= 0; --j) {
      if (lane == (j & 31)) {
        const double x = (j < 32 ? a0 : a1) / C[j * CS + j];
        coef[j] = x;
      }
      __syncwarp();
      const double xj = coef[j];
      if (lane < j) a0 -= C[j * CS + lane] * xj;
      if (lane + 32 < j) a1 -= C[j * CS + lane + 32] * xj;
    }
    __syncwarp();
  }

  // ---- 5. w_i, r_i:  (u_i - sum_k A_ik u_{N_k}) / sqrt(D_i) over ld columns ----
  const double rs = 1.0 / sqrt(Di);
  const double* ui = U + i * ldu;
  for (int c = 2 * lane; c < ld; c += 64) {
    double2 o = __ldg(reinterpret_cast<const double2*>(ui + c));
    int k = 0;
    for (; k + 4 <= q; k += 4) {
      double2 u[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) u[t] = __ldg(reinterpret_cast<const double2*>(U + (int64_t)Sidx[k + t] * ldu + c));
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double x = coef[k + t];
        o.x = fma(-x, u[t].x, o.x);
        o.y = fma(-x, u[t].y, o.y);
      }
    }
    for (; k < q; ++k) {
      const double2 u = __ldg(reinterpret_cast<const double2*>(U + (int64_t)Sidx[k] * ldu + c));
      const double x = coef[k];
      o.x = fma(-x, u.x, o.x);
      o.y = fma(-x, u.y, o.y);
    }
    o.x *= rs;
    o.y *= rs;
    *reinterpret_cast<double2*>(W + pos * ldw + c) = o;
  }
  if (B_out)
    for (int k = lane; k < mv; k += 32) B_out[i * mv + k] = k < q ? -coef[k] : 0.0;
  if (lane == 0) {
    Dpos[pos] = Di;
    if (D_out) D_out[i] = Di;
  }
}

template <int FAM, int RB>
static cudaError_t launch_rb(const VecchiaArgs& a, cudaStream_t s) {
  constexpr int NB = RB <= 4 ? 2 : 1;
  const size_t smem = (size_t)VW * vecchia_warp_doubles<RB>() * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(vecchia_kernel<FAM, RB, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const unsigned blocks = (unsigned)((a.npts + VW - 1) / VW);
  vecchia_kernel<FAM, RB, NB><<<blocks, VW * 32, smem, s>>>(a.U, a.ldu, a.mk, a.ld, a.X, a.nbr, a.mv, a.order,
                                                            a.npts, a.p, a.W, a.ldw, a.Dpos, a.B_out, a.D_out,
                                                            a.st);
  return cudaGetLastError();
}

template <int FAM>
static cudaError_t launch_fam(const VecchiaArgs& a, cudaStream_t s) {
  const int rb = (a.mv + 1 + 7) / 8;
  switch (rb) {
    case 1: return launch_rb<FAM, 1>(a, s);
    case 2: return launch_rb<FAM, 2>(a, s);
    case 3: return launch_rb<FAM, 3>(a, s);
    case 4: return launch_rb<FAM, 4>(a, s);
    case 5: return launch_rb<FAM, 5>(a, s);
    default: return launch_rb<FAM, 6>(a, s);
  }
}

cudaError_t launch_vecchia(const VecchiaArgs& a, cudaStream_t s) {
  if (a.npts == 0) return cudaSuccess;
  switch (a.p.family) {
    case FAM_M12: return launch_fam<FAM_M12>(a, s);
    case FAM_M32: return launch_fam<FAM_M32>(a, s);
    case FAM_M52: return launch_fam<FAM_M52>(a, s);
    default: return launch_fam<FAM_GAUSS>(a, s);
  }
}

}  // namespace vif
