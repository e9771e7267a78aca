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
#pragma once
#include "common.cuh"
#include "kernels.h"
#include <stdlib.h>

namespace vif {

constexpr int VW = 4;  // warps per block

// timing probe only (VIF_DEBUG_VECCHIA env, read at every launch): bit 0 skips the Gram phase,
// bit 1 skips the scalar phases.  Never set in tests or bench.py.
__constant__ int g_vif_debug;

template <int RB>
__host__ __device__ constexpr int vecchia_warp_doubles() {
  return RB * 8 * (RB * 8 + 1) + RB * 8;  // C (SP x (SP+1)) + coef (SP)
}

template <int FAM, int RB, int NB>
__global__ void __launch_bounds__(VW * 32) vecchia_smem_kernel(
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


// ------------------------------------------------------------------------------------------
// Register variant for s <= 32 (RB <= 4): the same five steps with the per-point scalar work
// reorganised so that it does not starve the DMMA pipe of the other resident warps:
//   - the s(s+1)/2 kernel evaluations are spread evenly over the lanes (flat lower-triangle
//     index), with the conditioning-set coordinates staged in shared memory;
//   - the Cholesky keeps row `lane` in registers (compile-time indexed, fully unrolled); column j
//     is broadcast through shared memory (double-buffered), so step j costs one store and
//     SP - j broadcast loads + FMAs per lane;
//   - the back substitution uses a shuffle per step;
//   - the W pass issues all s row loads of a 64-column chunk before the FMAs.
// Gram of the (up to 8*RB) rows rp[] over k in [0, mk): a ring of NBUF 8-k register chunks
// (16 B per lane per row block), refilled right after each chunk's 2 x RB(RB+1)/2 DMMAs -- no
// register copies, so a load that is still in flight never blocks the DMMA stream.
template <int RB, int NBUF>
__device__ __forceinline__ void gram_ring(const double* const (&rp)[RB], int mk, double (&acc)[RB * (RB + 1) / 2][2]) {
  double2 f[NBUF][RB];
#pragma unroll
  for (int c = 0; c < NBUF; ++c)
#pragma unroll
    for (int R = 0; R < RB; ++R)
      f[c][R] = (rp[R] != nullptr && 8 * c < mk) ? __ldg(reinterpret_cast<const double2*>(rp[R] + 8 * c))
                                                 : make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < mk; k0 += 8 * NBUF) {
#pragma unroll
    for (int c = 0; c < NBUF; ++c) {
      if (k0 + 8 * c < mk) {
        int t = 0;
#pragma unroll
        for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
          for (int R2 = 0; R2 <= R1; ++R2, ++t) dmma884(acc[t][0], acc[t][1], f[c][R1].x, f[c][R2].x);
        t = 0;
#pragma unroll
        for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
          for (int R2 = 0; R2 <= R1; ++R2, ++t) dmma884(acc[t][0], acc[t][1], f[c][R1].y, f[c][R2].y);
      }
      const int kn = k0 + 8 * NBUF + 8 * c;
#pragma unroll
      for (int R = 0; R < RB; ++R)
        f[c][R] = (rp[R] != nullptr && kn < mk) ? __ldg(reinterpret_cast<const double2*>(rp[R] + kn))
                                                : make_double2(0.0, 0.0);
    }
  }
}

// The same ring split in two: gram_fill issues the first NBUF chunks, gram_drain runs the DMMA
// loop.  Independent work placed between the two (the kernel evaluations of step 2) hides the
// latency of the first loads of every point.
template <int RB, int NBUF>
__device__ __forceinline__ void gram_fill(const double* const (&rp)[RB], int mk, double2 (&f)[NBUF][RB]) {
#pragma unroll
  for (int c = 0; c < NBUF; ++c)
#pragma unroll
    for (int R = 0; R < RB; ++R)
      f[c][R] = (rp[R] != nullptr && 8 * c < mk) ? __ldg(reinterpret_cast<const double2*>(rp[R] + 8 * c))
                                                 : make_double2(0.0, 0.0);
}
template <int RB, int NBUF>
__device__ __forceinline__ void gram_drain(const double* const (&rp)[RB], int mk, double (&acc)[RB * (RB + 1) / 2][2],
                                           double2 (&f)[NBUF][RB]) {
  for (int k0 = 0; k0 < mk; k0 += 8 * NBUF) {
#pragma unroll
    for (int c = 0; c < NBUF; ++c) {
      if (k0 + 8 * c < mk) {
        int t = 0;
#pragma unroll
        for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
          for (int R2 = 0; R2 <= R1; ++R2, ++t) dmma884(acc[t][0], acc[t][1], f[c][R1].x, f[c][R2].x);
        t = 0;
#pragma unroll
        for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
          for (int R2 = 0; R2 <= R1; ++R2, ++t) dmma884(acc[t][0], acc[t][1], f[c][R1].y, f[c][R2].y);
      }
      const int kn = k0 + 8 * NBUF + 8 * c;
#pragma unroll
      for (int R = 0; R < RB; ++R)
        f[c][R] = (rp[R] != nullptr && kn < mk) ? __ldg(reinterpret_cast<const double2*>(rp[R] + kn))
                                                : make_double2(0.0, 0.0);
    }
  }
}

// flat lower-triangle index e -> (r, c), c <= r
__device__ __forceinline__ void tri_rc(int e, int& r, int& c) {
  int rr = (int)((sqrtf_fast(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  if ((rr + 1) * (rr + 2) / 2 <= e) ++rr;
  if (rr * (rr + 1) / 2 > e) --rr;
  r = rr;
  c = e - rr * (rr + 1) / 2;
}

// K(X_S, X_S) + sigma^2 I on the lower triangle (minus the Gram already in C when SUB): the
// s(s-1)/2 off-diagonal evaluations spread evenly over the lanes, EU independent evaluations in
// flight per lane (each a ~20-deep dependent FP64 chain); the diagonal is sigma1^2 + sigma^2
// (tbl[0] = sigma1^2).  xs: pre-scaled coordinates (cov_fast).
template <int FAM, int EU, int SUB = 0>
__device__ __forceinline__ void eval_lower(const double* __restrict__ xs, int s, int CS, int d, double nugget,
                                           const double* __restrict__ tbl, int lane, double* __restrict__ C) {
  if (lane < s) {
    const double v = tbl[0] + nugget;
    C[lane * CS + lane] = SUB ? v - C[lane * CS + lane] : v;
  }
  const int ne = s * (s - 1) / 2;
  for (int e0 = lane; e0 < ne; e0 += 32 * EU) {
    double v[EU];
    int o[EU];
#pragma unroll
    for (int u = 0; u < EU; ++u) {
      const int e = e0 + 32 * u < ne ? e0 + 32 * u : 0;
      // strictly lower triangle: e -> (r, c), r > c
      int r = (int)((1.0f + sqrtf_fast(8.0f * (float)e + 1.0f)) * 0.5f);
      if (r * (r - 1) / 2 > e) --r;
      if ((r + 1) * r / 2 <= e) ++r;
      const int c = e - r * (r - 1) / 2;
      o[u] = e0 + 32 * u < ne ? r * CS + c : -1;
      v[u] = cov_fast<FAM>(xs + r * d, xs + c * d, d, tbl);
    }
#pragma unroll
    for (int u = 0; u < EU; ++u)
      if (o[u] >= 0) C[o[u]] = SUB ? v[u] - C[o[u]] : v[u];
  }
}

// stage the pre-scaled coordinates of S (lanes < s) for cov_fast
template <int FAM>
__device__ __forceinline__ void stage_xs(const double* __restrict__ X, int idx, int d, const CovParams& p, int lane,
                                         int s, double* __restrict__ xs) {
  if (lane < s)
    for (int k = 0; k < d; ++k) xs[lane * d + k] = X[(int64_t)idx * d + k] * (fam_scale<FAM>() * p.inv_ls[k]);
}

template <int RB>
__host__ __device__ constexpr int vreg_warp_doubles(int d) {
  return RB * 8 * (RB * 8 + 1) + 2 * RB * 8 + RB * 8 + RB * 8 * d;  // C, colbuf[2], coef, xs
}

template <int FAM, int RB, int NB, int MINB>
__global__ void __launch_bounds__(VW * 32, MINB) vecchia_reg_kernel(
    const double* __restrict__ U, int64_t ldu, int mk, int ld, const double* __restrict__ X,
    const int32_t* __restrict__ nbr, int mv, const int64_t* __restrict__ order, int64_t npts, CovParams p,
    double* __restrict__ W, int64_t ldw, double* __restrict__ Dpos, double* __restrict__ B_out,
    double* __restrict__ D_out, DevStatus* __restrict__ st) {
  constexpr int SP = RB * 8;
  constexpr int CS = SP + 1;
  constexpr int NT = RB * (RB + 1) / 2;
  static_assert(SP <= 32, "register variant needs s <= 32");
  extern __shared__ __align__(16) double vsm[];
  __shared__ int Sidx_all[VW][SP];
  __shared__ double tbl[64];
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* C = vsm + warp * vreg_warp_doubles<RB>(p.d);
  double* colbuf = C + SP * CS;   // [2][SP]
  double* coef = colbuf + 2 * SP; // [SP]
  double* xs = coef + SP;         // [SP][d]
  int* Sidx = Sidx_all[warp];
  const int64_t pos = (int64_t)blockIdx.x * VW + warp;
  if (pos >= npts) return;
  const int64_t i = order[pos];

  // ---- conditioning set and its (pre-scaled) coordinates ----
  const int nb0 = lane < mv ? nbr[i * mv + lane] : -1;
  const int q = __popc(__ballot_sync(0xffffffffu, nb0 >= 0));
  const int s = q + 1;
  const int myidx = lane < q ? nb0 : (lane == q ? (int)i : -1);
  if (lane < SP) Sidx[lane] = myidx;
  stage_xs<FAM>(X, myidx, p.d, p, lane, s, xs);
  __syncwarp();

  // ---- 1 + 2. Gram on DMMA; the kernel evaluations of step 2 (independent of the Gram) run
  //      between the ring fill and the DMMA loop, hiding the first loads of every point;
  //      C_S = K + sigma^2 I - G_S when the tiles leave the accumulators ----
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  const double* rp[RB];
#pragma unroll
  for (int R = 0; R < RB; ++R) {
    const int gi = Sidx[R * 8 + (lane >> 2)];
    rp[R] = gi >= 0 ? U + (int64_t)gi * ldu + 2 * (lane & 3) : nullptr;
  }
  {
    double2 f[NB][RB];
    gram_fill<RB, NB>(rp, mk, f);
    eval_lower<FAM, 4>(xs, s, CS, p.d, p.nugget, tbl, lane, C);
    if (!(g_vif_debug & 1)) gram_drain<RB, NB>(rp, mk, acc, f);  // debug probe: bit 0 skips the Gram
    __syncwarp();
    int t = 0;
#pragma unroll
    for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
      for (int R2 = 0; R2 <= R1; ++R2, ++t) {
        const int r = R1 * 8 + (lane >> 2), c = R2 * 8 + 2 * (lane & 3);
        if (r < s) {
          if (c <= r) C[r * CS + c] -= acc[t][0];
          if (c + 1 <= r) C[r * CS + c + 1] -= acc[t][1];
        }
      }
    __syncwarp();
    if (g_vif_debug & 2) {  // debug probe: bit 1 skips steps 3-5 (timing only; outputs invalid)
      if (lane == 0) Dpos[pos] = 1.0 + 1e-30 * C[0];
      return;
    }
  }

  // ---- 3. Cholesky, row `lane` in registers; padded rows (>= s) are identity ----
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
#pragma unroll
  for (int j = 0; j < SP; ++j) {
    const double djj = __shfl_sync(0xffffffffu, crow[j], j);
    if (j < s) {
      ok = ok && (djj > 0.0);
      if (j == s - 1) Di = djj;
    }
    // one inline reciprocal square root per step (no out-of-line div/sqrt subroutines):
    // lane j gets djj / sqrt(djj) = l_jj, lanes below get l_rj = c_rj / l_jj
    const double y = rsqrt_nr(djj);
    const double lrj = crow[j] * y;
    crow[j] = lrj;
    if (lane == j) myinv = y;
    if (j + 1 < SP) {
      double* cb = colbuf + (j & 1) * SP;
      if (lane < SP) cb[lane] = lrj;
      __syncwarp();
#pragma unroll
      for (int c = j + 1; c < SP; ++c) crow[c] = fma(-lrj, cb[c], crow[c]);
    }
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
  // rows of L to shared memory (row-major) for the back substitution
#pragma unroll
  for (int c = 0; c < SP; ++c)
    if (lane < SP) C[lane * CS + c] = crow[c];
  __syncwarp();

  // ---- 4. A_i^T = L_NN^{-T} l, l = row q of L; lane k holds x_k ----
  {
    const double inv_diag = myinv;  // 1 / own diagonal
    double a = lane < q ? C[q * CS + lane] : 0.0;
    for (int j = q - 1; j >= 0; --j) {
      const double xj = __shfl_sync(0xffffffffu, a * inv_diag, j);
      if (lane == j) a = xj;
      else if (lane < j) a = fma(-C[j * CS + lane], xj, a);
    }
    const double rs = rsqrt_nr(Di);
    // coefficients of the W row: -A_ik / sqrt(D) for k < q, 1 / sqrt(D) for i itself, 0 beyond
    if (lane < SP) coef[lane] = lane < q ? -a * rs : (lane == q ? rs : 0.0);
    if (B_out && lane < mv) B_out[i * mv + lane] = lane < q ? -a : 0.0;
  }
  __syncwarp();

  // ---- 5. w_i, r_i over ld columns: 512 columns per pass (8 chunks of 64 per lane-pair),
  //         rows two at a time -> 16 independent 16-byte loads in flight per lane ----
  for (int c0 = 0; c0 < ld; c0 += 512) {
    double2 o[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) o[t] = make_double2(0.0, 0.0);
    for (int k = 0; k < s; k += 2) {
      double2 u0[8], u1[8];
      const double* r0 = U + (int64_t)Sidx[k] * ldu + c0 + 2 * lane;
      const bool has1 = k + 1 < s;
      const double* r1 = has1 ? U + (int64_t)Sidx[k + 1] * ldu + c0 + 2 * lane : r0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const bool in = c0 + 2 * lane + 64 * t < ld;
        u0[t] = in ? __ldg(reinterpret_cast<const double2*>(r0 + 64 * t)) : make_double2(0.0, 0.0);
        u1[t] = (in && has1) ? __ldg(reinterpret_cast<const double2*>(r1 + 64 * t)) : make_double2(0.0, 0.0);
      }
      const double f0 = coef[k], f1 = has1 ? coef[k + 1] : 0.0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        o[t].x = fma(f0, u0[t].x, o[t].x);
        o[t].y = fma(f0, u0[t].y, o[t].y);
        o[t].x = fma(f1, u1[t].x, o[t].x);
        o[t].y = fma(f1, u1[t].y, o[t].y);
      }
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int c = c0 + 2 * lane + 64 * t;
      if (c < ld) *reinterpret_cast<double2*>(W + pos * ldw + c) = o[t];
    }
  }
  if (lane == 0) {
    Dpos[pos] = Di;
    if (D_out) D_out[i] = Di;
  }
}

// ------------------------------------------------------------------------------------------
// Mixed-precision solver variant for s <= 32.
// On B200 the DMMAs of the Gram and every scalar FP64 instruction share one FP64 unit per SMSP,
// and a scalar FP64 instruction of a warp waits behind the DMMAs that other warps keep issuing
// (tools/dmma_mix.cu).  The per-point FP64 Cholesky + back substitution (~800 FP64 warp
// instructions, profiles/r01_notes.md) is therefore replaced by
//   - an FP32 Cholesky of C_NN (FMA pipe; row `lane` in FP32 registers, column broadcast through
//     shared memory), used as a preconditioner, and
//   - A_i = C_NN^{-1} C_Ni by iterative refinement: a_0 = solve32(c), then twice
//     a += solve32(c - C_NN a) with the residual in FP64 (31 DFMA per lane per step),
// which converges to FP64 accuracy in two steps for the condition numbers of the residual
// blocks (contraction ~ kappa * 2^-24; kappa(C_NN) <= (s * (sigma1^2 + sigma^2)) / sigma^2).
// D_i = C_ii - C_iN A_i^T in FP64.  A point whose FP32 factorisation fails (pivot <= 0 or
// non-finite), whose final correction exceeds 1e-8 of |A_i|, or whose D_i <= 0 is redone by the
// plain FP64 Cholesky in shared memory, which alone decides VIF_ERR_NOT_PD (oracle step 3).
// The FP32 factor L32 is stored in the unused upper triangle of C (one float per double slot:
// L32[j][k] at double slot (k, j + 1)).
template <int SP>
__device__ __forceinline__ float tri_fwd32(const float (&cr)[SP], float inv, float v, int lane, int q) {
#pragma unroll
  for (int j = 0; j < SP; ++j) {
    if (j >= q) break;
    const float xj = __shfl_sync(0xffffffffu, v * inv, j);
    if (lane == j) v = xj;
    else if (lane > j) v = fmaf(-cr[j], xj, v);
  }
  return v;
}
template <int SP, int CS>
__device__ __forceinline__ float tri_bwd32(const float* __restrict__ Lf, float inv, float v, int lane, int q) {
  // L^T x = v with L[j][lane] at Lf[2 * (lane * CS + j + 1)]
#pragma unroll
  for (int j = SP - 1; j >= 0; --j) {
    if (j < q) {
      const float lj = lane < j ? Lf[2 * (lane * CS + j + 1)] : 0.0f;
      const float xj = __shfl_sync(0xffffffffu, v * inv, j);
      if (lane == j) v = xj;
      else if (lane < j) v = fmaf(-lj, xj, v);
    }
  }
  return v;
}

__device__ __forceinline__ float rsqrt_f32(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// plain FP64 right-looking Cholesky of C_S (lower triangle of C, lane per row) + back
// substitution: the fallback of the mixed solver.  Returns false on a pivot <= 0.
// On success: coef[k] = A_ik for k < q, and *Di.
template <int CS>
__device__ bool fp64_chol_solve(double* __restrict__ C, double* __restrict__ coef, int s, int q, int lane,
                                double* Di_out) {
  double Di = 0.0;
  for (int j = 0; j < s; ++j) {
    const double djj = C[j * CS + j];
    if (!(djj > 0.0)) return false;
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
  double a0 = lane < q ? C[q * CS + lane] : 0.0;
  for (int j = q - 1; j >= 0; --j) {
    if (lane == j) coef[j] = a0 / C[j * CS + j];
    __syncwarp();
    const double xj = coef[j];
    if (lane < j) a0 -= C[j * CS + lane] * xj;
  }
  __syncwarp();
  *Di_out = Di;
  return true;
}

// Steps 3-4 of the mixed solver (see above).  C: the warp's C_S (lower triangle, stride CS),
// cb32: [2][SP] floats, abuf: [SP] doubles.  Returns ok; on ok, a = A_ik on lane k < q (0 elsewhere)
// and Di.  On !ok the caller runs fp64_chol_solve.
template <int SP>
__device__ __forceinline__ bool mix_solve(double* __restrict__ C, float* __restrict__ cb32, double* __restrict__ abuf,
                                          int q, int lane, double& a, double& Di) {
  constexpr int CS = SP + 1;
  // ---- 3. FP32 Cholesky of C_NN (row `lane`; padded rows identity) ----
  float cr[SP];
#pragma unroll
  for (int c = 0; c < SP; ++c) {
    float v = c == lane ? 1.0f : 0.0f;
    if (lane < q && c <= lane) v = (float)C[lane * CS + c];
    cr[c] = v;
  }
  bool ok = true;
  float inv = 1.0f;
#pragma unroll
  for (int j = 0; j < SP; ++j) {
    if (j >= q) break;
    const float djj = __shfl_sync(0xffffffffu, cr[j], j);
    ok = ok && (djj > 0.0f) && (djj < 3.0e38f);
    const float y = rsqrt_f32(djj);
    const float l = cr[j] * y;
    cr[j] = l;
    if (lane == j) inv = y;
    float* cb = cb32 + (j & 1) * SP;
    if (lane < SP) cb[lane] = l;
    __syncwarp();
#pragma unroll
    for (int c = j + 1; c < SP; ++c) cr[c] = fmaf(-l, cb[c], cr[c]);
  }
  float* Lf = reinterpret_cast<float*>(C);
  a = 0.0;
  Di = 0.0;
  if (ok) {
    // L32 rows into the upper triangle of C: L32[lane][k] at double slot (k, lane + 1)
    if (lane < q) {
#pragma unroll
      for (int k = 0; k < SP; ++k)
        if (k <= lane) Lf[2 * (k * CS + lane + 1)] = cr[k];
    }
    __syncwarp();
    const double c_l = lane < q ? C[q * CS + lane] : 0.0;
    {
      // all lanes must run the solves: they contain warp shuffles (a ?: would skip them on lanes >= q)
      const float v = tri_bwd32<SP, CS>(Lf, inv, tri_fwd32<SP>(cr, inv, (float)c_l, lane, q), lane, q);
      a = lane < q ? (double)v : 0.0;
    }
    double dmax = 0.0;
#pragma unroll 1
    for (int it = 0; it < 2; ++it) {
      if (lane < SP) abuf[lane] = a;
      __syncwarp();
      double r0 = c_l, r1 = 0.0, r2 = 0.0, r3 = 0.0;
#pragma unroll
      for (int k = 0; k < SP; k += 4) {
        if (k < q) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int kk = k + u;
            if (kk < q && lane < q) {
              const double cv = C[kk <= lane ? lane * CS + kk : kk * CS + lane];
              const double ak = abuf[kk];
              if (u == 0) r0 = fma(-cv, ak, r0);
              if (u == 1) r1 = fma(-cv, ak, r1);
              if (u == 2) r2 = fma(-cv, ak, r2);
              if (u == 3) r3 = fma(-cv, ak, r3);
            }
          }
        }
      }
      __syncwarp();
      const double r = (r0 + r1) + (r2 + r3);
      const float v = tri_bwd32<SP, CS>(Lf, inv, tri_fwd32<SP>(cr, inv, (float)r, lane, q), lane, q);
      const double dd = lane < q ? (double)v : 0.0;
      a += dd;
      dmax = fabs(dd);
    }
    // convergence: final correction <= 1e-8 max|a| (otherwise the FP64 path redoes the point)
    double amax = fabs(a);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    double ca = lane < q ? c_l * a : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ca += __shfl_xor_sync(0xffffffffu, ca, o);
    Di = C[q * CS + q] - ca;
    ok = (dmax <= 1e-8 * amax) && (Di > 0.0);
#ifdef VIF_MIX_DEBUG
    if (q == 1 && lane < 2) printf("lane %d c_l %g a %g dmax %g amax %g Di %g inv %g cr0 %g\n", lane, c_l, a, dmax, amax, Di, (double)inv, (double)cr[0]);
#endif
  }
#ifdef VIF_MIX_DEBUG
  else if (q == 1 && lane == 0) printf("fp32 chol failed q=1 cr0 %g\n", (double)cr[0]);
#endif
  return ok;
}

template <int FAM, int RB, int NB, int MINB>
__global__ void __launch_bounds__(VW * 32, MINB) vecchia_mix_kernel(
    const double* __restrict__ U, int64_t ldu, int mk, int ld, const double* __restrict__ X,
    const int32_t* __restrict__ nbr, int mv, const int64_t* __restrict__ order, int64_t npts, CovParams p,
    double* __restrict__ W, int64_t ldw, double* __restrict__ Dpos, double* __restrict__ B_out,
    double* __restrict__ D_out, DevStatus* __restrict__ st) {
  constexpr int SP = RB * 8;
  constexpr int CS = SP + 1;
  constexpr int NT = RB * (RB + 1) / 2;
  static_assert(SP <= 32, "mixed solver variant needs s <= 32");
  extern __shared__ __align__(16) double vsm[];
  __shared__ int Sidx_all[VW][SP];
  __shared__ double tbl[64];
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* C = vsm + warp * vreg_warp_doubles<RB>(p.d);
  float* cb32 = reinterpret_cast<float*>(C + SP * CS);  // [2][SP] floats (in colbuf's 2*SP doubles)
  double* abuf = C + SP * CS + SP;                      // [SP] (second half of colbuf)
  double* coef = C + SP * CS + 2 * SP;                  // [SP]
  double* xs = coef + SP;                               // [SP][d]
  int* Sidx = Sidx_all[warp];
  const int64_t pos = (int64_t)blockIdx.x * VW + warp;
  if (pos >= npts) return;
  const int64_t i = order[pos];

  // ---- conditioning set and its coordinates ----
  const int nb0 = lane < mv ? nbr[i * mv + lane] : -1;
  const int q = __popc(__ballot_sync(0xffffffffu, nb0 >= 0));
  const int s = q + 1;
  const int myidx = lane < q ? nb0 : (lane == q ? (int)i : -1);
  if (lane < SP) Sidx[lane] = myidx;
  stage_xs<FAM>(X, myidx, p.d, p, lane, s, xs);
  __syncwarp();

  // ---- 1 + 2. Gram on DMMA with the kernel evaluations between ring fill and drain ----
  {
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
    gram_fill<RB, NB>(rp, mk, f);
    eval_lower<FAM, 4>(xs, s, CS, p.d, p.nugget, tbl, lane, C);
    gram_drain<RB, NB>(rp, mk, acc, f);
    __syncwarp();
    int t = 0;
#pragma unroll
    for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
      for (int R2 = 0; R2 <= R1; ++R2, ++t) {
        const int r = R1 * 8 + (lane >> 2), c = R2 * 8 + 2 * (lane & 3);
        if (r < s) {
          if (c <= r) C[r * CS + c] -= acc[t][0];
          if (c + 1 <= r) C[r * CS + c + 1] -= acc[t][1];
        }
      }
    __syncwarp();
  }

  // ---- 3 + 4. mixed-precision solve ----
  double a = 0.0, Di = 0.0;
  bool ok = mix_solve<SP>(C, cb32, abuf, q, lane, a, Di);
  if (!ok) {
    // FP64 fallback (rare): plain Cholesky in shared memory decides NOT_PD
    double Dd;
    if (!fp64_chol_solve<CS>(C, coef, s, q, lane, &Dd)) {
      if (lane == 0) atomicMin(&st->bad_row, (unsigned long long)i);
      for (int c = 2 * lane; c < ld; c += 64) *reinterpret_cast<double2*>(W + pos * ldw + c) = make_double2(0.0, 0.0);
      if (lane == 0) {
        Dpos[pos] = 1.0;
        if (D_out) D_out[i] = __longlong_as_double(0x7ff8000000000000LL);
      }
      return;
    }
    Di = Dd;
    a = lane < q ? coef[lane] : 0.0;
    __syncwarp();
  }
  {
    const double rs = rsqrt_nr(Di);
    if (lane < SP) coef[lane] = lane < q ? -a * rs : (lane == q ? rs : 0.0);
    if (B_out && lane < mv) B_out[i * mv + lane] = lane < q ? -a : 0.0;
  }
  __syncwarp();

  // ---- 5. w_i, r_i over ld columns (as in vecchia_reg_kernel) ----
  for (int c0 = 0; c0 < ld; c0 += 512) {
    double2 o[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) o[t] = make_double2(0.0, 0.0);
    for (int k = 0; k < s; k += 2) {
      double2 u0[8], u1[8];
      const double* r0 = U + (int64_t)Sidx[k] * ldu + c0 + 2 * lane;
      const bool has1 = k + 1 < s;
      const double* r1 = has1 ? U + (int64_t)Sidx[k + 1] * ldu + c0 + 2 * lane : r0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const bool in = c0 + 2 * lane + 64 * t < ld;
        u0[t] = in ? __ldg(reinterpret_cast<const double2*>(r0 + 64 * t)) : make_double2(0.0, 0.0);
        u1[t] = (in && has1) ? __ldg(reinterpret_cast<const double2*>(r1 + 64 * t)) : make_double2(0.0, 0.0);
      }
      const double f0 = coef[k], f1 = has1 ? coef[k + 1] : 0.0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        o[t].x = fma(f0, u0[t].x, o[t].x);
        o[t].y = fma(f0, u0[t].y, o[t].y);
        o[t].x = fma(f1, u1[t].x, o[t].x);
        o[t].y = fma(f1, u1[t].y, o[t].y);
      }
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int c = c0 + 2 * lane + 64 * t;
      if (c < ld) *reinterpret_cast<double2*>(W + pos * ldw + c) = o[t];
    }
  }
  if (lane == 0) {
    Dpos[pos] = Di;
    if (D_out) D_out[i] = Di;
  }
}

// ------------------------------------------------------------------------------------------
// Warp-specialised variant for s <= 32 (the production kernel for m_v <= 31).
// A CTA holds 4 warp pairs.  The "Gram" warp of a pair (warps 0-3) does only step 1: it streams
// the s rows of U through a 4-deep register ring (32 k in flight) into back-to-back DMMAs and
// writes the lower Gram tiles into one of two shared-memory slots.  The "solver" warp of the
// pair (warps 4-7, same SMSP) takes the slot and does steps 2-5 (kernel evaluations, Cholesky,
// back substitution, W row) while its Gram warp already streams the next point.  Slots are
// handed over with mbarriers (full: 32 producer arrivals, empty: 32 consumer arrivals).  With 2
// CTAs per SM every SMSP runs 2 Gram + 2 solver warps, so the DMMA pipe is fed by warps that
// never stall on the latency-bound scalar phases.
template <int RB>
__host__ __device__ constexpr int ws_slot_doubles() {
  return RB * 8 * (RB * 8 + 1);
}
template <int RB>
__host__ __device__ constexpr int ws_pair_doubles(int d) {
  return 2 * ws_slot_doubles<RB>() + 3 * RB * 8 + RB * 8 * d;  // 2 slots + colbuf[2][SP] + coef[SP] + xs
}

template <int FAM, int RB>
__global__ void __launch_bounds__(256, 2) vecchia_ws_kernel(
    const double* __restrict__ U, int64_t ldu, int mk, int ld, const double* __restrict__ X,
    const int32_t* __restrict__ nbr, int mv, const int64_t* __restrict__ order, int64_t npts, CovParams p,
    double* __restrict__ W, int64_t ldw, double* __restrict__ Dpos, double* __restrict__ B_out,
    double* __restrict__ D_out, DevStatus* __restrict__ st) {
  constexpr int SP = RB * 8;
  constexpr int CS = SP + 1;
  constexpr int NT = RB * (RB + 1) / 2;
  constexpr int NBUF = 4;
  constexpr int SLOT = ws_slot_doubles<RB>();
  static_assert(SP <= 32, "warp-specialised variant needs s <= 32");
  extern __shared__ __align__(16) double vsm[];
  __shared__ uint64_t full_bar[4][2], empty_bar[4][2];
  __shared__ int hdr_idx[4][2][SP];
  __shared__ long long hdr_pt[4][2][2];
  __shared__ int hdr_q[4][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp & 3;
  if (threadIdx.x < 8) {
    mbar_init(&full_bar[threadIdx.x >> 1][threadIdx.x & 1], 32);
    mbar_init(&empty_bar[threadIdx.x >> 1][threadIdx.x & 1], 32);
  }
  __syncthreads();
  double* base = vsm + pair * ws_pair_doubles<RB>(p.d);
  const int64_t pair_global = (int64_t)blockIdx.x * 4 + pair;
  const int64_t npairs = (int64_t)gridDim.x * 4;

  if (warp < 4) {
    // =========================== Gram warp ===========================
    for (int64_t t = 0, pos = pair_global; pos < npts; ++t, pos += npairs) {
      const int sl = (int)(t & 1);
      const unsigned use = (unsigned)(t >> 1);
      const int64_t i = order[pos];
      const int nb0 = lane < mv ? nbr[i * mv + lane] : -1;
      const int q = __popc(__ballot_sync(0xffffffffu, nb0 >= 0));
      const int myidx = lane < q ? nb0 : (lane == q ? (int)i : -1);
      const double* rp[RB];
#pragma unroll
      for (int R = 0; R < RB; ++R) {
        const int gi = __shfl_sync(0xffffffffu, myidx, R * 8 + (lane >> 2));
        rp[R] = gi >= 0 ? U + (int64_t)gi * ldu + 2 * (lane & 3) : nullptr;
      }
      double acc[NT][2];
#pragma unroll
      for (int tt = 0; tt < NT; ++tt) acc[tt][0] = acc[tt][1] = 0.0;
      double2 f[NBUF][RB];
#pragma unroll
      for (int c = 0; c < NBUF; ++c)
#pragma unroll
        for (int R = 0; R < RB; ++R)
          f[c][R] = (rp[R] != nullptr && 8 * c < mk) ? __ldg(reinterpret_cast<const double2*>(rp[R] + 8 * c))
                                                     : make_double2(0.0, 0.0);
      for (int k0 = 0; k0 < mk; k0 += 8 * NBUF) {
#pragma unroll
        for (int c = 0; c < NBUF; ++c) {
          if (k0 + 8 * c < mk) {
            int tt = 0;
#pragma unroll
            for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
              for (int R2 = 0; R2 <= R1; ++R2, ++tt) dmma884(acc[tt][0], acc[tt][1], f[c][R1].x, f[c][R2].x);
            tt = 0;
#pragma unroll
            for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
              for (int R2 = 0; R2 <= R1; ++R2, ++tt) dmma884(acc[tt][0], acc[tt][1], f[c][R1].y, f[c][R2].y);
          }
          const int kn = k0 + 8 * NBUF + 8 * c;
#pragma unroll
          for (int R = 0; R < RB; ++R)
            f[c][R] = (rp[R] != nullptr && kn < mk) ? __ldg(reinterpret_cast<const double2*>(rp[R] + kn))
                                                    : make_double2(0.0, 0.0);
        }
      }
      // hand the Gram tiles to the solver warp
      if (use > 0) mbar_wait(&empty_bar[pair][sl], (use - 1) & 1);
      double* C = base + sl * SLOT;
      {
        int tt = 0;
#pragma unroll
        for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
          for (int R2 = 0; R2 <= R1; ++R2, ++tt) {
            const int r = R1 * 8 + (lane >> 2), c = R2 * 8 + 2 * (lane & 3);
            C[r * CS + c] = acc[tt][0];
            C[r * CS + c + 1] = acc[tt][1];
          }
      }
      if (lane < SP) hdr_idx[pair][sl][lane] = myidx;
      if (lane == 0) {
        hdr_pt[pair][sl][0] = i;
        hdr_pt[pair][sl][1] = pos;
        hdr_q[pair][sl] = q;
      }
      mbar_arrive(&full_bar[pair][sl]);
    }
    return;
  }

  // =========================== solver warp ===========================
  double* colbuf = base + 2 * SLOT;  // [2][SP]
  double* coef = colbuf + 2 * SP;    // [SP]
  double* xs = coef + SP;            // [SP][d]
  for (int64_t t = 0, pos_t = pair_global; pos_t < npts; ++t, pos_t += npairs) {
    const int sl = (int)(t & 1);
    const unsigned use = (unsigned)(t >> 1);
    mbar_wait(&full_bar[pair][sl], use & 1);
    double* C = base + sl * SLOT;
    const int* Sidx = hdr_idx[pair][sl];
    const int64_t i = hdr_pt[pair][sl][0];
    const int64_t pos = hdr_pt[pair][sl][1];
    const int q = hdr_q[pair][sl];
    const int s = q + 1;
    if (lane < s) {
      const int gi = Sidx[lane];
      for (int k = 0; k < p.d; ++k) xs[lane * p.d + k] = X[(int64_t)gi * p.d + k];
    }
    __syncwarp();
    // ---- 2. C_S = K(X_S, X_S) - G_S + sigma^2 I (lower triangle, evenly over lanes) ----
    const int ne = s * (s + 1) / 2;
    for (int e = lane; e < ne; e += 32) {
      int r = (int)((sqrtf_fast(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
      if ((r + 1) * (r + 2) / 2 <= e) ++r;
      if (r * (r + 1) / 2 > e) --r;
      const int c = e - r * (r + 1) / 2;
      double v = cov<FAM>(xs + r * p.d, xs + c * p.d, p) - C[r * CS + c];
      if (r == c) v += p.nugget;
      C[r * CS + c] = v;
    }
    __syncwarp();
    // ---- 3. Cholesky, row `lane` in registers; padded rows are identity ----
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
        double* cb = colbuf + (j & 1) * SP;
        if (lane < SP) cb[lane] = lrj;
        __syncwarp();
#pragma unroll
        for (int c = j + 1; c < SP; ++c) crow[c] = fma(-lrj, cb[c], crow[c]);
      }
    }
    if (!ok) {
      if (lane == 0) atomicMin(&st->bad_row, (unsigned long long)i);
      for (int c = 2 * lane; c < ld; c += 64) *reinterpret_cast<double2*>(W + pos * ldw + c) = make_double2(0.0, 0.0);
      if (lane == 0) {
        Dpos[pos] = 1.0;
        if (D_out) D_out[i] = __longlong_as_double(0x7ff8000000000000LL);
      }
      __syncwarp();
      mbar_arrive(&empty_bar[pair][sl]);
      continue;
    }
#pragma unroll
    for (int c = 0; c < SP; ++c)
      if (lane < SP) C[lane * CS + c] = crow[c];
    __syncwarp();
    // ---- 4. A_i^T = L_NN^{-T} l (lane k ends with x_k) ----
    {
      double a = lane < q ? C[q * CS + lane] : 0.0;
      for (int j = q - 1; j >= 0; --j) {
        const double xj = __shfl_sync(0xffffffffu, a * myinv, j);
        if (lane == j) a = xj;
        else if (lane < j) a = fma(-C[j * CS + lane], xj, a);
      }
      const double rs = rsqrt_nr(Di);
      if (lane < SP) coef[lane] = lane < q ? -a * rs : (lane == q ? rs : 0.0);
      if (B_out && lane < mv) B_out[i * mv + lane] = lane < q ? -a : 0.0;
    }
    __syncwarp();
    // ---- 5. w_i, r_i over ld columns (16 loads in flight per lane) ----
    for (int c0 = 0; c0 < ld; c0 += 512) {
      double2 o[8];
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) o[tt] = make_double2(0.0, 0.0);
      for (int k = 0; k < s; k += 2) {
        double2 u0[8], u1[8];
        const double* r0 = U + (int64_t)Sidx[k] * ldu + c0 + 2 * lane;
        const bool has1 = k + 1 < s;
        const double* r1 = has1 ? U + (int64_t)Sidx[k + 1] * ldu + c0 + 2 * lane : r0;
#pragma unroll
        for (int tt = 0; tt < 8; ++tt) {
          const bool in = c0 + 2 * lane + 64 * tt < ld;
          u0[tt] = in ? __ldg(reinterpret_cast<const double2*>(r0 + 64 * tt)) : make_double2(0.0, 0.0);
          u1[tt] = (in && has1) ? __ldg(reinterpret_cast<const double2*>(r1 + 64 * tt)) : make_double2(0.0, 0.0);
        }
        const double f0 = coef[k], f1 = has1 ? coef[k + 1] : 0.0;
#pragma unroll
        for (int tt = 0; tt < 8; ++tt) {
          o[tt].x = fma(f0, u0[tt].x, o[tt].x);
          o[tt].y = fma(f0, u0[tt].y, o[tt].y);
          o[tt].x = fma(f1, u1[tt].x, o[tt].x);
          o[tt].y = fma(f1, u1[tt].y, o[tt].y);
        }
      }
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        const int c = c0 + 2 * lane + 64 * tt;
        if (c < ld) *reinterpret_cast<double2*>(W + pos * ldw + c) = o[tt];
      }
    }
    if (lane == 0) {
      Dpos[pos] = Di;
      if (D_out) D_out[i] = Di;
    }
    __syncwarp();
    mbar_arrive(&empty_bar[pair][sl]);
  }
}

// ------------------------------------------------------------------------------------------
// Production kernel for s <= 32: warp specialisation sized to the B200 FP64 pipe.
// Each SMSP has one FP64 unit that retires one DMMA.8x8x4 per 16 cycles (DMMA latency ~26
// cycles) and also executes the DFMAs of the scalar steps.  A CTA of 4 + 4*NS warps runs per SM:
//   Gram warp g (warps 0-3, one per SMSP): only step 1, streaming the s rows of U through the
//     register ring into back-to-back DMMAs; its Gram tiles go to slot (t mod NS) of its group;
//   solver warps (g, j) (warps 4 + 4j + g, same SMSP as g): steps 2-5 for every NS-th point of
//     the group (kernel evaluations, Cholesky, back substitution, W row).
// NS solvers per Gram warp keep the latency-bound scalar phases off the DMMA critical path.
// Slots are handed over with mbarriers (full / empty, 32 arrivals each).
template <int RB, int NS>
__host__ __device__ constexpr int ws3_doubles(int d) {
  // NS slots per group (SP x (SP+1)) + per solver: colbuf[2][SP] + coef[SP] + xs[SP][d]
  return 4 * NS * (RB * 8 * (RB * 8 + 1)) + 4 * NS * (3 * RB * 8 + RB * 8 * d);
}

// Steps 2-5 of one point for a solver warp of the warp-specialised kernels: C = the point's Gram
// slot (lower tiles of U_S U_S^T, stride SP + 1), Sidx = S (i last), scratch: colbuf[2][SP],
// coef[SP], xs[SP][d].  Writes W row `pos`, Dpos[pos], B_out[i], D_out[i].
template <int FAM, int RB>
__device__ __forceinline__ void ws_solve_point(double* __restrict__ C, const int* __restrict__ Sidx, int64_t i,
                                               int64_t pos, int q, double* __restrict__ colbuf,
                                               double* __restrict__ coef, double* __restrict__ xs,
                                               const double* __restrict__ U, int64_t ldu, int ld,
                                               const double* __restrict__ X, int mv, const CovParams& p,
                                               double* __restrict__ W, int64_t ldw, double* __restrict__ Dpos,
                                               double* __restrict__ B_out, double* __restrict__ D_out,
                                               DevStatus* __restrict__ st, const double* __restrict__ tbl,
                                               int lane) {
  constexpr int SP = RB * 8;
  constexpr int CS = SP + 1;
  const int s = q + 1;
  stage_xs<FAM>(X, lane < s ? Sidx[lane] : 0, p.d, p, lane, s, xs);
  __syncwarp();
  // ---- 2. C_S = K(X_S, X_S) + sigma^2 I - G_S (EU evaluations in flight per lane) ----
  eval_lower<FAM, 4, 1>(xs, s, CS, p.d, p.nugget, tbl, lane, C);
  __syncwarp();
  // ---- 3. Cholesky (row `lane` in registers) ----
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
#pragma unroll
  for (int jj = 0; jj < SP; ++jj) {
    const double djj = __shfl_sync(0xffffffffu, crow[jj], jj);
    if (jj < s) {
      ok = ok && (djj > 0.0);
      if (jj == s - 1) Di = djj;
    }
    const double y = rsqrt_nr(djj);
    const double lrj = crow[jj] * y;
    crow[jj] = lrj;
    if (lane == jj) myinv = y;
    if (jj + 1 < SP) {
      double* cb = colbuf + (jj & 1) * SP;
      if (lane < SP) cb[lane] = lrj;
      __syncwarp();
#pragma unroll
      for (int c = jj + 1; c < SP; ++c) crow[c] = fma(-lrj, cb[c], crow[c]);
    }
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
#pragma unroll
  for (int c = 0; c < SP; ++c)
    if (lane < SP) C[lane * CS + c] = crow[c];
  __syncwarp();
  // ---- 4. back substitution ----
  {
    double a = lane < q ? C[q * CS + lane] : 0.0;
    for (int jj = q - 1; jj >= 0; --jj) {
      const double xj = __shfl_sync(0xffffffffu, a * myinv, jj);
      if (lane == jj) a = xj;
      else if (lane < jj) a = fma(-C[jj * CS + lane], xj, a);
    }
    const double rs = rsqrt_nr(Di);
    if (lane < SP) coef[lane] = lane < q ? -a * rs : (lane == q ? rs : 0.0);
    if (B_out && lane < mv) B_out[i * mv + lane] = lane < q ? -a : 0.0;
  }
  __syncwarp();
  // ---- 5. W row ----
  for (int c0 = 0; c0 < ld; c0 += 512) {
    double2 o[8];
#pragma unroll
    for (int tt = 0; tt < 8; ++tt) o[tt] = make_double2(0.0, 0.0);
    for (int k = 0; k < s; k += 2) {
      double2 u0[8], u1[8];
      const double* r0 = U + (int64_t)Sidx[k] * ldu + c0 + 2 * lane;
      const bool has1 = k + 1 < s;
      const double* r1 = has1 ? U + (int64_t)Sidx[k + 1] * ldu + c0 + 2 * lane : r0;
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        const bool in = c0 + 2 * lane + 64 * tt < ld;
        u0[tt] = in ? __ldg(reinterpret_cast<const double2*>(r0 + 64 * tt)) : make_double2(0.0, 0.0);
        u1[tt] = (in && has1) ? __ldg(reinterpret_cast<const double2*>(r1 + 64 * tt)) : make_double2(0.0, 0.0);
      }
      const double f0 = coef[k], f1 = has1 ? coef[k + 1] : 0.0;
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        o[tt].x = fma(f0, u0[tt].x, o[tt].x);
        o[tt].y = fma(f0, u0[tt].y, o[tt].y);
        o[tt].x = fma(f1, u1[tt].x, o[tt].x);
        o[tt].y = fma(f1, u1[tt].y, o[tt].y);
      }
    }
#pragma unroll
    for (int tt = 0; tt < 8; ++tt) {
      const int c = c0 + 2 * lane + 64 * tt;
      if (c < ld) *reinterpret_cast<double2*>(W + pos * ldw + c) = o[tt];
    }
  }
  if (lane == 0) {
    Dpos[pos] = Di;
    if (D_out) D_out[i] = Di;
  }
}

template <int FAM, int RB, int NS>
__global__ void __launch_bounds__(128 + 128 * NS, 1) vecchia_ws3_kernel(
    const double* __restrict__ U, int64_t ldu, int mk, int ld, const double* __restrict__ X,
    const int32_t* __restrict__ nbr, int mv, const int64_t* __restrict__ order, int64_t npts, CovParams p,
    double* __restrict__ W, int64_t ldw, double* __restrict__ Dpos, double* __restrict__ B_out,
    double* __restrict__ D_out, DevStatus* __restrict__ st) {
  constexpr int SP = RB * 8;
  constexpr int CS = SP + 1;
  constexpr int NT = RB * (RB + 1) / 2;
  constexpr int SLOT = SP * CS;
  constexpr int SCR = 3 * SP;  // + SP * d
  static_assert(SP <= 32, "needs s <= 32");
  extern __shared__ __align__(16) double vsm[];
  __shared__ uint64_t full_bar[4][NS], empty_bar[4][NS];
  __shared__ int hdr_idx[4][NS][SP];
  __shared__ long long hdr_pt[4][NS][2];
  __shared__ int hdr_q[4][NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp & 3;
  if (threadIdx.x < 4 * NS) {
    mbar_init(&full_bar[threadIdx.x / NS][threadIdx.x % NS], 32);
    mbar_init(&empty_bar[threadIdx.x / NS][threadIdx.x % NS], 32);
  }
  __shared__ double tbl[64];
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  __syncthreads();
  double* slots = vsm + g * NS * SLOT;  // group g's NS slots
  const int64_t grp = (int64_t)blockIdx.x * 4 + g;
  const int64_t ngrp = (int64_t)gridDim.x * 4;

  if (warp < 4) {
    // ================= Gram warp =================
    for (int64_t t = 0, pos = grp; pos < npts; ++t, pos += ngrp) {
      const int sl = (int)(t % NS);
      const unsigned use = (unsigned)(t / NS);
      const int64_t i = order[pos];
      const int nb0 = lane < mv ? nbr[i * mv + lane] : -1;
      const int q = __popc(__ballot_sync(0xffffffffu, nb0 >= 0));
      const int myidx = lane < q ? nb0 : (lane == q ? (int)i : -1);
      const double* rp[RB];
#pragma unroll
      for (int R = 0; R < RB; ++R) {
        const int gi = __shfl_sync(0xffffffffu, myidx, R * 8 + (lane >> 2));
        rp[R] = gi >= 0 ? U + (int64_t)gi * ldu + 2 * (lane & 3) : nullptr;
      }
      double acc[NT][2];
#pragma unroll
      for (int tt = 0; tt < NT; ++tt) acc[tt][0] = acc[tt][1] = 0.0;
      gram_ring<RB, 4>(rp, mk, acc);
      if (use > 0) mbar_wait(&empty_bar[g][sl], (use - 1) & 1);
      double* C = slots + sl * SLOT;
      {
        int tt = 0;
#pragma unroll
        for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
          for (int R2 = 0; R2 <= R1; ++R2, ++tt) {
            const int r = R1 * 8 + (lane >> 2), c = R2 * 8 + 2 * (lane & 3);
            C[r * CS + c] = acc[tt][0];
            C[r * CS + c + 1] = acc[tt][1];
          }
      }
      if (lane < SP) hdr_idx[g][sl][lane] = myidx;
      if (lane == 0) {
        hdr_pt[g][sl][0] = i;
        hdr_pt[g][sl][1] = pos;
        hdr_q[g][sl] = q;
      }
      mbar_arrive(&full_bar[g][sl]);
    }
    return;
  }

  // ================= solver warp (group g, index j) =================
  const int j = (warp - 4) >> 2;
  double* scr = vsm + 4 * NS * SLOT + (size_t)(g * NS + j) * (SCR + SP * p.d);
  double* colbuf = scr;           // [2][SP]
  double* coef = colbuf + 2 * SP; // [SP]
  double* xs = coef + SP;         // [SP][d]
  double* C = slots + j * SLOT;
  const int* Sidx = hdr_idx[g][j];
  for (int64_t t = j, pos_t = grp + (int64_t)j * ngrp; pos_t < npts; t += NS, pos_t += (int64_t)NS * ngrp) {
    const unsigned use = (unsigned)(t / NS);
    mbar_wait(&full_bar[g][j], use & 1);
    const int64_t i = hdr_pt[g][j][0];
    const int64_t pos = hdr_pt[g][j][1];
    const int q = hdr_q[g][j];
    ws_solve_point<FAM, RB>(C, Sidx, i, pos, q, colbuf, coef, xs, U, ldu, ld, X, mv, p, W, ldw, Dpos, B_out, D_out,
                            st, tbl, lane);
    __syncwarp();
    mbar_arrive(&empty_bar[g][j]);
  }
}

// ------------------------------------------------------------------------------------------
// ws4: warp specialisation with a shared-memory ring for the Gram warps.
// Per SMSP (group g of the persistent CTA, one CTA per SM): one Gram warp and NS solver warps.
// The Gram warp streams the s rows of U for its points through an NR-deep ring of 8-column chunks
// (cp.async.cg, 16 B per lane per copy, L1 bypassed), continuously across point boundaries, so
// its DMMA stream never waits on a cold load; it needs no register ring, and with NR chunks in
// flight one warp keeps the SMSP's DMMA pipe fed.  The Gram tiles go to NS shared-memory slots
// (mbarrier full / empty hand-off, as in ws3); solver warps do steps 2-5 (ws_solve_point).
// Needs mk >= 8 * NR (the load side then leads the consume side by less than one point).
template <int RB, int NS, int NR>
__host__ __device__ constexpr size_t ws4_smem_bytes(int d) {
  return sizeof(double) * ((size_t)4 * NR * (RB * 8) * 8 + (size_t)4 * NS * (RB * 8) * (RB * 8 + 1) +
                           (size_t)4 * NS * (3 * RB * 8 + RB * 8 * d));
}

template <int FAM, int RB, int NS, int NR>
__global__ void __launch_bounds__(128 + 128 * NS, 1) vecchia_ws4_kernel(
    const double* __restrict__ U, int64_t ldu, int mk, int ld, const double* __restrict__ X,
    const int32_t* __restrict__ nbr, int mv, const int64_t* __restrict__ order, int64_t npts, CovParams p,
    double* __restrict__ W, int64_t ldw, double* __restrict__ Dpos, double* __restrict__ B_out,
    double* __restrict__ D_out, DevStatus* __restrict__ st) {
  constexpr int SP = RB * 8;
  constexpr int CS = SP + 1;
  constexpr int NT = RB * (RB + 1) / 2;
  constexpr int SLOT = SP * CS;
  constexpr int RING = SP * 8;  // one chunk: SP rows x 8 columns
  static_assert(SP <= 32, "needs s <= 32");
  static_assert(NR >= 2, "ring depth");
  extern __shared__ __align__(16) double vsm[];
  __shared__ uint64_t full_bar[4][NS], empty_bar[4][NS];
  __shared__ int hdr_idx[4][NS][SP];
  __shared__ long long hdr_pt[4][NS][2];
  __shared__ int hdr_q[4][NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp & 3;
  if (threadIdx.x < 4 * NS) {
    mbar_init(&full_bar[threadIdx.x / NS][threadIdx.x % NS], 32);
    mbar_init(&empty_bar[threadIdx.x / NS][threadIdx.x % NS], 32);
  }
  __shared__ double tbl[64];
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  __syncthreads();
  double* ring = vsm + (size_t)g * NR * RING;
  double* slots = vsm + (size_t)4 * NR * RING + (size_t)g * NS * SLOT;
  const int64_t grp = (int64_t)blockIdx.x * 4 + g;
  const int64_t ngrp = (int64_t)gridDim.x * 4;
  const int64_t npg = npts > grp ? (npts - 1 - grp) / ngrp + 1 : 0;  // points of this group

  if (warp < 4) {
    // ================= Gram warp =================
    if (npg == 0) return;
    const int nch = mk >> 3;
    // point-info pipeline: (i, neighbour row) of the load point L, of L+1 (in flight) and i of L+2
    auto ld_i = [&](int64_t t) -> int64_t { return t < npg ? order[grp + t * ngrp] : -1; };
    auto ld_nb = [&](int64_t i) -> int { return (i >= 0 && lane < mv) ? nbr[i * mv + lane] : -1; };
    int64_t p1_i = ld_i(1), p2_i = ld_i(2);
    int p1_nb = ld_nb(p1_i);
    int64_t L_i = ld_i(0);
    int L_nb = ld_nb(L_i);
    int L_q = __popc(__ballot_sync(0xffffffffu, L_nb >= 0));
    int L_idx = lane < L_q ? L_nb : (lane == L_q ? (int)L_i : -1);
    int64_t c_i = L_i;
    int c_q = L_q, c_idx = L_idx;
    // copy layout: 4 consecutive lanes move the 64 contiguous bytes of one row's chunk (2 sectors per
    // row per request, as a coalesced LDG.128), so lane l copies piece l % 4 of rows R * 8 + l / 4
    const double* rp[RB];
    auto set_rows = [&]() {
#pragma unroll
      for (int R = 0; R < RB; ++R) {
        const int gi = __shfl_sync(0xffffffffu, L_idx, R * 8 + (lane >> 2));
        rp[R] = gi >= 0 ? U + (int64_t)gi * ldu + 2 * (lane & 3) : nullptr;
      }
    };
    set_rows();
    int64_t lt = 0;  // load point
    int lc = 0;      // next chunk of the load point to issue
    const int64_t total = npg * nch;
    auto issue = [&]() {
      // next chunk in the stream: chunk lc of load point lt (advancing the point at lc == nch)
      if (lc == nch) {
        lc = 0;
        ++lt;
        c_i = L_i; c_q = L_q; c_idx = L_idx;  // the consume side is still on lt - 1
        L_i = p1_i;
        L_nb = p1_nb;
        p1_i = p2_i;
        p1_nb = ld_nb(p1_i);
        p2_i = ld_i(lt + 2);
        L_q = __popc(__ballot_sync(0xffffffffu, L_nb >= 0));
        L_idx = lane < L_q ? L_nb : (lane == L_q ? (int)L_i : -1);
        set_rows();
      }
      if (lt < npg) {
        double* dst = ring + (size_t)((lt * nch + lc) % NR) * RING + (lane >> 2) * 8 + 2 * (lane & 3);
#pragma unroll
        for (int R = 0; R < RB; ++R)
          cp_async16(dst + R * 64, rp[R] ? rp[R] + lc * 8 : U, rp[R] != nullptr);
      }
      cp_async_commit();
      ++lc;
    };
#pragma unroll 1
    for (int k = 0; k < NR - 1; ++k) issue();

    double acc[NT][2];
    int64_t t = 0;  // consume point
    int cc = 0;     // its chunk
#pragma unroll 1
    for (int64_t gch = 0; gch < total; ++gch) {
      cp_async_wait<NR - 2>();
      __syncwarp();
      if (cc == 0) {
#pragma unroll
        for (int u = 0; u < NT; ++u) acc[u][0] = acc[u][1] = 0.0;
      }
      const double* sl = ring + (size_t)(gch % NR) * RING + 2 * (lane & 3);
      double2 f[RB];
#pragma unroll
      for (int R = 0; R < RB; ++R) f[R] = *reinterpret_cast<const double2*>(sl + (R * 8 + (lane >> 2)) * 8);
      {
        int u = 0;
#pragma unroll
        for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
          for (int R2 = 0; R2 <= R1; ++R2, ++u) dmma884(acc[u][0], acc[u][1], f[R1].x, f[R2].x);
        u = 0;
#pragma unroll
        for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
          for (int R2 = 0; R2 <= R1; ++R2, ++u) dmma884(acc[u][0], acc[u][1], f[R1].y, f[R2].y);
      }
      issue();  // refills the slot read in the previous iteration (all lanes passed the syncwarp above)
      if (++cc == nch) {
        // hand the Gram tiles of point t to its solver
        cc = 0;
        const int sl_i = (int)(t % NS);
        const unsigned use = (unsigned)(t / NS);
        if (use > 0) mbar_wait(&empty_bar[g][sl_i], (use - 1) & 1);
        double* C = slots + sl_i * SLOT;
        int u = 0;
#pragma unroll
        for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
          for (int R2 = 0; R2 <= R1; ++R2, ++u) {
            const int r = R1 * 8 + (lane >> 2), c = R2 * 8 + 2 * (lane & 3);
            C[r * CS + c] = acc[u][0];
            C[r * CS + c + 1] = acc[u][1];
          }
        if (lane < SP) hdr_idx[g][sl_i][lane] = c_idx;
        if (lane == 0) {
          hdr_pt[g][sl_i][0] = c_i;
          hdr_pt[g][sl_i][1] = grp + t * ngrp;
          hdr_q[g][sl_i] = c_q;
        }
        mbar_arrive(&full_bar[g][sl_i]);
        ++t;
      }
    }
    cp_async_wait<0>();
    return;
  }

  // ================= solver warp (group g, index j) =================
  const int j = (warp - 4) >> 2;
  double* scr = vsm + (size_t)4 * NR * RING + (size_t)4 * NS * SLOT + (size_t)(g * NS + j) * (3 * SP + SP * p.d);
  double* colbuf = scr;
  double* coef = colbuf + 2 * SP;
  double* xs = coef + SP;
  double* C = slots + j * SLOT;
  const int* Sidx = hdr_idx[g][j];
  for (int64_t t = j; t < npg; t += NS) {
    const unsigned use = (unsigned)(t / NS);
    mbar_wait(&full_bar[g][j], use & 1);
    if (!(g_vif_debug & 4))  // debug probe: bit 2 skips the solver work (timing only)
      ws_solve_point<FAM, RB>(C, Sidx, hdr_pt[g][j][0], hdr_pt[g][j][1], hdr_q[g][j], colbuf, coef, xs, U, ldu, ld, X,
                              mv, p, W, ldw, Dpos, B_out, D_out, st, tbl, lane);
    __syncwarp();
    mbar_arrive(&empty_bar[g][j]);
  }
}

static void sync_debug_flag(cudaStream_t s) {
  const char* dbg = getenv("VIF_DEBUG_VECCHIA");
  static int last = 0;
  const int v = dbg ? atoi(dbg) : 0;
  if (v != last) {
    cudaMemcpyToSymbolAsync(g_vif_debug, &v, sizeof(int), 0, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    last = v;
  }
}

template <int FAM, int RB, int NS, int NR>
static cudaError_t launch_ws4(const VecchiaArgs& a, cudaStream_t s) {
  sync_debug_flag(s);
  const size_t smem = ws4_smem_bytes<RB, NS, NR>(a.p.d);
  static size_t attr = 0;
  if (attr < smem) {
    cudaError_t e = cudaFuncSetAttribute(vecchia_ws4_kernel<FAM, RB, NS, NR>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = nsm;  // persistent: one CTA (4 groups) per SM
  const int64_t need = (a.npts + 3) / 4;
  if (grid > need) grid = need;
  vecchia_ws4_kernel<FAM, RB, NS, NR><<<(unsigned)grid, 128 + 128 * NS, smem, s>>>(
      a.U, a.ldu, a.mk, a.ld, a.X, a.nbr, a.mv, a.order, a.npts, a.p, a.W, a.ldw, a.Dpos, a.B_out, a.D_out, a.st);
  return cudaGetLastError();
}

template <int FAM, int RB, int NS>
static cudaError_t launch_ws3(const VecchiaArgs& a, cudaStream_t s) {
  const size_t smem = (size_t)ws3_doubles<RB, NS>(a.p.d) * sizeof(double);
  static size_t attr = 0;
  if (attr < smem) {
    cudaError_t e = cudaFuncSetAttribute(vecchia_ws3_kernel<FAM, RB, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = nsm;  // persistent: one CTA (4 groups) per SM
  const int64_t need = (a.npts + 3) / 4;
  if (grid > need) grid = need;
  vecchia_ws3_kernel<FAM, RB, NS><<<(unsigned)grid, 128 + 128 * NS, smem, s>>>(
      a.U, a.ldu, a.mk, a.ld, a.X, a.nbr, a.mv, a.order, a.npts, a.p, a.W, a.ldw, a.Dpos, a.B_out, a.D_out, a.st);
  return cudaGetLastError();
}

template <int FAM, int RB>
static cudaError_t launch_rb(const VecchiaArgs& a, cudaStream_t s) {
  constexpr int NB = RB <= 4 ? 2 : 1;
  const unsigned blocks = (unsigned)((a.npts + VW - 1) / VW);
  // default: per-warp register variant; "ws" selects the warp-specialised variant (measured slower
  // on B200: DMMA and the solver warps' DFMA share the FP64 pipe, profiles/r01_notes.md)
  static const char* variant = getenv("VIF_VECCHIA_VARIANT");
  const bool use_ws = variant && variant[0] == 'w';
  if constexpr (RB <= 4) {
    if (variant && variant[0] == '4' && a.mk >= 64) return launch_ws4<FAM, RB, 3, 8>(a, s);
    if (variant && variant[0] == '5' && a.mk >= 64) return launch_ws4<FAM, RB, 2, 8>(a, s);
    if (variant && variant[0] == '6' && a.mk >= 48) return launch_ws4<FAM, RB, 3, 6>(a, s);
    if (variant && variant[0] == '7' && a.mk >= 96) return launch_ws4<FAM, RB, 3, 12>(a, s);
    if (variant && variant[0] == '8' && a.mk >= 128) return launch_ws4<FAM, RB, 2, 16>(a, s);
    if (variant && variant[0] == '2') return launch_ws3<FAM, RB, 2>(a, s);
    if (variant && variant[0] == '3') return launch_ws3<FAM, RB, 3>(a, s);
    if (use_ws) {
      const size_t smem = (size_t)4 * ws_pair_doubles<RB>(a.p.d) * sizeof(double);
      static size_t wattr = 0;
      if (wattr < smem) {
        cudaError_t e = cudaFuncSetAttribute(vecchia_ws_kernel<FAM, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        wattr = smem;
      }
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      int64_t grid = 2LL * nsm;                       // persistent: 2 CTAs (8 warp pairs) per SM
      const int64_t need = (a.npts + 3) / 4;
      if (grid > need) grid = need;
      vecchia_ws_kernel<FAM, RB><<<(unsigned)grid, 256, smem, s>>>(a.U, a.ldu, a.mk, a.ld, a.X, a.nbr, a.mv, a.order,
                                                                  a.npts, a.p, a.W, a.ldw, a.Dpos, a.B_out,
                                                                  a.D_out, a.st);
      return cudaGetLastError();
    }
    const size_t smem = (size_t)VW * vreg_warp_doubles<RB>(a.p.d) * sizeof(double);
    // VIF_VREG_CFG = "<ring depth><min blocks/SM>" for A/B runs; default "34"
    static const char* cfg_env = getenv("VIF_VREG_CFG");
    const int cfg = cfg_env ? atoi(cfg_env) : 34;
    decltype(&vecchia_reg_kernel<FAM, RB, 3, 4>) kern;
    switch (cfg) {
      case 24: kern = vecchia_reg_kernel<FAM, RB, 2, 4>; break;
      case 44: kern = vecchia_reg_kernel<FAM, RB, 4, 4>; break;
      case 33: kern = vecchia_reg_kernel<FAM, RB, 3, 3>; break;
      case 43: kern = vecchia_reg_kernel<FAM, RB, 4, 3>; break;
      case 25: kern = vecchia_reg_kernel<FAM, RB, 2, 5>; break;
      case 26: kern = vecchia_reg_kernel<FAM, RB, 2, 6>; break;
      case 234: kern = vecchia_mix_kernel<FAM, RB, 3, 4>; break;
      case 224: kern = vecchia_mix_kernel<FAM, RB, 2, 4>; break;
      case 225: kern = vecchia_mix_kernel<FAM, RB, 2, 5>; break;
      default: kern = vecchia_reg_kernel<FAM, RB, 3, 4>; break;
    }
    static size_t attr = 0;
    if (attr < smem) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr = smem;
    }
    {
      const char* dbg = getenv("VIF_DEBUG_VECCHIA");
      static int last = 0;
      const int v = dbg ? atoi(dbg) : 0;
      if (v != last) {
        cudaMemcpyToSymbolAsync(g_vif_debug, &v, sizeof(int), 0, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        last = v;
      }
    }
    kern<<<blocks, VW * 32, smem, s>>>(a.U, a.ldu, a.mk, a.ld, a.X, a.nbr, a.mv, a.order, a.npts, a.p, a.W, a.ldw,
                                       a.Dpos, a.B_out, a.D_out, a.st);
  } else {
    const size_t smem = (size_t)VW * vecchia_warp_doubles<RB>() * sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(vecchia_smem_kernel<FAM, RB, NB>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    vecchia_smem_kernel<FAM, RB, NB><<<blocks, VW * 32, smem, s>>>(a.U, a.ldu, a.mk, a.ld, a.X, a.nbr, a.mv,
                                                                   a.order, a.npts, a.p, a.W, a.ldw, a.Dpos,
                                                                   a.B_out, a.D_out, a.st);
  }
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

}  // namespace vif
