// k_vecchia.cuh -- K2 + K3 fused: the batched residual-process Vecchia factor and the
// whitened Woodbury rows w_i, r_i.  Instantiated once per covariance family
// (k_vecchia_<family>.cu), dispatched by k_vecchia.cu.
//
// One warp per point i, conditioning set S = (N(i)..., i), s = |N(i)| + 1 <= 8 * RB:
//   1. Gram  G_S = U_S U_S^T over k in [0, mk) on the FP64 tensor core: the s rows of U are
//      gathered straight from L2/HBM into registers (16 B per lane per 8 k, NB chunks in flight);
//      lane l carries k = k0 + 2(l%4) + {0,1} of row l/4 of each 8-row block, which is both the A
//      and the B fragment of mma.m8n8k4 (a consistent k permutation on both operands), so only the
//      RB (RB+1)/2 lower 8x8 tiles are issued.
//   2. C_S = K(X_S, X_S) - G_S + sigma^2 I (nugget by index identity, reading c2) into shared memory;
//      in the register kernel the kernel evaluations (cov_fast) run between the first loads of
//      the Gram and its DMMA loop.
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
__host__ __device__ constexpr int vecchia_warp_doubles(int d) {
  // L (packed lower triangle) + coef (SP) + an 8 x 8 block inverse + the pre-scaled coordinates (SP x d)
  return RB * 8 * (RB * 8 + 1) / 2 + RB * 8 + 64 + RB * 8 * d;
}

template <int FAM, int RB, int NB, int MINB = 3>
__global__ void __launch_bounds__(VW * 32, MINB) vecchia_smem_kernel(
    const double* __restrict__ U, int64_t ldu, int mk, int ld, const double* __restrict__ X,
    const double* __restrict__ Uq, const double* __restrict__ Xq, const int32_t* __restrict__ nbr, int mv, const int64_t* __restrict__ order, int64_t npts, CovParams p,
    double* __restrict__ W, int64_t ldw, double* __restrict__ Dpos, double* __restrict__ B_out,
    double* __restrict__ D_out, DevStatus* __restrict__ st, double* __restrict__ gstate,
    unsigned long long* __restrict__ cmax) {
  constexpr int SP = RB * 8;
  constexpr int NT = RB * (RB + 1) / 2;
  extern __shared__ __align__(16) double vsm[];
  auto li = [](int r, int c) { return r * (r + 1) / 2 + c; };  // packed lower-triangle index
  __shared__ int Sidx_all[VW][SP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* C = vsm + warp * vecchia_warp_doubles<RB>(p.d);
  double* coef = C + SP * (SP + 1) / 2;
  double* linv = coef + SP;
  double* xs = linv + 64;
  __shared__ double tbl[64];
  int* Sidx = Sidx_all[warp];
  const int64_t pos = (int64_t)blockIdx.x * VW + warp;
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  __syncthreads();
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
  // pre-scaled coordinates of S for cov_fast
  for (int t = lane; t < s; t += 32)
    for (int k = 0; k < p.d; ++k)
      xs[t * p.d + k] = (t == q ? Xq : X)[(int64_t)Sidx[t] * p.d + k] * (fam_scale<FAM>() * p.inv_ls[k]);

  // ---- 1. Gram on DMMA ----
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  const double* rp[RB];
#pragma unroll
  for (int R = 0; R < RB; ++R) {
    const int row = R * 8 + (lane >> 2), gi = Sidx[row];
    rp[R] = gi >= 0 ? (row == q ? Uq : U) + (int64_t)gi * ldu + 2 * (lane & 3) : nullptr;  // row q: the point (Uq)
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

  // ---- 2. residual covariance block C_S - U_S U_S^T + nugget I, kept in the DMMA fragment layout
  //         (lane (g, t) of tile (R1, R2) holds rows R1*8+g, columns R2*8+2t, +1); padding rows and
  //         columns are identity ----
  const int g8 = lane >> 2, t4 = lane & 3;
  {
    int t = 0;
#pragma unroll
    for (int R1 = 0; R1 < RB; ++R1)
#pragma unroll
      for (int R2 = 0; R2 <= R1; ++R2, ++t) {
        const int r = R1 * 8 + g8;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int c = R2 * 8 + 2 * t4 + j;
          double v = r == c ? 1.0 : 0.0;
          if (c <= r && r < s) {
            v = cov_fast<FAM>(xs + r * p.d, xs + c * p.d, p.d, tbl) - acc[t][j];
            if (r == c) v += p.nugget;
          }
          acc[t][j] = v;
        }
      }
  }

  // ---- 3. blocked right-looking Cholesky of C_S (i last), 8 x 8 blocks.  Block column J: the
  //         diagonal block is factored (and inverted) redundantly by every lane from shared memory;
  //         the panel L_RJ = C_RJ L_JJ^{-T} and the trailing update C_R1R2 -= L_R1J L_R2J^T are
  //         DMMA products on the fragments (k-slot t <-> column 2t / 2t+1, so both operands are the
  //         lane's own fragment entries).  L ends in C (packed lower triangle) for steps 4-5. ----
  bool ok = true;
  double Di = 0.0;
#pragma unroll
  for (int J = 0; J < RB; ++J) {
    const int tJJ = J * (J + 1) / 2 + J;
    if (2 * t4 <= g8) C[li(J * 8 + g8, J * 8 + 2 * t4)] = acc[tJJ][0];
    if (2 * t4 + 1 <= g8) C[li(J * 8 + g8, J * 8 + 2 * t4 + 1)] = acc[tJJ][1];
    __syncwarp();
    double Lb[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) Lb[r][c] = C[li(J * 8 + r, J * 8 + c)];
    double inv[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const double djj = Lb[jj][jj];
      if (J * 8 + jj < s) ok = ok && (djj > 0.0);
      if (J * 8 + jj == q) Di = djj;
      const double y = rsqrt_nr(djj);
      inv[jj] = y;
      Lb[jj][jj] = djj * y;
#pragma unroll
      for (int r = jj + 1; r < 8; ++r) Lb[r][jj] *= y;
#pragma unroll
      for (int r = jj + 1; r < 8; ++r)
#pragma unroll
        for (int c = jj + 1; c <= r; ++c) Lb[r][c] = fma(-Lb[r][jj], Lb[c][jj], Lb[r][c]);
    }
    __syncwarp();  // every lane has read the block
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) C[li(J * 8 + r, J * 8 + c)] = Lb[r][c];  // same value from every lane
    if (J + 1 < RB) {
      // column jj of L_JJ^{-1} by forward substitution, into linv (same value from every lane)
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        double col[8];
        col[jj] = inv[jj];
#pragma unroll
        for (int r = jj + 1; r < 8; ++r) {
          double sm = 0.0;
#pragma unroll
          for (int k = jj; k < r; ++k) sm = fma(Lb[r][k], col[k], sm);
          col[r] = -sm * inv[r];
        }
#pragma unroll
        for (int r = jj; r < 8; ++r) linv[r * 8 + jj] = col[r];
      }
      __syncwarp();
      const double li0 = 2 * t4 <= g8 ? linv[g8 * 8 + 2 * t4] : 0.0;
      const double li1 = 2 * t4 + 1 <= g8 ? linv[g8 * 8 + 2 * t4 + 1] : 0.0;
#pragma unroll
      for (int R = J + 1; R < RB; ++R) {
        const int tRJ = R * (R + 1) / 2 + J;
        double n0 = 0.0, n1 = 0.0;
        dmma884(n0, n1, acc[tRJ][0], li0);
        dmma884(n0, n1, acc[tRJ][1], li1);
        acc[tRJ][0] = n0;
        acc[tRJ][1] = n1;
      }
#pragma unroll
      for (int R1 = J + 1; R1 < RB; ++R1)
#pragma unroll
        for (int R2 = J + 1; R2 <= R1; ++R2) {
          const int t12 = R1 * (R1 + 1) / 2 + R2, t1 = R1 * (R1 + 1) / 2 + J, t2 = R2 * (R2 + 1) / 2 + J;
          dmma884(acc[t12][0], acc[t12][1], -acc[t1][0], acc[t2][0]);
          dmma884(acc[t12][0], acc[t12][1], -acc[t1][1], acc[t2][1]);
        }
      __syncwarp();  // linv is rewritten by the next block column
    }
  }
  // the panels of L into C (the diagonal blocks are there already)
#pragma unroll
  for (int R = 1; R < RB; ++R)
#pragma unroll
    for (int J = 0; J < R; ++J) {
      const int tRJ = R * (R + 1) / 2 + J;
      C[li(R * 8 + g8, J * 8 + 2 * t4)] = acc[tRJ][0];
      C[li(R * 8 + g8, J * 8 + 2 * t4 + 1)] = acc[tRJ][1];
    }
  __syncwarp();
  if (!ok) {
    if (lane == 0) atomicMin(&st->bad_row, (unsigned long long)i);
    for (int c = 2 * lane; c < ld; c += 64) *reinterpret_cast<double2*>(W + pos * ldw + c) = make_double2(0.0, 0.0);
    if (lane == 0) {
      Dpos[pos] = 1.0;
      if (D_out) D_out[i] = __longlong_as_double(0x7ff8000000000000LL);
    }
    return;
  }

  // ---- 4. A_i^T = L_NN^{-T} l, l = row q of L; lane k holds x_k and x_{k+32} (branch-free shuffles) ----
  {
    const double inv0 = lane < s ? 1.0 / C[li(lane, lane)] : 0.0;
    const double inv1 = lane + 32 < s ? 1.0 / C[li(lane + 32, lane + 32)] : 0.0;
    double a0 = lane < q ? C[li(q, lane)] : 0.0;
    double a1 = lane + 32 < q ? C[li(q, lane + 32)] : 0.0;
    for (int j = q - 1; j >= 0; --j) {
      const double* Lj = C + li(j, 0);  // (reads past column j stay inside the triangle: j < SP - 1)
      const double xj = __shfl_sync(0xffffffffu, j < 32 ? a0 * inv0 : a1 * inv1, j & 31);
      const double l0 = Lj[lane], l1 = Lj[(lane + 32) < SP ? lane + 32 : lane];
      a0 = lane == j ? xj : (lane < j ? fma(-l0, xj, a0) : a0);
      a1 = lane + 32 == j ? xj : (lane + 32 < j ? fma(-l1, xj, a1) : a1);
    }
    const double rs = rsqrt_nr(Di);
    // coefficients of the W row: -A_ik / sqrt(D) for k < q, 1 / sqrt(D) for i itself, 0 beyond
    if (lane < SP) coef[lane] = lane < q ? -a0 * rs : (lane == q ? rs : 0.0);
    if (lane + 32 < SP) coef[lane + 32] = lane + 32 < q ? -a1 * rs : (lane + 32 == q ? rs : 0.0);
    if (B_out) {
      if (lane < mv) B_out[i * mv + lane] = lane < q ? -a0 : 0.0;
      if (lane + 32 < mv) B_out[i * mv + lane + 32] = lane + 32 < q ? -a1 : 0.0;
    }
    if (gstate) {  // vif_grad: L (packed like C, identity padding rows), A_i, 1/L_jj, D_i for its first pass
      constexpr int LP = SP * (SP + 1) / 2;
      double* sp = gstate + pos * (int64_t)vif_state_doubles<RB>();
      for (int e = lane; e < LP; e += 32) sp[e] = C[e];
      if (lane < SP) {
        sp[LP + lane] = lane < q ? a0 : 0.0;
        sp[LP + SP + lane] = lane < s ? inv0 : 1.0;
      }
      if (lane + 32 < SP) {
        sp[LP + lane + 32] = lane + 32 < q ? a1 : 0.0;
        sp[LP + SP + lane + 32] = lane + 32 < s ? inv1 : 1.0;
      }
      if (lane == 0) {
        sp[LP + 3 * SP] = Di;
        sp[LP + 3 * SP + 1] = 1.0;
      }
    }
  }
  __syncwarp();

  // ---- 5. w_i, r_i over ld columns: 512 columns per pass (8 chunks of 64 per lane-pair), rows two
  //         at a time -> 16 independent 16-byte loads in flight per lane ----
  for (int c0 = 0; c0 < ld; c0 += 512) {
    double2 o[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) o[t] = make_double2(0.0, 0.0);
    for (int k = 0; k < s; k += 2) {
      double2 u0[8], u1[8];
      const double* r0 = (k == q ? Uq : U) + (int64_t)Sidx[k] * ldu + c0 + 2 * lane;
      const bool has1 = k + 1 < s;
      const double* r1 = has1 ? (k + 1 == q ? Uq : U) + (int64_t)Sidx[k + 1] * ldu + c0 + 2 * lane : r0;
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
    if (cmax) {  // K4's column maxima of |W| (bit patterns), 64 interleaved copies to spread the atomics
      unsigned long long* cm = cmax + (size_t)(pos & 63) * ld;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int c = c0 + 2 * lane + 64 * t;
        if (c < ld) {
          atomicMax(cm + c, (unsigned long long)__double_as_longlong(fabs(o[t].x)));
          atomicMax(cm + c + 1, (unsigned long long)__double_as_longlong(fabs(o[t].y)));
        }
      }
    }
  }
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
// (row s-1 is the point itself, read from Xq: the training X, or the prediction inputs)
template <int FAM>
__device__ __forceinline__ void stage_xs(const double* __restrict__ X, const double* __restrict__ Xq, int idx, int d,
                                         const CovParams& p, int lane, int s, double* __restrict__ xs) {
  if (lane < s) {
    const double* x = (lane == s - 1 ? Xq : X) + (int64_t)idx * d;
    for (int k = 0; k < d; ++k) xs[lane * d + k] = x[k] * (fam_scale<FAM>() * p.inv_ls[k]);
  }
}

template <int RB>
__host__ __device__ constexpr int vreg_warp_doubles(int d) {
  return RB * 8 * (RB * 8 + 1) + 2 * RB * 8 + RB * 8 + RB * 8 * d;  // C, colbuf[2], coef, xs
}

// SELF: the point's own row / coordinates come from Uq / Xq (prediction); false for the factor
// DD > 0: the input dimension as a compile-time constant (the coordinate loops of the kernel
// evaluations unroll and their index arithmetic folds; d = 2 is instantiated)
template <int FAM, int RB, int NB, int MINB, bool SELF = false, int DD = 0>
__global__ void __launch_bounds__(VW * 32, MINB) vecchia_reg_kernel(
    const double* __restrict__ U, int64_t ldu, int mk, int ld, const double* __restrict__ X,
    const double* __restrict__ Uq, const double* __restrict__ Xq, const int32_t* __restrict__ nbr, int mv, const int64_t* __restrict__ order, int64_t npts, CovParams p,
    double* __restrict__ W, int64_t ldw, double* __restrict__ Dpos, double* __restrict__ B_out,
    double* __restrict__ D_out, DevStatus* __restrict__ st, double* __restrict__ gstate,
    unsigned long long* __restrict__ cmax) {
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
  const int dd = DD > 0 ? DD : p.d;
  double* C = vsm + warp * vreg_warp_doubles<RB>(dd);
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
  stage_xs<FAM>(X, SELF ? Xq : X, myidx, dd, p, lane, s, xs);
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
    const int row = R * 8 + (lane >> 2), gi = Sidx[row];
    rp[R] = gi >= 0 ? (SELF && row == q ? Uq : U) + (int64_t)gi * ldu + 2 * (lane & 3) : nullptr;  // row q: the point (Uq)
  }
  {
    double2 f[NB][RB];
    gram_fill<RB, NB>(rp, mk, f);
    eval_lower<FAM, 4>(xs, s, CS, dd, p.nugget, tbl, lane, C);
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
    if (gstate) {  // vif_grad: L (packed, identity padding rows), A_i, 1/L_jj, D_i for its first pass
      constexpr int LP = SP * (SP + 1) / 2;
      double* sp = gstate + pos * (int64_t)vif_state_doubles<RB>();
      for (int e = lane; e < LP; e += 32) {
        int r = (int)((sqrtf_fast(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
        if ((r + 1) * (r + 2) / 2 <= e) ++r;
        if (r * (r + 1) / 2 > e) --r;
        sp[e] = C[r * CS + e - r * (r + 1) / 2];
      }
      if (lane < SP) {
        sp[LP + lane] = lane < q ? a : 0.0;
        sp[LP + SP + lane] = inv_diag;
      }
      if (lane == 0) {
        sp[LP + 3 * SP] = Di;
        sp[LP + 3 * SP + 1] = 1.0;
      }
    }
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
      const double* r0 = (SELF && k == q ? Uq : U) + (int64_t)Sidx[k] * ldu + c0 + 2 * lane;
      const bool has1 = k + 1 < s;
      const double* r1 = has1 ? (SELF && k + 1 == q ? Uq : U) + (int64_t)Sidx[k + 1] * ldu + c0 + 2 * lane : r0;
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
    if (cmax) {  // K4's column maxima of |W| (bit patterns), 64 interleaved copies to spread the atomics
      unsigned long long* cm = cmax + (size_t)(pos & 63) * ld;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int c = c0 + 2 * lane + 64 * t;
        if (c < ld) {
          atomicMax(cm + c, (unsigned long long)__double_as_longlong(fabs(o[t].x)));
          atomicMax(cm + c + 1, (unsigned long long)__double_as_longlong(fabs(o[t].y)));
        }
      }
    }
  }
  if (lane == 0) {
    Dpos[pos] = Di;
    if (D_out) D_out[i] = Di;
  }
}

template <int FAM, int RB>
static cudaError_t launch_reg(const VecchiaArgs& a, cudaStream_t s) {
  const unsigned blocks = (unsigned)((a.npts + VW - 1) / VW);
  const size_t smem = (size_t)VW * vreg_warp_doubles<RB>(a.p.d) * sizeof(double);
  // ring depth 3, 4 blocks (16 warps) per SM (measured: depth 2 / 5 blocks slower, profiles/r01_notes.md)
  decltype(&vecchia_reg_kernel<FAM, RB, 3, 4>) kern;
  if (a.Uself) {
    kern = vecchia_reg_kernel<FAM, RB, 3, 4, true>;
  } else {
    static const char* gen_env = getenv("VIF_VECCHIA_GENERIC_D");  // A/B: runtime-d loops at d = 2 too
    const int dd = (gen_env && gen_env[0] == '1') ? 0 : a.p.d;
    if (dd == 2) kern = vecchia_reg_kernel<FAM, RB, 3, 4, false, 2>;
    else kern = vecchia_reg_kernel<FAM, RB, 3, 4>;
  }
  {
    cudaError_t e = smem_optin(kern, smem);  // static shared memory comes on top
    if (e != cudaSuccess) return e;
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
  kern<<<blocks, VW * 32, smem, s>>>(a.U, a.ldu, a.mk, a.ld, a.X, a.Uself ? a.Uself : a.U, a.Xself ? a.Xself : a.X,
                                     a.nbr, a.mv, a.order, a.npts, a.p, a.W, a.ldw, a.Dpos, a.B_out, a.D_out, a.st,
                                     a.state, a.cmax);
  return cudaGetLastError();
}

template <int FAM, int RB>
static cudaError_t launch_smem(const VecchiaArgs& a, cudaStream_t s) {
  const unsigned blocks = (unsigned)((a.npts + VW - 1) / VW);
  const size_t smem = (size_t)VW * vecchia_warp_doubles<RB>(a.p.d) * sizeof(double);
  // Gram ring depth 1 (a 2-deep ring measured slower at 12 warps/SM, profiles/r01_notes.md)
  auto kern = vecchia_smem_kernel<FAM, RB, 1>;
  {
    cudaError_t e = smem_optin(kern, smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<blocks, VW * 32, smem, s>>>(a.U, a.ldu, a.mk, a.ld, a.X, a.Uself ? a.Uself : a.U,
                                                                 a.Xself ? a.Xself : a.X, a.nbr, a.mv,
                                                                 a.order, a.npts, a.p, a.W, a.ldw, a.Dpos,
                                                                 a.B_out, a.D_out, a.st, a.state, a.cmax);
  return cudaGetLastError();
}

template <int FAM, int RB>
static cudaError_t launch_rb(const VecchiaArgs& a, cudaStream_t s) {
  // s <= 32: the per-warp register kernel.  Measured and rejected on B200 (profiles/r01_notes.md):
  // warp-specialised Gram / solver warps (register ring or cp.async shared-memory ring) and a
  // mixed-precision (FP32 Cholesky + FP64 refinement) solver.
  // (measured slower for s <= 32, profiles/r02_notes.md: the blocked DMMA Cholesky of the s > 32 kernel,
  // 9.8-10.5 vs 8.2 ms at n = 300k; a software-pipelined warp that overlaps point k's Cholesky / solve / W
  // pass with point k+1's Gram chunk by chunk, 46.7 vs 27.8 ms at n = 1M -- 242 registers, 8 warps per SM)
  if constexpr (RB <= 4) return launch_reg<FAM, RB>(a, s);
  else return launch_smem<FAM, RB>(a, s);
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
