// k_ugemm.cu -- K1: whitened inducing-point features U = K(X,Z) L_m^{-T} (reading c4).
//
// Two launches per evaluation:
//   K1a kx_eval:  S[p][b] = k(x_i(p), z_b) for the rank's rows (p = position), zero for b in [m, mk);
//                 also writes U_aug[i][mk] = y_i and the zero pad columns (mk, ld).
//   K1b gemm_tn:  U_aug[i][a] = sum_{b <= a} S[p][b] Linv[a][b]  -- an FP64 DMMA GEMM whose B
//                 operand is lower triangular, so K-blocks above the diagonal are skipped
//                 (n m^2 flops instead of 2 n m^2).
// Rows are the rank's chunk-cyclic rows: position p -> global row
//   i = (p / chunk) * world * chunk + rank * chunk + p % chunk.
#include "common.cuh"
#include "kernels.h"
#include <stdlib.h>

namespace vif {

__device__ __forceinline__ int64_t pos_to_row(int64_t p, int64_t chunk, int world, int rank) {
  return (p / chunk) * (int64_t)world * chunk + (int64_t)rank * chunk + p % chunk;
}

template <int FAM>
__global__ void __launch_bounds__(256) kx_eval_kernel(const double* __restrict__ X, const double* __restrict__ Z,
                                                      const double* __restrict__ y, int64_t n, int64_t npos,
                                                      int64_t chunk, int world, int rank, int64_t pos0, int m,
                                                      int mk, CovParams p, double* __restrict__ S, int lds,
                                                      double* __restrict__ Uaug, int ld) {
  // one warp per row; lanes stride over the columns.  Z and the 8 row coordinates are staged in
  // shared memory pre-scaled for cov_fast (broadcast reads; a runtime-indexed register array would
  // live in local memory).
  extern __shared__ double kx_zs[];        // m x d
  __shared__ double kx_x[8][VIF_MAX_D];
  __shared__ double tbl[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pos = (int64_t)blockIdx.x * 8 + warp;
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  for (int e = threadIdx.x; e < m * p.d; e += blockDim.x) kx_zs[e] = Z[e] * (fam_scale<FAM>() * p.inv_ls[e % p.d]);
  const int64_t i = pos < npos ? pos_to_row(pos0 + pos, chunk, world, rank) : n;
  const bool valid = i < n;
  if (lane < p.d) kx_x[warp][lane] = valid ? X[i * p.d + lane] * (fam_scale<FAM>() * p.inv_ls[lane]) : 0.0;
  __syncthreads();
  if (pos >= npos) return;
  const double* x = kx_x[warp];
  double* srow = S + pos * (int64_t)lds;
#pragma unroll 4
  for (int b = lane; b < mk; b += 32) {
    double v = 0.0;
    if (valid && b < m) v = cov_fast<FAM>(x, kx_zs + b * p.d, p.d, tbl);
    srow[b] = v;
  }
  if (valid) {
    double* urow = Uaug + i * (int64_t)ld;
    for (int c = mk + lane; c < ld; c += 32) urow[c] = (c == mk) ? y[i] : 0.0;
  }
}

// Specialisation for a compile-time input dimension D (the generic kernel above spends most of its
// issue slots on index arithmetic: ncu shows ~140 warp-instructions per 32 evaluations, issue-bound
// at 88%).  Rows strided over the grid (Z and the exp table staged once per CTA, no modulo), the
// row's coordinates in registers, 32 columns per lane step.
template <int FAM, int D>
__global__ void __launch_bounds__(256) kx_eval_d_kernel(const double* __restrict__ X, const double* __restrict__ Z,
                                                        const double* __restrict__ y, int64_t n, int64_t npos,
                                                        int64_t chunk, int world, int rank, int64_t pos0, int m,
                                                        int mk, CovParams p, double* __restrict__ S, int lds,
                                                        double* __restrict__ Uaug, int ld) {
  extern __shared__ double kx_zs[];  // mk x D, zero rows past m
  __shared__ double tbl[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  double sc[D];
#pragma unroll
  for (int k = 0; k < D; ++k) sc[k] = fam_scale<FAM>() * p.inv_ls[k];
  for (int b = threadIdx.x; b < mk; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < D; ++k) kx_zs[b * D + k] = b < m ? Z[b * D + k] * sc[k] : 0.0;
  }
  __syncthreads();
  for (int64_t pos = (int64_t)blockIdx.x * 8 + warp; pos < npos; pos += (int64_t)gridDim.x * 8) {
    const int64_t i = pos_to_row(pos0 + pos, chunk, world, rank);
    const bool valid = i < n;
    double x[D];
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = valid ? X[i * D + k] * sc[k] : 0.0;
    double* srow = S + pos * (int64_t)lds;
    if (!valid) {
      for (int b = lane; b < mk; b += 32) srow[b] = 0.0;
      continue;
    }
    auto eval = [&](int b) -> double {
      const double* z = kx_zs + b * D;
      double t2;
      {
        const double d0 = x[0] - z[0];
        t2 = d0 * d0;
#pragma unroll
        for (int k = 1; k < D; ++k) {
          const double dk = x[k] - z[k];
          t2 = fma(dk, dk, t2);
        }
      }
      if (FAM == FAM_GAUSS) return sig2_exp_neg(t2, tbl);
      const double t = sqrt_fast(t2);
      const double E = sig2_exp_neg(t, tbl);
      return FAM == FAM_M12 ? E : (FAM == FAM_M32 ? fma(E, t, E) : fma(E, fma(t2, 1.0 / 3.0, t), E));
    };
    const int mfull = m & ~31;  // columns of whole 32-wide steps: no mask
#pragma unroll 4
    for (int b = lane; b < mfull; b += 32) srow[b] = eval(b);
    for (int b = mfull + lane; b < mk; b += 32) srow[b] = b < m ? eval(b) : 0.0;
    if (valid) {
      double* urow = Uaug + i * (int64_t)ld;
      for (int c = mk + lane; c < ld; c += 32) urow[c] = (c == mk) ? y[i] : 0.0;
    }
  }
}

// C[row(p)][c] = sum_k A[p][k] B[c][k], A: npos x K (lda), B: N x K (ldb); B lower-triangular when tri.
// 128 x 64 CTA tile, BK = 32, 8 warps (4 x 2) of 32 x 32, 3-stage cp.async pipeline.
// smem rows padded to 40 doubles (320 B = 64 mod 128 B) so the 16-byte fragment loads
// (k-pair per lane, see below) are bank-conflict free.
namespace {
// BK = 16 keeps the ring at 110 KB so two CTAs (16 warps) share an SM and one CTA's prologue /
// epilogue overlaps the other's main loop (rows padded to 24 doubles = 64 mod 128 B)
constexpr int GBM = 128, GBN = 64, GBK = 16, GST = 3, GPAD = GBK + 8;
constexpr int GCH = GBK / 2;  // 16-byte chunks per tile row
}

__global__ void __launch_bounds__(256, 2) gemm_tn_kernel(const double* __restrict__ A, int64_t lda, int64_t npos,
                                                      const double* __restrict__ B, int64_t ldb, int N, int K,
                                                      int tri, double* __restrict__ C, int64_t ldc, int64_t n,
                                                      int64_t chunk, int world, int rank, int64_t pos0,
                                                      double alpha, int accum) {
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                            // [GST][GBM][GPAD]
  double* Bs = gsm + GST * GBM * GPAD;         // [GST][GBN][GPAD]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 1, wn = warp & 1;     // 4 x 2 warps
  // 1-D grid, column block fastest: the ncb CTAs that share an A row block run together and
  // read it from L2 instead of DRAM
  const int ncb = (N + GBN - 1) / GBN;
  const int64_t row0 = (int64_t)(blockIdx.x / ncb) * GBM;
  const int col0 = (blockIdx.x % ncb) * GBN;
  int kend = K;
  if (tri && col0 + GBN < kend) kend = col0 + GBN;
  const int nkt = (kend + GBK - 1) / GBK;
  // a warp's 32 columns end at col0 + 32 (wn + 1): with a triangular B it skips later K-tiles
  const int kend_w = tri ? min(kend, col0 + 32 * (wn + 1)) : kend;

  auto load_stage = [&](int st, int kt) {
    const int k0 = kt * GBK;
    double* as = As + st * GBM * GPAD;
    double* bs = Bs + st * GBN * GPAD;
#pragma unroll
    for (int j = 0; j < GBM * GCH / 256; ++j) {  // A: GBM rows x GCH chunks of 16 B
      const int e = tid + j * 256;
      const int r = e / GCH, c2 = (e % GCH) * 2;
      const int64_t gr = row0 + r;
      const bool ok = gr < npos && k0 + c2 < kend;
      const double* src = ok ? A + gr * lda + k0 + c2 : A;
      cp_async16(as + r * GPAD + c2, src, ok);
    }
#pragma unroll
    for (int j = 0; j < GBN * GCH / 256; ++j) {  // B: GBN rows x GCH chunks
      const int e = tid + j * 256;
      const int r = e / GCH, c2 = (e % GCH) * 2;
      const int gc = col0 + r;
      const bool ok = gc < N && k0 + c2 < kend;
      const double* src = ok ? B + (int64_t)gc * ldb + k0 + c2 : B;
      cp_async16(bs + r * GPAD + c2, src, ok);
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < GST - 1; ++s) {
    if (s < nkt) load_stage(s, s);
    cp_async_commit();
  }
  const int fr = lane >> 2, fk = (lane & 3) * 2;
  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<GST - 2>();
    __syncthreads();
    {
      const int nk = kt + GST - 1;
      if (nk < nkt) load_stage(nk % GST, nk);
      cp_async_commit();
    }
    if (kt * GBK >= kend_w) continue;
    const double* as = As + (kt % GST) * GBM * GPAD + (wm * 32 + fr) * GPAD + fk;
    const double* bs = Bs + (kt % GST) * GBN * GPAD + (wn * 32 + fr) * GPAD + fk;
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 8) {
      // each lane holds k = kk + fk + {0,1} of its row: two k-steps of 4 with a consistent
      // permutation of k on both operands (the contraction is order-independent)
      double2 af[4], bf[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) af[t] = *reinterpret_cast<const double2*>(as + t * 8 * GPAD + kk);
#pragma unroll
      for (int t = 0; t < 4; ++t) bf[t] = *reinterpret_cast<const double2*>(bs + t * 8 * GPAD + kk);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a].x, bf[b].x);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a].y, bf[b].y);
    }
  }
  cp_async_wait<0>();
  const bool pair = !((N | ldc) & 1);  // 16-byte stores need an even N and ldc
  // epilogue: lane holds C[fr][2*(lane&3) + {0,1}] of each 8x8 tile
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t p = row0 + wm * 32 + a * 8 + fr;
    if (p >= npos) continue;
    const int64_t i = pos_to_row(pos0 + p, chunk, world, rank);
    if (i >= n) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int c = col0 + wn * 32 + b * 8 + (lane & 3) * 2;
      if (c < N) {
        if (pair) {
          double2* dst = reinterpret_cast<double2*>(C + i * ldc + c);
          double2 v = make_double2(alpha * acc[a][b][0], alpha * acc[a][b][1]);
          if (accum) {  // C += alpha A B^T (gradient path)
            const double2 o = *dst;
            v.x += o.x;
            v.y += o.y;
          }
          *dst = v;
        } else {  // odd N or ldc (Laplace path: one right-hand side)
          double* dst = C + i * ldc + c;
          dst[0] = alpha * acc[a][b][0] + (accum ? dst[0] : 0.0);
          if (c + 1 < N) dst[1] = alpha * acc[a][b][1] + (accum ? dst[1] : 0.0);
        }
      }
    }
  }
}

cudaError_t launch_u_features(const double* X, const double* Z, const double* y, int64_t n, int64_t pos0,
                              int64_t npos, int64_t chunk, int world, int rank, int m, int mk, const CovParams& p,
                              const double* Linv, double* S, double* Uaug, int ld, cudaStream_t s, int lds) {
  if (lds <= 0) lds = mk;
  if (npos == 0) return cudaSuccess;
  const int blocks = (int)((npos + 7) / 8);
  const size_t zbytes = (size_t)m * p.d * sizeof(double);
  auto go = [&](auto kern) -> cudaError_t {
    {
      cudaError_t e = smem_optin(kern, zbytes);
      if (e != cudaSuccess) return e;
    }
    kern<<<blocks, 256, zbytes, s>>>(X, Z, y, n, npos, chunk, world, rank, pos0, m, mk, p, S + pos0 * lds, lds,
                                     Uaug, ld);
    return cudaSuccess;
  };
  cudaError_t e0 = cudaSuccess;
  static const char* gen_env = getenv("VIF_KX_GENERIC");
  const bool generic = gen_env && gen_env[0] == '1';
  auto god = [&](auto kern, int D) -> cudaError_t {
    const size_t zb = (size_t)mk * D * sizeof(double);
    int nb = (int)((npos + 7) / 8);
    if (nb > 148 * 8) nb = 148 * 8;
    {
      cudaError_t e = smem_optin(kern, zb);  // static shared memory comes on top
      if (e != cudaSuccess) return e;
    }
    kern<<<nb, 256, zb, s>>>(X, Z, y, n, npos, chunk, world, rank, pos0, m, mk, p, S + pos0 * lds, lds, Uaug, ld);
    return cudaSuccess;
  };
#define VIF_KX_D(DV)                                                      \
  switch (p.family) {                                                     \
    case FAM_M12: e0 = god(kx_eval_d_kernel<FAM_M12, DV>, DV); break;     \
    case FAM_M32: e0 = god(kx_eval_d_kernel<FAM_M32, DV>, DV); break;     \
    case FAM_M52: e0 = god(kx_eval_d_kernel<FAM_M52, DV>, DV); break;     \
    default: e0 = god(kx_eval_d_kernel<FAM_GAUSS, DV>, DV); break;        \
  }
  // the benchmark configurations' dimensions (d = 2: configs 1-3; 3: config 5; 5: the Laplace
  // workload; 10: config 4)
  if (!generic && p.d == 2) {
    VIF_KX_D(2)
  } else if (!generic && p.d == 3) {
    VIF_KX_D(3)
  } else if (!generic && p.d == 5) {
    VIF_KX_D(5)
  } else if (!generic && p.d == 10) {
    VIF_KX_D(10)
  } else {
    switch (p.family) {
      case FAM_M12: e0 = go(kx_eval_kernel<FAM_M12>); break;
      case FAM_M32: e0 = go(kx_eval_kernel<FAM_M32>); break;
      case FAM_M52: e0 = go(kx_eval_kernel<FAM_M52>); break;
      default: e0 = go(kx_eval_kernel<FAM_GAUSS>); break;
    }
  }
#undef VIF_KX_D
  if (e0 != cudaSuccess) return e0;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || mk == 0) return e;
  const size_t smem = (size_t)GST * (GBM + GBN) * GPAD * sizeof(double);
  e = smem_optin(gemm_tn_kernel, smem);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)(((npos + GBM - 1) / GBM) * ((mk + GBN - 1) / GBN));
  gemm_tn_kernel<<<grid, 256, smem, s>>>(S + pos0 * lds, lds, npos, Linv, mk, mk, mk, 1, Uaug, ld, n, chunk, world, rank,
                                         pos0, 1.0, 0);
  return cudaGetLastError();
}

// C[p][c] (+)= alpha sum_k A[p][k] B[c][k] for p < nrows, c < N (single rank: row p -> p); B lower
// triangular (k <= c) when tri.  Used by the gradient path (dU, Phi, Gamma).
cudaError_t launch_gemm_tn(const double* A, int64_t lda, int64_t nrows, const double* B, int64_t ldb, int N, int K,
                           int tri, double* C, int64_t ldc, double alpha, int accum, cudaStream_t s) {
  if (nrows == 0 || N == 0) return cudaSuccess;
  const size_t smem = (size_t)GST * (GBM + GBN) * GPAD * sizeof(double);
  {
    cudaError_t e = smem_optin(gemm_tn_kernel, smem);
    if (e != cudaSuccess) return e;
  }
  const unsigned grid = (unsigned)(((nrows + GBM - 1) / GBM) * ((N + GBN - 1) / GBN));
  gemm_tn_kernel<<<grid, 256, smem, s>>>(A, lda, nrows, B, ldb, N, K, tri, C, ldc, nrows, nrows, 1, 0, 0, alpha, accum);
  return cudaGetLastError();
}

}  // namespace vif
