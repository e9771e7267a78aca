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
#include "tma.cuh"
#include <stdlib.h>

namespace vif {

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

// C[row(p)][c] (+)= alpha sum_k A[p][k] B[c][k], A: npos x K (lda), B: N x K (ldb); B lower-triangular
// (B[c][k] = 0 for k > c) when tri, so K-tiles past a column block's last column are skipped.
//
// Blackwell tile movement: a producer warp streams BK = 16-wide k-slices of the A rows (128 x 16) and B
// rows (BN x 16) with cp.async.bulk.tensor (boxes of 16 doubles x rows, SWIZZLE_128B) through a GS-stage
// shared-memory ring, completing on per-stage "full" mbarriers; (BM / 32) x (BN / 32) consumer warps of
// 32 x 32 wait on "full", run the DMMAs and release the stage on its "empty" mbarrier (no CTA barrier in
// the main loop).  Persistent: one CTA per SM walks a static tile schedule, and the producer runs ahead
// into the next tile while the consumers store the last one.  96 x 128 tiles (12 consumer warps + the producer = 13 warps, at most
// 4 per SMSP, so 128 registers each), or 128 x 64 for N <= 64.
//
// Fragments (k contiguous in both operands): lane l holds row l/4 of an 8-row block and the k-pair
// kk + 2(l%4) + {0,1} (one 16-byte load), used as two k-steps with the same k permutation on both
// operands.  Under the 128-B swizzle the 8 rows x 4 chunks of a fragment load hit every bank 4 times:
// four wavefronts for 512 bytes, conflict-free.
namespace {
constexpr int GBK = 16, GS = 4;
template <int BM, int BN>
struct GemmCfg {
  static constexpr int WM = BM / 32;                 // consumer warp rows
  static constexpr int NCW = WM * (BN / 32);         // consumer warps
  static constexpr int THREADS = 32 * (NCW + 1);
  static constexpr int ABYTES = BM * 128;           // one stage of A: BM rows x 16 doubles
  static constexpr int BBYTES = BN * 128;
  static constexpr int STAGE = ABYTES + BBYTES;
  static constexpr size_t SMEM = (size_t)GS * STAGE + 1024 + 2 * GS * 8;
};
}  // namespace

template <int BM, int BN>
__global__ void __launch_bounds__(GemmCfg<BM, BN>::THREADS, 1) gemm_tn_tma_kernel(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t npos, int N, int K,
    int tri, double* __restrict__ C, int64_t ldc, int64_t n, int64_t chunk, int world, int rank, int64_t pos0,
    double alpha, int accum) {
  using Cfg = GemmCfg<BM, BN>;
  extern __shared__ uint8_t g_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(g_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + GS * Cfg::STAGE);
  uint64_t* empty = full + GS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // persistent CTAs, static schedule: CTA b takes tiles b, b + G, b + 2G, ...; tile t -> row block t / ncb and
  // column block (t + t / ncb) % ncb, so the G tiles in flight at once cover few row blocks (A from L2) and a
  // CTA's sequence rotates through the column blocks (a triangular B makes them cost 1 : 2 : ... : ncb)
  const int ncb = (N + BN - 1) / BN;
  const int ntiles = (int)(((npos + BM - 1) / BM) * ncb);
  auto tile_of = [&](int t, int64_t& row0, int& col0, int& nkt) {
    const int rb = t / ncb;
    row0 = (int64_t)rb * BM;
    col0 = ((t + rb) % ncb) * BN;
    int kend = K;
    if (tri && col0 + BN < kend) kend = col0 + BN;
    nkt = (kend + GBK - 1) / GBK;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < GS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == Cfg::NCW) {  // ---------------- producer: runs ahead across tile boundaries ----------------
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      int it = 0;  // global stage counter of this CTA
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int64_t row0;
        int col0, nkt;
        tile_of(t, row0, col0, nkt);
        for (int kt = 0; kt < nkt; ++kt, ++it) {
          const int s = it % GS;
          if (it >= GS) mbar_wait(&empty[s], (unsigned)(((it / GS) + 1) & 1));
          mbar_expect_tx(&full[s], Cfg::STAGE);
          uint8_t* st = sm + s * Cfg::STAGE;
          tma_load_2d(st, &tmA, kt * GBK, (int)row0, &full[s]);
          tma_load_2d(st + Cfg::ABYTES, &tmB, kt * GBK, col0, &full[s]);
        }
      }
    }
    return;
  }

  // ---------------- consumers: (BM/32) x (BN/32) warps of 32 x 32 ----------------
  const int wm = warp % Cfg::WM, wn = warp / Cfg::WM;
  const int fr = lane >> 2, t4 = lane & 3;
  // byte offsets inside a stage of the 16-byte fragment loads: row (block*8 + fr), k-pair chunk kh*4 + t4
  uint32_t offA[2][4], offB[2][4];
#pragma unroll
  for (int kh = 0; kh < 2; ++kh)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int ra = wm * 32 + q * 8 + fr, rb = wn * 32 + q * 8 + fr;
      offA[kh][q] = (uint32_t)(ra * 128 + (((kh * 4 + t4) ^ (ra & 7)) << 4));
      offB[kh][q] = (uint32_t)(Cfg::ABYTES + rb * 128 + (((kh * 4 + t4) ^ (rb & 7)) << 4));
    }
  const uint32_t sbase = smem_u32(sm);
  const bool pair = !((N | ldc) & 1);  // 16-byte stores need an even N and ldc
  int it = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int64_t row0;
    int col0, nkt;
    tile_of(t, row0, col0, nkt);
    // a warp's 32 columns end at col0 + 32 (wn + 1): with a triangular B it skips later K-tiles
    int kend_w = tri ? min(K, col0 + 32 * (wn + 1)) : K;
    const int nkt_w = (kend_w + GBK - 1) / GBK;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int kt = 0; kt < nkt; ++kt, ++it) {
      const int s = it % GS;
      mbar_wait(&full[s], (unsigned)((it / GS) & 1));
      if (kt < nkt_w) {
        const uint32_t st = sbase + s * Cfg::STAGE;
#pragma unroll
        for (int kh = 0; kh < 2; ++kh) {
          double2 af[4], bf[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            af[q] = lds_f64x2(st + offA[kh][q]);
            bf[q] = lds_f64x2(st + offB[kh][q]);
          }
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
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // epilogue (the producer is already filling the next tile's stages): lane holds C[fr][2*(lane&3) + {0,1}]
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int64_t p = row0 + wm * 32 + a * 8 + fr;
      if (p >= npos) continue;
      const int64_t i = pos_to_row(pos0 + p, chunk, world, rank);
      if (i >= n) continue;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int c = col0 + wn * 32 + b * 8 + t4 * 2;
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
}

// host: the TMA GEMM on A (npos x K, lda) and B (N x K, ldb); 96 x 128 tiles, 128 x 64 when N <= 64
static cudaError_t gemm_tn_tma(const double* A, int64_t lda, int64_t npos, const double* B, int64_t ldb, int N, int K,
                               int tri, double* C, int64_t ldc, int64_t n, int64_t chunk, int world, int rank,
                               int64_t pos0, double alpha, int accum, cudaStream_t s) {
  if (npos <= 0 || N <= 0) return cudaSuccess;
  if (K <= 0) return cudaErrorInvalidValue;
  auto go = [&](auto kern, auto cfg) -> cudaError_t {
    using Cfg = decltype(cfg);
    constexpr int BM = Cfg::WM * 32, BN = Cfg::NCW / Cfg::WM * 32;
    CUtensorMap ta, tb;
    cudaError_t e = make_tmap_f64(&ta, A, (uint64_t)npos, (uint64_t)K, (uint64_t)lda, BM);
    if (e != cudaSuccess) return e;
    e = make_tmap_f64(&tb, B, (uint64_t)N, (uint64_t)K, (uint64_t)ldb, BN);
    if (e != cudaSuccess) return e;
    e = smem_optin(kern, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = ((npos + BM - 1) / BM) * ((N + BN - 1) / BN);
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, sms);  // persistent: one CTA per SM
    kern<<<grid, Cfg::THREADS, Cfg::SMEM, s>>>(ta, tb, npos, N, K, tri, C, ldc, n, chunk, world, rank, pos0, alpha,
                                                accum);
    return cudaGetLastError();
  };
  if (N <= 64) return go(gemm_tn_tma_kernel<128, 64>, GemmCfg<128, 64>{});
  return go(gemm_tn_tma_kernel<96, 128>, GemmCfg<96, 128>{});
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
  return gemm_tn_tma(S + pos0 * lds, lds, npos, Linv, mk, mk, mk, 1, Uaug, ld, n, chunk, world, rank, pos0, 1.0, 0,
                     s);
}

// C[p][c] (+)= alpha sum_k A[p][k] B[c][k] for p < nrows, c < N (single rank: row p -> p); B lower
// triangular (k <= c) when tri.  Used by the gradient path (dU, Phi, Gamma).
cudaError_t launch_gemm_tn(const double* A, int64_t lda, int64_t nrows, const double* B, int64_t ldb, int N, int K,
                           int tri, double* C, int64_t ldc, double alpha, int accum, cudaStream_t s) {
  return gemm_tn_tma(A, lda, nrows, B, ldb, N, K, tri, C, ldc, nrows, nrows, 1, 0, 0, alpha, accum, s);
}

}  // namespace vif
