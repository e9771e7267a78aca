// k_gemm.cu -- the two dense FP64 DMMA contractions of the path on one 128 x 128 CTA-tile engine:
//
//   K1b  U_aug[i][a] = sum_{b <= a} S[p][b] Linv[a][b]      (A1: U = K(X,Z) L_m^{-T})
//        "TN": both operands K-contiguous; Linv lower triangular, so each warp stops at its own
//        diagonal (k < its last column) and CTAs never read K-blocks above the diagonal.
//   K4   G[a][b] += sum_p W[p][a] W[p][b]  over a row slab  (A6: [W r]^T [W r])
//        "NT": both operands M-contiguous; only lower 128x128 tiles, and inside a diagonal tile
//        the 6 warps whose 32x32 sub-tile lies above the diagonal skip their MMAs.
//
// 512 threads = 16 warps in a 4 x 4 grid of 32 x 32 warp tiles (16 DMMA 8x8 tiles each);
// BK = 16; 4-stage cp.async ring (one __syncthreads per K-tile).  Shared rows are padded to
// 64 (mod 128) bytes so that the 8-row fragment loads of a warp hit distinct bank halves:
//   TN tile [row][k] stride 24 doubles, fragments are 16-byte loads of a k-pair (the k order of
//      mma.m8n8k4 is permuted identically on both operands);
//   NT tile [k][col] stride 136 doubles, fragments are 8-byte loads.
#include "common.cuh"
#include "kernels.h"

namespace vif {

namespace {
constexpr int EB = 128;      // CTA tile (M and N)
constexpr int EK = 16;       // K-tile
constexpr int ES = 4;        // stages
constexpr int TN_LD = EK + 8;    // 24 doubles = 192 B = 64 mod 128
constexpr int NT_LD = EB + 8;    // 136 doubles = 1088 B = 64 mod 128
constexpr int TN_STAGE = 2 * EB * TN_LD;  // doubles per stage (A + B)
constexpr int NT_STAGE = 2 * EK * NT_LD;
}  // namespace

__device__ __forceinline__ int64_t pos_to_row_g(int64_t p, int64_t chunk, int world, int rank) {
  return (p / chunk) * (int64_t)world * chunk + (int64_t)rank * chunk + p % chunk;
}

// ------------------------------------------------------------------------------------------ TN
__global__ void __launch_bounds__(512, 1) gemm_tn_tri_kernel(const double* __restrict__ A, int64_t lda, int64_t npos,
                                                             const double* __restrict__ B, int64_t ldb, int N,
                                                             double* __restrict__ C, int64_t ldc, int64_t n,
                                                             int64_t chunk, int world, int rank, int64_t pos0,
                                                             int ncb) {
  extern __shared__ __align__(16) double esm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int cb = blockIdx.x % ncb;                 // column block fastest: row block shared in L2
  const int64_t row0 = (int64_t)(blockIdx.x / ncb) * EB;
  const int col0 = cb * EB;
  const int kend = min(N, col0 + EB);              // B lower triangular: k <= last column
  const int kend_w = min(kend, col0 + 32 * wn + 32);
  const int nkt = (kend + EK - 1) / EK;

  auto load_stage = [&](int st, int kt) {
    const int k0 = kt * EK;
    double* as = esm + st * TN_STAGE;
    double* bs = as + EB * TN_LD;
#pragma unroll
    for (int j = 0; j < 2; ++j) {  // A: 128 rows x 8 chunks = 1024
      const int e = tid + j * 512;
      const int r = e >> 3, c2 = (e & 7) * 2;
      const int64_t gr = row0 + r;
      const bool ok = gr < npos && k0 + c2 < kend;
      cp_async16(as + r * TN_LD + c2, ok ? A + gr * lda + k0 + c2 : A, ok);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {  // B: 128 rows x 8 chunks
      const int e = tid + j * 512;
      const int r = e >> 3, c2 = (e & 7) * 2;
      const int gc = col0 + r;
      const bool ok = gc < N && k0 + c2 < kend;
      cp_async16(bs + r * TN_LD + c2, ok ? B + (int64_t)gc * ldb + k0 + c2 : B, ok);
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < ES - 1; ++s) {
    if (s < nkt) load_stage(s, s);
    cp_async_commit();
  }
  const int fr = lane >> 2, fk = (lane & 3) * 2;
  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<ES - 2>();
    __syncthreads();
    {
      const int nk = kt + ES - 1;
      if (nk < nkt) load_stage(nk % ES, nk);
      cp_async_commit();
    }
    if (kt * EK < kend_w) {
      const double* as = esm + (kt % ES) * TN_STAGE + (wm * 32 + fr) * TN_LD + fk;
      const double* bs = esm + (kt % ES) * TN_STAGE + EB * TN_LD + (wn * 32 + fr) * TN_LD + fk;
#pragma unroll
      for (int kk = 0; kk < EK; kk += 8) {
        double2 af[4], bf[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) af[t] = *reinterpret_cast<const double2*>(as + t * 8 * TN_LD + kk);
#pragma unroll
        for (int t = 0; t < 4; ++t) bf[t] = *reinterpret_cast<const double2*>(bs + t * 8 * TN_LD + kk);
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
  }
  cp_async_wait<0>();
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t p = row0 + wm * 32 + a * 8 + fr;
    if (p >= npos) continue;
    const int64_t i = pos_to_row_g(pos0 + p, chunk, world, rank);
    if (i >= n) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int c = col0 + wn * 32 + b * 8 + (lane & 3) * 2;
      if (c < N) *reinterpret_cast<double2*>(C + i * ldc + c) = make_double2(acc[a][b][0], acc[a][b][1]);
    }
  }
}

// ------------------------------------------------------------------------------------------ NT
__device__ __forceinline__ void syrk_tile_ij(int t, int& I, int& J) {
  int i = 0;
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  I = i;
  J = t - i * (i + 1) / 2;
}

__global__ void __launch_bounds__(512, 1) syrk_nt_kernel(const double* __restrict__ W, int64_t ldw, int64_t nrows,
                                                         int ncols, int ntiles, int64_t rows_per_split,
                                                         double* __restrict__ Gpart) {
  extern __shared__ __align__(16) double esm[];
  const int t = blockIdx.x % ntiles;   // tiles fastest: the CTAs of one row slab run together (L2 reuse)
  const int split = blockIdx.x / ntiles;
  int I, J;
  syrk_tile_ij(t, I, J);
  const bool diag = I == J;
  const int64_t r0 = (int64_t)split * rows_per_split;
  const int64_t r1 = min(nrows, r0 + rows_per_split);
  const int nkt = r0 < r1 ? (int)((r1 - r0 + EK - 1) / EK) : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const bool active = !(diag && wn > wm);  // 32x32 sub-tile entirely above the diagonal
  const int a0 = I * EB, b0 = J * EB;

  auto load_stage = [&](int st, int kt) {
    const int64_t k0 = r0 + (int64_t)kt * EK;
    double* as = esm + st * NT_STAGE;
    double* bs = as + EK * NT_LD;
#pragma unroll
    for (int j = 0; j < 2; ++j) {  // 16 rows x 64 chunks = 1024
      const int e = tid + j * 512;
      const int r = e >> 6, c2 = (e & 63) * 2;
      const int64_t gr = k0 + r;
      const bool okr = gr < r1;
      {
        const bool ok = okr && a0 + c2 < ncols;
        cp_async16(as + r * NT_LD + c2, ok ? W + gr * ldw + a0 + c2 : W, ok);
      }
      if (!diag) {
        const bool ok = okr && b0 + c2 < ncols;
        cp_async16(bs + r * NT_LD + c2, ok ? W + gr * ldw + b0 + c2 : W, ok);
      }
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < ES - 1; ++s) {
    if (s < nkt) load_stage(s, s);
    cp_async_commit();
  }
  const int fk = lane & 3, fc = lane >> 2;
  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<ES - 2>();
    __syncthreads();
    {
      const int nk = kt + ES - 1;
      if (nk < nkt) load_stage(nk % ES, nk);
      cp_async_commit();
    }
    if (active) {
      const double* as = esm + (kt % ES) * NT_STAGE + fk * NT_LD + wm * 32 + fc;
      const double* bs = esm + (kt % ES) * NT_STAGE + (diag ? 0 : EK * NT_LD) + fk * NT_LD + wn * 32 + fc;
#pragma unroll
      for (int kk = 0; kk < EK; kk += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) af[q] = as[kk * NT_LD + q * 8];
#pragma unroll
        for (int q = 0; q < 4; ++q) bf[q] = bs[kk * NT_LD + q * 8];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
      }
    }
  }
  cp_async_wait<0>();
  double* out = Gpart + (size_t)blockIdx.x * EB * EB;
  const int fr = lane >> 2, fcc = (lane & 3) * 2;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = wm * 32 + a * 8 + fr, c = wn * 32 + b * 8 + fcc;
      *reinterpret_cast<double2*>(out + r * EB + c) = make_double2(acc[a][b][0], acc[a][b][1]);
    }
}

__global__ void syrk_nt_reduce_kernel(const double* __restrict__ Gpart, int ntiles, int nsplit, int ncols,
                                      double* __restrict__ G, int ldg) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)ntiles * EB * EB) return;
  const int t = (int)(e / (EB * EB));
  const int rc = (int)(e % (EB * EB));
  int I, J;
  syrk_tile_ij(t, I, J);
  const int a = I * EB + rc / EB, b = J * EB + rc % EB;
  if (a >= ncols || b >= ncols || b > a) return;
  double s = 0.0;
  for (int sp = 0; sp < nsplit; ++sp) s += Gpart[((size_t)sp * ntiles + t) * EB * EB + rc];
  G[(size_t)a * ldg + b] = s;
}

// ------------------------------------------------------------------------------------------ host
cudaError_t launch_gemm_tn_tri(const double* S, int64_t lds, int64_t npos, const double* Linv, int ldl, int N,
                               double* U, int64_t ldu, int64_t n, int64_t chunk, int world, int rank,
                               int64_t pos0, cudaStream_t s) {
  if (npos == 0 || N == 0) return cudaSuccess;
  const size_t smem = (size_t)ES * TN_STAGE * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tn_tri_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int ncb = (N + EB - 1) / EB;
  const int64_t nrb = (npos + EB - 1) / EB;
  gemm_tn_tri_kernel<<<(unsigned)(nrb * ncb), 512, smem, s>>>(S, lds, npos, Linv, ldl, N, U, ldu, n, chunk, world,
                                                              rank, pos0, ncb);
  return cudaGetLastError();
}

int syrk_nt_ntiles(int ncols) {
  const int nt1 = (ncols + EB - 1) / EB;
  return nt1 * (nt1 + 1) / 2;
}

int syrk_nt_nsplit(int ncols, int64_t nrows, int num_sms) {
  const int nt = syrk_nt_ntiles(ncols);
  int64_t ns = (4LL * num_sms + nt - 1) / nt;       // ~4 waves of 1 CTA / SM
  const int64_t max_by_rows = (nrows + 511) / 512;   // >= 512 rows per split
  if (ns > max_by_rows) ns = max_by_rows;
  if (ns < 1) ns = 1;
  return (int)ns;
}

size_t syrk_nt_part_doubles(int ncols, int nsplit) { return (size_t)syrk_nt_ntiles(ncols) * nsplit * EB * EB; }

cudaError_t launch_syrk_nt(const double* W, int64_t ldw, int64_t nrows, int ncols, int nsplit, double* Gpart,
                           double* G, int ldg, cudaStream_t s) {
  const int nt = syrk_nt_ntiles(ncols);
  const int64_t rps = nrows > 0 ? (nrows + nsplit - 1) / nsplit : 0;
  const size_t smem = (size_t)ES * NT_STAGE * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(syrk_nt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  syrk_nt_kernel<<<nt * nsplit, 512, smem, s>>>(W, ldw, nrows, ncols, nt, rps, Gpart);
  const int64_t tot = (int64_t)nt * EB * EB;
  syrk_nt_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(Gpart, nt, nsplit, ncols, G, ldg);
  return cudaGetLastError();
}

}  // namespace vif
