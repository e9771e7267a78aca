// k_ozaki.cu -- K4 on the integer tensor cores: G = [W r]^T [W r] ("M"; whitened, reading c4) as an
// exact sum of int8 x int8 products (an Ozaki-type splitting of FP64 into integer digit slices).
//
// Why.  FP64 has no tcgen05 kind; the FP64 tensor path is warp-level DMMA at 37.1 TF/s.  tcgen05 kind::i8
// runs at ~2.9 POPS on this B200 (tools/tc_i8_probe.cu), so an FP64 product rebuilt from 28 int8 products
// runs at ~100 TF/s FP64-equivalent -- 2.7x the DMMA peak -- with int32 accumulation that is EXACT.
//
// Splitting (per column a of W, global over the rows): e_a = exponent with max_k |W_ka| < 2^(e_a - 1);
// X_ka = rint(W_ka 2^(55 - e_a)) (|X| <= 2^54, one rounding of 2^-55 relative to the column maximum);
// X = sum_{p=0..6} d_p 256^(6-p) with balanced digits d_1..d_6 in [-128, 127] and |d_0| <= 65.  Then
//     W_ka W_kb = 2^(e_a + e_b - 14) sum_{p,q} d_p(a) d_q(b) 2^(-8(p+q)),
// truncated to the levels L = p + q <= 6 (28 products; the dropped levels are below 2^-51 of the
// column-maximum product, measured at config 3: |G - G_exact| <= 1e-16 |G|max, the same as FP64).
// Level L's products sum in int32: at most 7 pairs x 2^14 x rows -- exact for <= 16,384 rows per
// accumulation (OZ_CHUNK).
//
// Kernels.  (1) oz_colmax: column maxima (atomicMax on the bit patterns of |W|).  (2) oz_slice: W ->
// digit slices Ws[p][a][k] (int8, k contiguous: the K-major tcgen05 operand), through a shared-memory
// transpose of 64 x 64 tiles.  (3) oz_syrk_kernel: persistent, one CTA per SM, units = (128 x 64 output
// tile, row split of <= 16,384 rows); warp 0 streams TMA boxes {32 rows of k, 128 or 64 columns, 7 slices}
// through a 4-stage ring; warp 1 issues per stage 10 tcgen05.mma.kind::i8: A slice p (128 columns of W)
// times the CONCATENATED B slices 0..6-p (64 columns each, contiguous in shared memory), accumulating
// into TMEM columns 64p.. -- so level L lands in columns [64L, 64L + 64) (448 of the 512 TMEM columns)
// without any bookkeeping; warps 2-5 drain the 7 levels per unit (tcgen05.ld), combine them in FP64
// (Horner in 2^-8) and write the unit's partial tile.  (4) oz_reduce: deterministic sum over the splits,
// scaled by 2^(e_a + e_b - 14).
#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"
#include "tma.cuh"

#include <algorithm>

namespace vif {

namespace {
constexpr int OZ_S = 7;           // digit slices
constexpr int OZ_BM = 128;        // tile rows (a) = TMEM lanes
constexpr int OZ_BN = 64;         // tile columns (b) per level
constexpr int OZ_BK = 32;         // k (rows of W) per stage = one MMA K
constexpr int OZ_STAGES = 4;
constexpr int OZ_CHUNK = 16384;   // rows per int32 accumulation
constexpr int OZ_A_BYTES = OZ_S * OZ_BM * OZ_BK;
constexpr int OZ_B_BYTES = OZ_S * OZ_BN * OZ_BK;
constexpr int OZ_STAGE_BYTES = OZ_A_BYTES + OZ_B_BYTES;
constexpr size_t OZ_SMEM = (size_t)OZ_STAGES * OZ_STAGE_BYTES + 1024 + 256;
constexpr int OZ_EPI_LD = 33;  // staging row stride (doubles): conflict-free column writes and row reads
constexpr int OZ_GEPI = 8;     // epilogue warps of the K1 GEMM: two per TMEM lane quarter (16-column chunks)
constexpr int OZ_GLD = 17;     // their staging row stride (doubles)
constexpr size_t OZ_GEMM_SMEM = OZ_SMEM + (size_t)OZ_GEPI * 32 * OZ_GLD * 8 + 512;
constexpr int OZ_TROWS = 64;      // slicer tile
}  // namespace

// scale exponent of a column from its maximum (bit pattern of a non-negative double): max < 2^(e - 1);
// clamped so that 2^(55 - e) stays a normal double
__device__ __forceinline__ int oz_exp(unsigned long long bits) {
  const double mx = __longlong_as_double((long long)bits);
  if (!(mx > 0.0)) return 0;
  int e;
  frexp(mx, &e);
  return max(e + 1, -960);
}

// lower tiles (I, J) of the (ceil(ncols/128) x ceil(ncols/64)) grid that touch the lower triangle: J <= 2I + 1
__host__ __device__ __forceinline__ void oz_tile(int t, int nJ, int& I, int& J) {
  int i = 0;
  for (;;) {
    const int c = min(2 * i + 2, nJ);
    if (t < c) break;
    t -= c;
    ++i;
  }
  I = i;
  J = t;
}

static int oz_ntiles(int nI, int nJ) {
  int t = 0;
  for (int i = 0; i < nI; ++i) t += std::min(2 * i + 2, nJ);
  return t;
}

__global__ void __launch_bounds__(256) oz_colmax_kernel(const double* __restrict__ W, int64_t ldw, int64_t nrows,
                                                        int ncols, int64_t rows_per_cta,
                                                        unsigned long long* __restrict__ cmax) {
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min(nrows, r0 + rows_per_cta);
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
    double m0 = 0.0, m1 = 0.0, m2 = 0.0, m3 = 0.0;
    int64_t r = r0;
    for (; r + 3 < r1; r += 4) {
      m0 = fmax(m0, fabs(W[r * ldw + c]));
      m1 = fmax(m1, fabs(W[(r + 1) * ldw + c]));
      m2 = fmax(m2, fabs(W[(r + 2) * ldw + c]));
      m3 = fmax(m3, fabs(W[(r + 3) * ldw + c]));
    }
    for (; r < r1; ++r) m0 = fmax(m0, fabs(W[r * ldw + c]));
    m0 = fmax(fmax(m0, m1), fmax(m2, m3));
    if (m0 > 0.0) atomicMax(&cmax[c], (unsigned long long)__double_as_longlong(m0));
  }
}

// cmax[c] = max over the 64 interleaved copies written by the vecchia W pass (bit patterns of |w| >= 0 order
// like the values; a NaN pattern exceeds every finite one, as oz_colmax_kernel's atomicMax would keep it)
__global__ void oz_colmax_fold_kernel(const unsigned long long* __restrict__ c64, int ncols,
                                      unsigned long long* __restrict__ cmax) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  unsigned long long m = 0;
  for (int k = 0; k < 64; ++k) m = max(m, c64[(size_t)k * ncols + c]);
  cmax[c] = m;
}

// W rows [0, nrows) -> Ws[kb][p][a][k mod 32] for a < ncp, k < nrp (zero digits outside the matrix); a
// non-finite entry sets *flag (the reduction then returns NaN, as the FP64 contraction would).
// Digits without a carry chain: with Y = X + 0x808080808080 the six low bytes y_j of Y give d = y_j - 128
// (= y_j ^ 0x80 as a signed byte) and the top digit is Y >> 48 (arithmetic): X = sum_j (y_j - 128) 256^j +
// (Y >> 48) 256^6.  A thread owns one column and 16 rows; byte j of four rows is packed into one word with
// three byte permutes and stored to the transposed tile T[p][col][rows] (word stride 17: conflict-free).
__global__ void __launch_bounds__(256) oz_slice_kernel(const double* __restrict__ W, int64_t ldw, int64_t nrows,
                                                       int ncols, const unsigned long long* __restrict__ cmax,
                                                       int8_t* __restrict__ Ws, int64_t ncp, int* __restrict__ flag) {
  __shared__ uint32_t T[OZ_S][64][OZ_TROWS / 4 + 1];
  const int64_t r0 = (int64_t)blockIdx.x * OZ_TROWS;
  const int c0 = blockIdx.y * 64;
  const int col = threadIdx.x & 63, rg = threadIdx.x >> 6;  // rows rg*16 .. rg*16 + 15
  const int c = c0 + col;
  const double sc = c < ncols ? ldexp(1.0, 55 - oz_exp(cmax[c])) : 0.0;
  bool bad = false;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t r = r0 + rg * 16 + g * 4 + i;
      double w = (r < nrows && c < ncols) ? W[r * ldw + c] : 0.0;
      if (!isfinite(w)) {
        bad = true;
        w = 0.0;
      }
      const long long Y = __double2ll_rn(w * sc) + 0x808080808080LL;
      lo[i] = (uint32_t)Y;
      hi[i] = (uint32_t)((unsigned long long)Y >> 32);
    }
    const int wi = rg * 4 + g;
    // slice p >= 1 <-> byte j = 6 - p of Y (biased); slice 0 <-> byte 6 (hi byte 2, unbiased)
#pragma unroll
    for (int p = 1; p < OZ_S; ++p) {
      const int j = 6 - p;
      const uint32_t* src = j < 4 ? lo : hi;
      const uint32_t sel = (uint32_t)((j & 3) | (((j & 3) + 4) << 4));
      const uint32_t x = __byte_perm(src[0], src[1], sel), y = __byte_perm(src[2], src[3], sel);
      T[p][col][wi] = __byte_perm(x, y, 0x5410) ^ 0x80808080u;
    }
    {
      const uint32_t x = __byte_perm(hi[0], hi[1], 0x62), y = __byte_perm(hi[2], hi[3], 0x62);
      T[0][col][wi] = __byte_perm(x, y, 0x5410);
    }
  }
  if (bad) atomicOr(flag, 1);
  __syncthreads();
  // out: for each k-block kb of the tile and slice p, columns c0..c0+63 are 2 KB contiguous (32 B each);
  // 16-byte stores (half h of a column's 32 bytes), a warp instruction writes 512 contiguous bytes
  constexpr int NKB = OZ_TROWS / OZ_BK;
  static_assert(NKB * OZ_S * 64 * 2 % 256 == 0, "whole iterations");
#pragma unroll
  for (int it = 0; it < NKB * OZ_S * 64 * 2 / 256; ++it) {
    const int e = it * 256 + threadIdx.x;
    const int h = e & 1, cl = (e >> 1) & 63, pk = e >> 7;
    const int p = pk % OZ_S, kb = pk / OZ_S;
    const int64_t kbg = blockIdx.x * NKB + kb;
    const uint32_t* tw = &T[p][cl][kb * (OZ_BK / 4) + 4 * h];
    *reinterpret_cast<uint4*>(Ws + (((kbg * OZ_S + p) * ncp + c0 + cl) * OZ_BK) + 16 * h) =
        make_uint4(tw[0], tw[1], tw[2], tw[3]);
  }
}

// One stage of MMAs (issued by one thread): A slice p (OZ_BM rows) times the concatenated B slices
// 0..6-p (OZ_BN rows each, contiguous in shared memory) into TMEM columns OZ_BN p ..: level L = p + q lands in
// columns [OZ_BN L, OZ_BN (L + 1)).  On the first stage of a tile slice 0 of A initialises every level.
__device__ __forceinline__ void oz_issue_stage(uint32_t tmem, uint32_t a0, bool first) {
  const uint32_t b0 = a0 + OZ_A_BYTES;
#pragma unroll
  for (int p = 0; p < OZ_S; ++p) {
#pragma unroll
    for (int q0 = 0; q0 < OZ_S - p; q0 += 4) {
      const int nq = min(4, OZ_S - p - q0);
      tc_mma_i8(tmem + (uint32_t)(OZ_BN * (p + q0)), tc_desc_sw32(a0 + p * OZ_BM * OZ_BK),
                tc_desc_sw32(b0 + q0 * OZ_BN * OZ_BK), tc_idesc_i8(OZ_BM, OZ_BN * nq), (!first) | (p > 0));
    }
  }
}

// int32 -> double, exact: 2^52 + 2^31 + v has v + 2^31 in its low mantissa bits (one LOP + one DADD on the
// FP64 pipe instead of a conversion)
__device__ __forceinline__ double oz_i2d(uint32_t v) {
  return __hiloint2double(0x43300000, (int)(v ^ 0x80000000u)) - 4503601774854144.0;
}

// 32 accumulator columns of this thread's TMEM lane (ta = lane quarter + column), all 7 levels combined in
// FP64: t = sum_L acc_L 2^(-8L) (Horner from the last level)
__device__ __forceinline__ void oz_drain32(uint32_t ta, double (&t)[32]) {
  uint32_t v[32];
  tc_ld32(ta + (uint32_t)((OZ_S - 1) * OZ_BN), v);
  tc_wait_ld();
#pragma unroll
  for (int j = 0; j < 32; ++j) t[j] = oz_i2d(v[j]);
#pragma unroll 1
  for (int L = OZ_S - 2; L >= 0; --L) {
    tc_ld32(ta + (uint32_t)(L * OZ_BN), v);
    tc_wait_ld();
#pragma unroll
    for (int j = 0; j < 32; ++j) t[j] = fma(t[j], 0.00390625, oz_i2d(v[j]));
  }
}

__global__ void __launch_bounds__(192, 1)
    oz_syrk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int nunits,
                   int ntiles, int nJ, int fullgrid, int64_t rps, int64_t nrp, double* __restrict__ Gpart) {
  extern __shared__ uint8_t oz_raw[];
  uint8_t* st = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(st + OZ_STAGES * OZ_STAGE_BYTES);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* tfull = empty + OZ_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < OZ_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    fence_mbar_init();
  }
  if (warp == 1) tc_alloc<512>(tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tbase;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      int64_t it = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        int I, J;
        if (fullgrid) {
          I = (u % ntiles) / nJ;
          J = (u % ntiles) % nJ;
        } else {
          oz_tile(u % ntiles, nJ, I, J);
        }
        const int64_t k0 = (int64_t)(u / ntiles) * rps, k1 = min(nrp, k0 + rps);
        for (int64_t k = k0; k < k1; k += OZ_BK, ++it) {
          const int s = (int)(it % OZ_STAGES);
          if (it >= OZ_STAGES) mbar_wait(&empty[s], (uint32_t)(((it / OZ_STAGES) - 1) & 1));
          uint8_t* a = st + s * OZ_STAGE_BYTES;
          mbar_expect_tx(&full[s], OZ_STAGE_BYTES);
          tma_load_4d(a, &tmA, 0, I * OZ_BM, 0, (int)(k / OZ_BK), &full[s]);
          tma_load_4d(a + OZ_A_BYTES, &tmB, 0, J * OZ_BN, 0, (int)(k / OZ_BK), &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    int64_t it = 0;
    int ul = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++ul) {
      const int64_t k0 = (int64_t)(u / ntiles) * rps, k1 = min(nrp, k0 + rps);
      if (ul > 0) mbar_wait(tempty, (uint32_t)((ul - 1) & 1));  // the epilogue has drained the last unit
      tc_fence_after();
      for (int64_t k = k0; k < k1; k += OZ_BK, ++it) {
        const int s = (int)(it % OZ_STAGES);
        mbar_wait(&full[s], (uint32_t)((it / OZ_STAGES) & 1));
        tc_fence_after();
        if (lane == 0) {
          oz_issue_stage(tmem, smem_u32(st + s * OZ_STAGE_BYTES), k == k0);
          tc_commit(&empty[s]);
          if (k + OZ_BK >= k1) tc_commit(tfull);
        }
        __syncwarp();
      }
    }
  } else {
    const int q = warp & 3;  // the TMEM lane quarter this warp may read
    const int row = q * 32 + lane;
    int ul = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++ul) {
      mbar_wait(tfull, (uint32_t)(ul & 1));
      tc_fence_after();
      double* out = Gpart + ((size_t)u * OZ_BM + row) * OZ_BN;
#pragma unroll 1
      for (int h = 0; h < OZ_BN / 32; ++h) {
        double t[32];
        oz_drain32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * 32), t);
#pragma unroll
        for (int j = 0; j < 32; j += 2) *reinterpret_cast<double2*>(out + h * 32 + j) = make_double2(t[j], t[j + 1]);
      }
      tc_fence_before();
      mbar_arrive(tempty);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tc_free<512>(tmem);
}

// G[a][b] (a < M, b < N) = 2^(e_a + e_b - 14) sum over the row splits (fixed order); full: every tile of the
// nI x nJ grid (C = A^T B), else the lower tiles of the SYRK (oz_tile)
__global__ void oz_reduce_kernel(const double* __restrict__ Gpart, int ntiles, int nsplit, int nJ, int full, int M,
                                 int N, const unsigned long long* __restrict__ cmaxA,
                                 const unsigned long long* __restrict__ cmaxB, const int* __restrict__ flag,
                                 double* __restrict__ G, int64_t ldg, int accumulate) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)ntiles * OZ_BM * OZ_BN) return;
  const int t = (int)(e / (OZ_BM * OZ_BN));
  const int i = (int)((e / OZ_BN) % OZ_BM), j = (int)(e % OZ_BN);
  int I, J;
  if (full) {
    I = t / nJ;
    J = t % nJ;
  } else {
    oz_tile(t, nJ, I, J);
  }
  const int a = I * OZ_BM + i, b = J * OZ_BN + j;
  if (a >= M || b >= N) return;
  double s = 0.0;
  for (int sp = 0; sp < nsplit; ++sp) s += Gpart[(((size_t)sp * ntiles + t) * OZ_BM + i) * OZ_BN + j];
  double v = ldexp(s, oz_exp(cmaxA[a]) + oz_exp(cmaxB[b]) - 14);
  if (*flag) v = __longlong_as_double(0x7ff8000000000000LL);
  G[(size_t)a * ldg + b] = accumulate ? G[(size_t)a * ldg + b] + v : v;
}

// ================================================================== K1 on the integer tensor cores
// U_aug[i][j] = sum_{k <= j} S[p][k] Linv[j][k] (reading c4), S = K(X, Z) with i = row(p):
// both operands are split per ROW (of S: position p; of Linv: output column j) -- the scale factors then
// sit outside the k sum: U = 2^(e_p + e_j - 14) sum_L acc_L 2^(-8L).

// K1a: one warp per position.  Pass 1 finds the row's smallest scaled distance t2 to the inducing points
// (2D + 1 operations per column, no exponential): the row maximum of S is the covariance at that distance,
// which fixes the row's scale e_p before any value is formed.  Pass 2 evaluates S and writes the digit
// slices Ss[kb][q][pos][k mod 32] straight from registers: lane l evaluates the four consecutive columns
// 128t + 4l + j (one 4-byte store per slice), reading Z from a permuted table (column b at 128 (b/128) +
// 32 (b%4) + (b%128)/4, so the lanes of a step read consecutive entries; padding columns sit at 1e100 and
// evaluate to 0).  Also writes the y column and the zero pad columns of U_aug (as kx_eval does).
template <int FAM, int D>
__global__ void __launch_bounds__(256) kx_slice_kernel(const double* __restrict__ X, const double* __restrict__ Z,
                                                       const double* __restrict__ y, int64_t n, int64_t npos,
                                                       int64_t chunk, int world, int rank, int64_t pos0, int m,
                                                       int mk, int KP, CovParams p, int8_t* __restrict__ Ss,
                                                       int64_t kbA, int* __restrict__ erow,
                                                       double* __restrict__ Uaug, int ld) {
  extern __shared__ double kxs_sm[];  // KPr x D, permuted
  __shared__ double tbl[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KPr = (KP + 127) & ~127;
  double* zs = kxs_sm;
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  double sc[D];
#pragma unroll
  for (int k = 0; k < D; ++k) sc[k] = fam_scale<FAM>() * p.inv_ls[k];
  for (int b = threadIdx.x; b < KPr; b += blockDim.x) {
    const int q = (b & ~127) + 32 * (b & 3) + ((b & 127) >> 2);
#pragma unroll
    for (int k = 0; k < D; ++k) zs[q * D + k] = b < m ? Z[b * D + k] * sc[k] : 1e100;
  }
  __syncthreads();
  auto cov_t2 = [&](double t2) -> double {
    if (FAM == FAM_GAUSS) return sig2_exp_neg(t2, tbl);
    const double t = sqrt_fast(t2);
    const double E = sig2_exp_neg(t, tbl);
    return FAM == FAM_M12 ? E : (FAM == FAM_M32 ? fma(E, t, E) : fma(E, fma(t2, 1.0 / 3.0, t), E));
  };
  for (int64_t pos = (int64_t)blockIdx.x * 8 + warp; pos < npos; pos += (int64_t)gridDim.x * 8) {
    const int64_t i = pos_to_row(pos0 + pos, chunk, world, rank);
    if (i >= n) continue;  // padding position: its output rows are never written
    double x[D];
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = X[i * D + k] * sc[k];
    auto dist2 = [&](int q) -> double {
      const double* z = zs + q * D;
      const double d0 = x[0] - z[0];
      double t2 = d0 * d0;
#pragma unroll
      for (int k = 1; k < D; ++k) {
        const double dk = x[k] - z[k];
        t2 = fma(dk, dk, t2);
      }
      return t2;
    };
    // the four consecutive columns 128 t + 4 lane + j (values v[j]) as 7 digit slices, one 4-byte store each
    auto emit = [&](int t, const double (&v)[4], double scl) {
      uint32_t lo[4], hi[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const long long Y = __double2ll_rn(v[j] * scl) + 0x808080808080LL;
        lo[j] = (uint32_t)Y;
        hi[j] = (uint32_t)((unsigned long long)Y >> 32);
      }
      const int b0 = 128 * t + 4 * lane;
      if (b0 >= KP) return;
      // row-block-major: [R][kb][q][128 rows][32 B] -- a row block's slices are one contiguous 7 x 4 KB x kb run
      int8_t* dst = Ss + ((((pos >> 7) * kbA + (b0 >> 5)) * OZ_S) * OZ_BM + (pos & 127)) * OZ_BK + (b0 & 31);
#pragma unroll
      for (int q = 1; q < OZ_S; ++q) {
        const int j = 6 - q;
        const uint32_t* src = j < 4 ? lo : hi;
        const uint32_t sel = (uint32_t)((j & 3) | (((j & 3) + 4) << 4));
        const uint32_t xx = __byte_perm(src[0], src[1], sel), yy = __byte_perm(src[2], src[3], sel);
        *reinterpret_cast<uint32_t*>(dst + q * OZ_BM * OZ_BK) = __byte_perm(xx, yy, 0x5410) ^ 0x80808080u;
      }
      {
        const uint32_t xx = __byte_perm(hi[0], hi[1], 0x62), yy = __byte_perm(hi[2], hi[3], 0x62);
        *reinterpret_cast<uint32_t*>(dst) = __byte_perm(xx, yy, 0x5410);
      }
    };
    if (KPr <= 512) {
      // <= 512 columns: the 16 scaled squared distances of pass 1 stay in registers for pass 2
      double t2c[16];
      double t2min = 1e300;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        t2c[u] = 32 * u < KPr ? dist2(lane + 32 * u) : 1e300;
        t2min = fmin(t2min, t2c[u]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t2min = fmin(t2min, __shfl_xor_sync(0xffffffffu, t2min, o));
      const int er = oz_exp((unsigned long long)__double_as_longlong(cov_t2(t2min)));
      if (lane == 0) erow[pos] = er;
      const double scl = ldexp(1.0, 55 - er);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (128 * t < KPr) {
          double v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = cov_t2(t2c[4 * t + j]);
          emit(t, v, scl);
        }
      }
    } else {
      double t2min = 1e300;
#pragma unroll 4
      for (int q = lane; q < KPr; q += 32) t2min = fmin(t2min, dist2(q));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t2min = fmin(t2min, __shfl_xor_sync(0xffffffffu, t2min, o));
      const double rmax = cov_t2(t2min);  // the covariance decreases with the distance
      const int er = oz_exp((unsigned long long)__double_as_longlong(rmax));
      if (lane == 0) erow[pos] = er;
      const double scl = ldexp(1.0, 55 - er);
      for (int t = 0; t < KPr / 128; ++t) {
        double v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = cov_t2(dist2(128 * t + 32 * j + lane));
        emit(t, v, scl);
      }
    }
    {
      double* urow = Uaug + i * (int64_t)ld;
      for (int c = mk + lane; c < ld; c += 32) urow[c] = (c == mk) ? y[i] : 0.0;
    }
  }
}


// rows of a general row-major matrix A (M x K, lda) -> digit slices with a per-row scale, in the row-block-major
// layout of the K1 GEMM ([R][kb][q][128 rows][32 B], R = row / 128) and e_r in erow (INT_MAX: the row holds a
// non-finite value -- the GEMM then writes NaN for it); one warp per row, two passes over the row (the second
// from L1/L2): the maximum, then four consecutive columns per lane packed into one 4-byte store per slice
__global__ void __launch_bounds__(256) oz_rowslice_kernel(const double* __restrict__ A, int64_t lda, int64_t M,
                                                          int K, int KP, int8_t* __restrict__ out,
                                                          int* __restrict__ erow) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kbA = KP / OZ_BK;
  for (int64_t r = (int64_t)blockIdx.x * 8 + warp; r < M; r += (int64_t)gridDim.x * 8) {
    const double* a = A + r * lda;
    double mx = 0.0;
    bool bad = false;
    for (int b = lane; b < K; b += 32) {
      const double v = a[b];
      bad |= !isfinite(v);
      mx = fmax(mx, fabs(v));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad = __any_sync(0xffffffffu, bad);
    const int er = oz_exp((unsigned long long)__double_as_longlong(mx));
    if (lane == 0) erow[r] = bad ? 0x7fffffff : er;
    const double scl = bad ? 0.0 : ldexp(1.0, 55 - er);
    for (int b0 = 4 * lane; b0 < KP; b0 += 128) {
      uint32_t lo[4], hi[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double v = b0 + j < K ? a[b0 + j] : 0.0;
        const long long Y = __double2ll_rn(v * scl) + 0x808080808080LL;
        lo[j] = (uint32_t)Y;
        hi[j] = (uint32_t)((unsigned long long)Y >> 32);
      }
      int8_t* dst = out + ((((r >> 7) * kbA + (b0 >> 5)) * OZ_S) * OZ_BM + (r & 127)) * OZ_BK + (b0 & 31);
#pragma unroll
      for (int q = 1; q < OZ_S; ++q) {
        const int j = 6 - q;
        const uint32_t* src = j < 4 ? lo : hi;
        const uint32_t sel = (uint32_t)((j & 3) | (((j & 3) + 4) << 4));
        const uint32_t xx = __byte_perm(src[0], src[1], sel), yy = __byte_perm(src[2], src[3], sel);
        *reinterpret_cast<uint32_t*>(dst + q * OZ_BM * OZ_BK) = __byte_perm(xx, yy, 0x5410) ^ 0x80808080u;
      }
      {
        const uint32_t xx = __byte_perm(hi[0], hi[1], 0x62), yy = __byte_perm(hi[2], hi[3], 0x62);
        *reinterpret_cast<uint32_t*>(dst) = __byte_perm(xx, yy, 0x5410);
      }
    }
  }
}

// The same for rows of <= 128 NCH columns, one read: lane l loads columns 128 t + 4 l .. + 3 of every 128-column
// block t (16-byte loads; a warp instruction covers 1 KB contiguous), all NCH x 4 values stay in registers for
// the maximum and the digit split, and every load of the row is issued before the first is used
template <int NCH>
__global__ void __launch_bounds__(256) oz_rowslice_reg_kernel(const double* __restrict__ A, int64_t lda, int64_t M,
                                                              int K, int KP, int8_t* __restrict__ out,
                                                              int* __restrict__ erow) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kbA = KP / OZ_BK;
  for (int64_t r = (int64_t)blockIdx.x * 8 + warp; r < M; r += (int64_t)gridDim.x * 8) {
    const double* a = A + r * lda;
    double v[NCH][4];
#pragma unroll
    for (int t = 0; t < NCH; ++t) {
      const int b0 = 128 * t + 4 * lane;
      if (b0 + 3 < K) {
        const double2 x = __ldcs(reinterpret_cast<const double2*>(a + b0));
        const double2 y = __ldcs(reinterpret_cast<const double2*>(a + b0 + 2));
        v[t][0] = x.x; v[t][1] = x.y; v[t][2] = y.x; v[t][3] = y.y;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[t][j] = b0 + j < K ? a[b0 + j] : 0.0;
      }
    }
    double mx = 0.0;
    bool bad = false;
#pragma unroll
    for (int t = 0; t < NCH; ++t)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bad |= !isfinite(v[t][j]);
        mx = fmax(mx, fabs(v[t][j]));
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad = __any_sync(0xffffffffu, bad);
    const int er = oz_exp((unsigned long long)__double_as_longlong(mx));
    if (lane == 0) erow[r] = bad ? 0x7fffffff : er;
    const double scl = bad ? 0.0 : ldexp(1.0, 55 - er);
#pragma unroll
    for (int t = 0; t < NCH; ++t) {
      const int b0 = 128 * t + 4 * lane;
      if (b0 >= KP) continue;
      uint32_t lo[4], hi[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const long long Y = __double2ll_rn(v[t][j] * scl) + 0x808080808080LL;
        lo[j] = (uint32_t)Y;
        hi[j] = (uint32_t)((unsigned long long)Y >> 32);
      }
      int8_t* dst = out + ((((r >> 7) * kbA + (b0 >> 5)) * OZ_S) * OZ_BM + (r & 127)) * OZ_BK + (b0 & 31);
#pragma unroll
      for (int q = 1; q < OZ_S; ++q) {
        const int j = 6 - q;
        const uint32_t* src = j < 4 ? lo : hi;
        const uint32_t sel = (uint32_t)((j & 3) | (((j & 3) + 4) << 4));
        const uint32_t xx = __byte_perm(src[0], src[1], sel), yy = __byte_perm(src[2], src[3], sel);
        *reinterpret_cast<uint32_t*>(dst + q * OZ_BM * OZ_BK) = __byte_perm(xx, yy, 0x5410) ^ 0x80808080u;
      }
      {
        const uint32_t xx = __byte_perm(hi[0], hi[1], 0x62), yy = __byte_perm(hi[2], hi[3], 0x62);
        *reinterpret_cast<uint32_t*>(dst) = __byte_perm(xx, yy, 0x5410);
      }
    }
  }
}

// rows of a small row-major matrix A (nrows x ncols, lda) -> digit slices out[kb][q][r][k mod 32] for
// r < nrows_p, k < 32 nkb (zeros outside A), with the per-row scale 2^e_r in rscale[r]; one warp per row
__global__ void __launch_bounds__(256) oz_rows_slice_kernel(const double* __restrict__ A, int64_t lda, int nrows,
                                                            int ncols, int nrows_p, int nkb, int8_t* __restrict__ out,
                                                            double* __restrict__ rscale) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + warp;
  if (r >= nrows_p) return;
  const int KP = nkb * OZ_BK;
  double mx = 0.0;
  bool bad = false;
  for (int b = lane; b < KP; b += 32)
    if (r < nrows && b < ncols) {
      const double v = A[(int64_t)r * lda + b];
      bad |= !isfinite(v);
      mx = fmax(mx, fabs(v));
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  bad = __any_sync(0xffffffffu, bad);
  const int er = oz_exp((unsigned long long)__double_as_longlong(mx));
  if (lane == 0) rscale[r] = bad ? __longlong_as_double(0x7ff8000000000000LL) : ldexp(1.0, er);
  const double scl = bad ? 0.0 : ldexp(1.0, 55 - er);
  for (int b = lane; b < KP; b += 32) {
    const double v = (r < nrows && b < ncols) ? A[(int64_t)r * lda + b] : 0.0;
    long long X = __double2ll_rn(v * scl);
    int8_t* dst = out + (((int64_t)(b >> 5) * OZ_S) * nrows_p + r) * OZ_BK + (b & 31);
#pragma unroll
    for (int q = OZ_S - 1; q >= 1; --q) {
      int d = (int)(X & 255);
      d -= (d & 128) << 1;
      dst[(int64_t)q * nrows_p * OZ_BK] = (int8_t)d;
      X = (X - d) >> 8;
    }
    dst[0] = (int8_t)X;
  }
}

// 16 accumulator columns, all 7 levels: the 7 TMEM loads are in flight together (one wait)
__device__ __forceinline__ void oz_drain16(uint32_t ta, double (&t)[16]) {
  uint32_t v[OZ_S][16];
#pragma unroll
  for (int L = 0; L < OZ_S; ++L) tc_ld16(ta + (uint32_t)(L * OZ_BN), v[L]);
  tc_wait_ld();
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    double a = oz_i2d(v[OZ_S - 1][j]);
#pragma unroll
    for (int L = OZ_S - 2; L >= 0; --L) a = fma(a, 0.00390625, oz_i2d(v[L][j]));
    t[j] = a;
  }
}

// K1b: persistent; unit = a row block R of 128 positions with all its column tiles J = nJ-1 .. 0 (every unit
// has the same triangular work, and the row block's A slices stay in L2 from tile to tile); per tile the
// k-blocks 0 .. kend(J) - 1; epilogue scales by 2^(e_p - 14) * 2^(e_j) and
// writes U_aug rows (global row of each position) for columns j < ncols_out.
__global__ void __launch_bounds__(64 + 32 * OZ_GEPI, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int nR, int nJ,
                   int kbmax, int tri, const int* __restrict__ erow, const double* __restrict__ cscale,
                   double* __restrict__ Uaug, int ld, int64_t n, int64_t chunk, int world, int rank, int64_t pos0,
                   int64_t npos, int ncols_out) {
  extern __shared__ uint8_t oz_raw[];
  uint8_t* st = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(st + OZ_STAGES * OZ_STAGE_BYTES);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* tfull = empty + OZ_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < OZ_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 32 * OZ_GEPI);
    fence_mbar_init();
  }
  if (warp == 1) tc_alloc<512>(tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tbase;
  const int nunits = nR;  // unit = one row block, all its column tiles (largest first): A stays in L2 between tiles
  auto kend = [&](int J) { return tri ? min(kbmax, 2 * J + 2) : kbmax; };

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      int64_t it = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int R = u;
        for (int J = nJ - 1; J >= 0; --J) {
          for (int kb = 0; kb < kend(J); ++kb, ++it) {
            const int s = (int)(it % OZ_STAGES);
            if (it >= OZ_STAGES) mbar_wait(&empty[s], (uint32_t)(((it / OZ_STAGES) - 1) & 1));
            uint8_t* a = st + s * OZ_STAGE_BYTES;
            mbar_expect_tx(&full[s], OZ_STAGE_BYTES);
            tma_load_4d(a, &tmA, 0, 0, 0, R * kbmax + kb, &full[s]);
            tma_load_4d(a + OZ_A_BYTES, &tmB, 0, J * OZ_BN, 0, kb, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    int64_t it = 0;
    int tl = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      for (int J = nJ - 1; J >= 0; --J) {
        if (tl > 0) mbar_wait(tempty, (uint32_t)((tl - 1) & 1));
        tc_fence_after();
        const int ke = kend(J);
        for (int kb = 0; kb < ke; ++kb, ++it) {
          const int s = (int)(it % OZ_STAGES);
          mbar_wait(&full[s], (uint32_t)((it / OZ_STAGES) & 1));
          tc_fence_after();
          if (lane == 0) {
            oz_issue_stage(tmem, smem_u32(st + s * OZ_STAGE_BYTES), kb == 0);
            tc_commit(&empty[s]);
            if (kb + 1 == ke) tc_commit(tfull);
          }
          __syncwarp();
        }
        ++tl;
      }
    }
  } else {
    const int q = warp & 3;              // TMEM lane quarter (rows q*32 ..)
    const int hh = (warp - 2) >> 2;      // column half of every tile this warp drains
    const int row = q * 32 + lane;
    double* stg = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(tbase) + 256) + (size_t)(warp - 2) * 32 * OZ_GLD;
    int tl = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int R = u;
      const int64_t pos = (int64_t)R * OZ_BM + row;
      int64_t i = n;
      double rs = 0.0;
      if (pos < npos) {
        i = pos_to_row(pos0 + pos, chunk, world, rank);
        const int er = erow[pos];
        rs = er == 0x7fffffff ? __longlong_as_double(0x7ff8000000000000LL) : ldexp(1.0, er - 14);
      }
      for (int J = nJ - 1; J >= 0; --J) {
        mbar_wait(tfull, (uint32_t)(tl & 1));
        tc_fence_after();
        double t[2][16];
        oz_drain16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(hh * 32), t[0]);
        oz_drain16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(hh * 32 + 16), t[1]);
        tc_fence_before();
        mbar_arrive(tempty);  // TMEM read: the MMA warp may start the next tile
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
          for (int j = 0; j < 16; ++j) stg[lane * OZ_GLD + j] = t[c][j] * rs;
          __syncwarp();
          // two rows per step: lanes 0-15 row r, 16-31 row r + 1, 16 consecutive columns (128 B) each
          const int jc = J * OZ_BN + hh * 32 + c * 16 + (lane & 15);
          const double cs = jc < ncols_out ? cscale[jc] : 0.0;
#pragma unroll 4
          for (int r = 0; r < 32; r += 2) {
            const int rr = r + (lane >> 4);
            const int64_t pr = (int64_t)R * OZ_BM + q * 32 + rr;
            const int64_t ir = __shfl_sync(0xffffffffu, i, rr);
            if (pr < npos && ir < n && jc < ncols_out) __stcs(Uaug + ir * (int64_t)ld + jc, stg[rr * OZ_GLD + (lane & 15)] * cs);
          }
          __syncwarp();
        }
        ++tl;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tc_free<512>(tmem);
}

// ------------------------------------------------------------------ host
namespace {
struct OzPlan {
  int nI, nJ, ntiles, nsplit;
  int64_t ncp, nrp, rps;
};

OzPlan oz_plan(int ncols, int64_t nrows, int sms, int ncolsB = 0) {
  OzPlan P{};
  P.nI = (ncols + OZ_BM - 1) / OZ_BM;
  P.nJ = ((ncolsB > 0 ? ncolsB : ncols) + OZ_BN - 1) / OZ_BN;
  P.ntiles = ncolsB > 0 ? P.nI * P.nJ : oz_ntiles(P.nI, P.nJ);
  P.ncp = (int64_t)P.nI * OZ_BM;
  P.nrp = std::max<int64_t>(OZ_TROWS, (nrows + OZ_TROWS - 1) / OZ_TROWS * OZ_TROWS);
  // row splits of <= OZ_CHUNK rows (multiples of OZ_BK); among 1-2x the minimum count, the smallest makespan
  // (waves of `sms` units x rows per unit)
  const int64_t smin = (P.nrp + OZ_CHUNK - 1) / OZ_CHUNK;
  double best = 1e300;
  for (int64_t ns = smin; ns <= 2 * smin; ++ns) {
    int64_t rps = (P.nrp + ns - 1) / ns;
    rps = (rps + OZ_BK - 1) / OZ_BK * OZ_BK;
    const int64_t nsp = (P.nrp + rps - 1) / rps;
    const int64_t units = nsp * P.ntiles;
    const double cost = (double)((units + sms - 1) / sms) * (double)rps;
    if (cost < best * (1.0 - 1e-9)) {
      best = cost;
      P.nsplit = (int)nsp;
      P.rps = rps;
    }
  }
  return P;
}
}  // namespace

bool syrk_i8_supported(int ncols) { return ncols >= 1 && ncols <= 4096; }

size_t syrk_i8_ws_bytes(int ncols, int64_t cap_rows) {
  const OzPlan P = oz_plan(ncols, cap_rows, 148);
  return (size_t)OZ_S * P.ncp * P.nrp;
}

// every chunk of <= cap_rows rows plans at most 2 x its minimum split count (oz_plan)
size_t syrk_i8_part_doubles(int ncols, int64_t cap_rows) {
  const OzPlan P = oz_plan(ncols, cap_rows, 148);
  const int64_t smin = (P.nrp + OZ_CHUNK - 1) / OZ_CHUNK;
  return (size_t)(2 * smin) * P.ntiles * OZ_BM * OZ_BN;
}

size_t syrk_i8_aux_bytes(int ncols) { return (size_t)((ncols + 127) / 128 * 128) * 8 + 256; }

cudaError_t launch_syrk_i8(const double* W, int64_t ldw, int64_t nrows, int ncols, int8_t* ws, int64_t cap_rows,
                           double* Gpart, void* aux, double* G, int ldg, int sms, cudaStream_t s,
                           const unsigned long long* cmax64) {
  if (!syrk_i8_supported(ncols) || cap_rows < 1 || (ldw & 1) || (reinterpret_cast<uintptr_t>(W) & 15))
    return cudaErrorInvalidValue;
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(aux);
  const int ncp0 = (ncols + 127) / 128 * 128;
  int* flag = reinterpret_cast<int*>(cmax + ncp0);
  cudaError_t e = cudaMemsetAsync(aux, 0, syrk_i8_aux_bytes(ncols), s);
  if (e != cudaSuccess) return e;
  if (cmax64) {
    // the column maxima came with the rows (the vecchia W pass): fold the 64 copies
    oz_colmax_fold_kernel<<<(ncols + 255) / 256, 256, 0, s>>>(cmax64, ncols, cmax);
  } else if (nrows > 0) {
    const int ctas = 4 * sms;
    const int64_t rpc = (nrows + ctas - 1) / ctas;
    oz_colmax_kernel<<<(unsigned)((nrows + rpc - 1) / rpc), 256, 0, s>>>(W, ldw, nrows, ncols, rpc, cmax);
  }
  e = smem_optin(oz_syrk_kernel, OZ_SMEM);
  if (e != cudaSuccess) return e;
  int64_t done = 0;
  int chunk = 0;
  do {
    const int64_t rows = std::min<int64_t>(cap_rows, nrows - done);
    const OzPlan P = oz_plan(ncols, rows, sms);
    dim3 gs((unsigned)(P.nrp / OZ_TROWS), (unsigned)(P.ncp / 64));
    oz_slice_kernel<<<gs, 256, 0, s>>>(W + (size_t)done * ldw, ldw, rows, ncols, cmax, ws, P.ncp, flag);
    CUtensorMap ta, tb;
    e = make_tmap_i8_slices(&ta, ws, (uint64_t)(P.nrp / OZ_BK), (uint64_t)P.ncp, OZ_S, OZ_BM);
    if (e != cudaSuccess) return e;
    e = make_tmap_i8_slices(&tb, ws, (uint64_t)(P.nrp / OZ_BK), (uint64_t)P.ncp, OZ_S, OZ_BN);
    if (e != cudaSuccess) return e;
    const int units = P.nsplit * P.ntiles;
    oz_syrk_kernel<<<std::min(units, sms), 192, OZ_SMEM, s>>>(ta, tb, units, P.ntiles, P.nJ, 0, P.rps, P.nrp, Gpart);
    const int64_t tot = (int64_t)P.ntiles * OZ_BM * OZ_BN;
    oz_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(Gpart, P.ntiles, P.nsplit, P.nJ, 0, ncols, ncols,
                                                                   cmax, cmax, flag, G, ldg, chunk > 0);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    done += rows;
    ++chunk;
  } while (done < nrows);
  return cudaSuccess;
}

// ------------------------------------------------------------------ K1 host
bool ufeat_i8_supported(int d, int mk) { return (d == 2 || d == 3 || d == 5 || d == 10) && mk >= 8 && mk <= 4096; }

static int64_t k1_nposp(int64_t rows) { return std::max<int64_t>(OZ_BM, (rows + OZ_BM - 1) / OZ_BM * OZ_BM); }
static int k1_kb(int mk) { return (mk + OZ_BK - 1) / OZ_BK; }
static int k1_nJ(int mk) { return (mk + OZ_BN - 1) / OZ_BN; }

size_t ufeat_i8_ws_bytes(int mk, int64_t cap_rows) { return (size_t)OZ_S * k1_nposp(cap_rows) * k1_kb(mk) * OZ_BK; }

size_t ufeat_i8_aux_bytes(int mk, int64_t cap_rows) {
  const size_t lsl = (size_t)OZ_S * k1_nJ(mk) * OZ_BN * k1_kb(mk) * OZ_BK;  // Linv slices
  return (lsl + 255) / 256 * 256 + (size_t)k1_nJ(mk) * OZ_BN * 8 + (size_t)k1_nposp(cap_rows) * 4 + 512;
}

cudaError_t launch_u_features_i8(const double* X, const double* Z, const double* y, int64_t n, int64_t pos0,
                                 int64_t npos, int64_t chunk, int world, int rank, int m, int mk, const CovParams& p,
                                 const double* Linv, double* Uaug, int ld, int8_t* ws, int64_t cap_rows, void* aux,
                                 int sms, cudaStream_t s) {
  if (!ufeat_i8_supported(p.d, mk) || cap_rows < 1) return cudaErrorInvalidValue;
  if (npos <= 0) return cudaSuccess;
  const int kb = k1_kb(mk), nJ = k1_nJ(mk), KP = kb * OZ_BK;
  char* a = reinterpret_cast<char*>(aux);
  int8_t* lsl = reinterpret_cast<int8_t*>(a);
  const size_t lsl_b = ((size_t)OZ_S * nJ * OZ_BN * KP + 255) / 256 * 256;
  double* cscale = reinterpret_cast<double*>(a + lsl_b);
  int* erow = reinterpret_cast<int*>(a + lsl_b + (size_t)nJ * OZ_BN * 8);
  // B: the rows of Linv (output columns j), once per call
  oz_rows_slice_kernel<<<(nJ * OZ_BN + 7) / 8, 256, 0, s>>>(Linv, mk, mk, mk, nJ * OZ_BN, kb, lsl, cscale);
  CUtensorMap tb;
  cudaError_t e = make_tmap_i8_slices(&tb, lsl, (uint64_t)kb, (uint64_t)nJ * OZ_BN, OZ_S, OZ_BN);
  if (e != cudaSuccess) return e;
  e = smem_optin(oz_gemm_kernel, OZ_GEMM_SMEM);
  if (e != cudaSuccess) return e;
  const size_t kx_smem = (size_t)((KP + 127) / 128 * 128) * p.d * 8;
  for (int64_t c0 = 0; c0 < npos; c0 += cap_rows) {
    const int64_t rows = std::min<int64_t>(cap_rows, npos - c0);
    const int64_t nposp = k1_nposp(rows);
    auto go = [&](auto kern) -> cudaError_t {
      cudaError_t e1 = smem_optin(kern, kx_smem);
      if (e1 != cudaSuccess) return e1;
      int per_sm = 0;  // one full wave of resident blocks (the rows are grid-strided)
      e1 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, kx_smem);
      if (e1 != cudaSuccess) return e1;
      const int nb = (int)std::min<int64_t>((rows + 7) / 8, (int64_t)sms * std::max(per_sm, 1));
      kern<<<nb, 256, kx_smem, s>>>(X, Z, y, n, rows, chunk, world, rank, pos0 + c0, m, mk, KP, p, ws, (int64_t)kb,
                                    erow, Uaug, ld);
      return cudaGetLastError();
    };
#define VIF_KXS(DV)                                                 \
  switch (p.family) {                                               \
    case FAM_M12: e = go(kx_slice_kernel<FAM_M12, DV>); break;      \
    case FAM_M32: e = go(kx_slice_kernel<FAM_M32, DV>); break;      \
    case FAM_M52: e = go(kx_slice_kernel<FAM_M52, DV>); break;      \
    default: e = go(kx_slice_kernel<FAM_GAUSS, DV>); break;         \
  }
    if (p.d == 2) {
      VIF_KXS(2)
    } else if (p.d == 3) {
      VIF_KXS(3)
    } else if (p.d == 5) {
      VIF_KXS(5)
    } else {
      VIF_KXS(10)
    }
#undef VIF_KXS
    if (e != cudaSuccess) return e;
    CUtensorMap ta;
    e = make_tmap_i8_slices(&ta, ws, (uint64_t)kb * (nposp / OZ_BM), (uint64_t)OZ_BM, OZ_S, OZ_BM);
    if (e != cudaSuccess) return e;
    const int nR = (int)(nposp / OZ_BM);
    const int units = nR;
    oz_gemm_kernel<<<std::min(units, sms), 64 + 32 * OZ_GEPI, OZ_GEMM_SMEM, s>>>(ta, tb, nR, nJ, kb, 1, erow, cscale, Uaug, ld, n, chunk,
                                                               world, rank, pos0 + c0, rows, mk);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}


// ------------------------------------------------------------------ general C = A B^T on the integer tensor cores
size_t gemm_i8_ws_bytes(int K, int64_t cap_rows) { return (size_t)OZ_S * k1_nposp(cap_rows) * k1_kb(K) * OZ_BK; }

size_t gemm_i8_aux_bytes(int N, int K, int64_t cap_rows) { return ufeat_i8_aux_bytes(std::max(N, K), cap_rows); }

cudaError_t launch_gemm_tn_i8(const double* A, int64_t lda, int64_t M, const double* B, int64_t ldb, int N, int K,
                              int tri, double* C, int64_t ldc, int8_t* ws, int64_t cap_rows, void* aux, int sms,
                              cudaStream_t s) {
  if (N < 1 || K < 1 || N > 4096 || K > 4096 || cap_rows < 1) return cudaErrorInvalidValue;
  if (M <= 0) return cudaSuccess;
  const int kb = k1_kb(K), nJ = k1_nJ(N), KP = kb * OZ_BK;
  char* a = reinterpret_cast<char*>(aux);
  int8_t* bsl = reinterpret_cast<int8_t*>(a);
  const size_t bsl_b = ((size_t)OZ_S * nJ * OZ_BN * KP + 255) / 256 * 256;
  double* cscale = reinterpret_cast<double*>(a + bsl_b);
  int* erow = reinterpret_cast<int*>(a + bsl_b + (size_t)nJ * OZ_BN * 8);
  oz_rows_slice_kernel<<<(nJ * OZ_BN + 7) / 8, 256, 0, s>>>(B, ldb, N, K, nJ * OZ_BN, kb, bsl, cscale);
  CUtensorMap tb;
  cudaError_t e = make_tmap_i8_slices(&tb, bsl, (uint64_t)kb, (uint64_t)nJ * OZ_BN, OZ_S, OZ_BN);
  if (e != cudaSuccess) return e;
  e = smem_optin(oz_gemm_kernel, OZ_GEMM_SMEM);
  if (e != cudaSuccess) return e;
  for (int64_t c0 = 0; c0 < M; c0 += cap_rows) {
    const int64_t rows = std::min<int64_t>(cap_rows, M - c0);
    const int64_t nposp = k1_nposp(rows);
    const int nb = (int)std::min<int64_t>((rows + 7) / 8, (int64_t)sms * 8);
    // rows of <= 512 columns from registers in one read (16-byte loads need lda even and A 16-byte aligned)
    const bool reg = KP <= 512 && (lda & 1) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
    if (reg && KP <= 256)
      oz_rowslice_reg_kernel<2><<<nb, 256, 0, s>>>(A + c0 * lda, lda, rows, K, KP, ws, erow);
    else if (reg)
      oz_rowslice_reg_kernel<4><<<nb, 256, 0, s>>>(A + c0 * lda, lda, rows, K, KP, ws, erow);
    else
      oz_rowslice_kernel<<<nb, 256, 0, s>>>(A + c0 * lda, lda, rows, K, KP, ws, erow);
    CUtensorMap ta;
    e = make_tmap_i8_slices(&ta, ws, (uint64_t)kb * (nposp / OZ_BM), (uint64_t)OZ_BM, OZ_S, OZ_BM);
    if (e != cudaSuccess) return e;
    const int nR = (int)(nposp / OZ_BM);
    // identity row map: pos_to_row(p, chunk = rows, world = 1, rank = 0) = p
    oz_gemm_kernel<<<std::min(nR, sms), 64 + 32 * OZ_GEPI, OZ_GEMM_SMEM, s>>>(
        ta, tb, nR, nJ, kb, tri, erow, cscale, C + c0 * ldc, (int)ldc, rows, rows, 1, 0, 0, rows, N);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ------------------------------------------------------------------ C = A^T B over rows on the integer tensor cores
// A: nrows x M (lda), B: nrows x N (ldb); C (M x N, ldc).  Per-column scales of A and B (global over the rows),
// digit slices of both in ws (rows in chunks so that both fit), the SYRK kernel over every (128 x 64) tile,
// reduction with the two exponent sets.
size_t gemm_tt_i8_aux_bytes(int M, int N) {
  return (size_t)((M + 127) / 128 * 128 + (N + 127) / 128 * 128) * 8 + 256;
}

size_t gemm_tt_i8_part_doubles(int M, int N, int64_t chunk_rows) {
  const OzPlan P = oz_plan(M, chunk_rows, 148, N);
  const int64_t smin = (P.nrp + OZ_CHUNK - 1) / OZ_CHUNK;
  return (size_t)(2 * smin) * P.ntiles * OZ_BM * OZ_BN;
}

// rows per chunk so that the slices of A and B fit ws_bytes
int64_t gemm_tt_i8_chunk(int M, int N, size_t ws_bytes) {
  const int64_t ncpA = (M + 127) / 128 * 128, ncpB = (N + 127) / 128 * 128;
  int64_t c = (int64_t)(ws_bytes / ((size_t)OZ_S * (ncpA + ncpB)));
  c = c / OZ_TROWS * OZ_TROWS;
  return c;
}

cudaError_t launch_gemm_tt_i8(const double* A, int64_t lda, int M, const double* B, int64_t ldb, int N, int64_t nrows,
                              double* C, int64_t ldc, int8_t* ws, size_t ws_bytes, double* Gpart, void* aux, int sms,
                              cudaStream_t s) {
  if (M < 1 || N < 1 || M > 4096 || N > 4096 || (lda & 1) || (ldb & 1) ||
      (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15))
    return cudaErrorInvalidValue;
  const int64_t crows = gemm_tt_i8_chunk(M, N, ws_bytes);
  if (crows < OZ_TROWS) return cudaErrorInvalidValue;
  const int ncpA = (M + 127) / 128 * 128, ncpB = (N + 127) / 128 * 128;
  unsigned long long* cmaxA = reinterpret_cast<unsigned long long*>(aux);
  unsigned long long* cmaxB = cmaxA + ncpA;
  int* flag = reinterpret_cast<int*>(cmaxB + ncpB);
  cudaError_t e = cudaMemsetAsync(aux, 0, gemm_tt_i8_aux_bytes(M, N), s);
  if (e != cudaSuccess) return e;
  if (nrows > 0) {
    const int ctas = 4 * sms;
    const int64_t rpc = (nrows + ctas - 1) / ctas;
    oz_colmax_kernel<<<(unsigned)((nrows + rpc - 1) / rpc), 256, 0, s>>>(A, lda, nrows, M, rpc, cmaxA);
    oz_colmax_kernel<<<(unsigned)((nrows + rpc - 1) / rpc), 256, 0, s>>>(B, ldb, nrows, N, rpc, cmaxB);
  }
  e = smem_optin(oz_syrk_kernel, OZ_SMEM);
  if (e != cudaSuccess) return e;
  int64_t done = 0;
  int chunk = 0;
  do {
    const int64_t rows = std::min<int64_t>(crows, nrows - done);
    const OzPlan P = oz_plan(M, rows, sms, N);
    int8_t* wsB = ws + (size_t)OZ_S * ncpA * P.nrp;
    oz_slice_kernel<<<dim3((unsigned)(P.nrp / OZ_TROWS), (unsigned)(ncpA / 64)), 256, 0, s>>>(
        A + (size_t)done * lda, lda, rows, M, cmaxA, ws, ncpA, flag);
    oz_slice_kernel<<<dim3((unsigned)(P.nrp / OZ_TROWS), (unsigned)(ncpB / 64)), 256, 0, s>>>(
        B + (size_t)done * ldb, ldb, rows, N, cmaxB, wsB, ncpB, flag);
    CUtensorMap ta, tb;
    e = make_tmap_i8_slices(&ta, ws, (uint64_t)(P.nrp / OZ_BK), (uint64_t)ncpA, OZ_S, OZ_BM);
    if (e != cudaSuccess) return e;
    e = make_tmap_i8_slices(&tb, wsB, (uint64_t)(P.nrp / OZ_BK), (uint64_t)ncpB, OZ_S, OZ_BN);
    if (e != cudaSuccess) return e;
    const int units = P.nsplit * P.ntiles;
    oz_syrk_kernel<<<std::min(units, sms), 192, OZ_SMEM, s>>>(ta, tb, units, P.ntiles, P.nJ, 1, P.rps, P.nrp, Gpart);
    const int64_t tot = (int64_t)P.ntiles * OZ_BM * OZ_BN;
    oz_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(Gpart, P.ntiles, P.nsplit, P.nJ, 1, M, N, cmaxA,
                                                                   cmaxB, flag, C, ldc, chunk > 0);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    done += rows;
    ++chunk;
  } while (done < nrows);
  return cudaSuccess;
}


// ================================================================== neighbour search on the integer tensor cores
// vif_neighbors (readings c5-c7): the same exhaustive search as knn_kernel (k_knn.cu) with the
// Gram blocks u_Q u_C^T of the whitened features as exact int8 digit-slice products (reading c18): the rows of
// U are split per row (oz_rowslice), a CTA owns 128 consecutive queries and sweeps the candidate tiles of 64
// predecessors.  Warp 0 streams {32 k, 128 query rows, 7 slices} and {32 k, 64 candidate rows, 7 slices} TMA
// boxes through a 3-stage ring, warp 1 issues the 10 MMAs per stage into the 7 level accumulators (TMEM
// columns [64 L, 64 L + 64)), warps 2-5 (one thread per query = its TMEM lane) drain 16 candidates at a
// time, form rho_c = k(x_i, x_j) - u_i.u_j and the score |rho_c| / sqrt(rho_ii rho_jj) exactly as knn_kernel
// does (16 independent chains), and merge the few that beat the query's threshold (in increasing index: ties
// keep the lower index) into its sorted top-m_v list in shared memory.
namespace {
constexpr int KN_STAGES = 3;
constexpr int KN_Q = 128, KN_C = 64;
constexpr int KN_MAXMV = 47;
}  // namespace

// shared memory of the variant: ST ring stages, NH = EW / 4 partial lists per query, the tile's candidates
static size_t knn_i8_smem(int mv, int EW, int ST) {
  return (size_t)ST * OZ_STAGE_BYTES + 1024 + 256 + (size_t)(EW / 4) * KN_Q * mv * (sizeof(double) + sizeof(int)) +
         8 + (size_t)KN_C * (VIF_MAX_D + 2) * sizeof(double);
}

template <int FAM, int EW, int ST, int DD = 0>
__global__ void __launch_bounds__(64 + 32 * EW, 1)
    knn_i8_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmC, int kbmax,
                  const int* __restrict__ erow, const double* __restrict__ X, int64_t n, CovParams p,
                  const double* __restrict__ isd, const int* __restrict__ deg, int mv, int32_t* __restrict__ out,
                  int qoff, int qstride) {
  extern __shared__ uint8_t oz_raw[];
  uint8_t* st = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_raw) + 1023) & ~uintptr_t(1023));
  constexpr int NH = EW / 4;  // epilogue warps per TMEM lane quarter: each takes 64 / NH candidates of a tile
  constexpr int CW = KN_C / NH;
  uint64_t* full = reinterpret_cast<uint64_t*>(st + ST * OZ_STAGE_BYTES);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + KN_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(tempty + 1);
  double* lv = reinterpret_cast<double*>(st + ST * OZ_STAGE_BYTES + 256);  // [NH][KN_Q][mv] list scores
  int* li = reinterpret_cast<int*>(lv + NH * KN_Q * mv);                     // [NH][KN_Q][mv] list indices
  double* xc = reinterpret_cast<double*>(li + ((NH * KN_Q * mv + 1) & ~1));  // [KN_C][VIF_MAX_D]
  double* isc = xc + KN_C * VIF_MAX_D;                                             // [KN_C]
  double* esc = isc + KN_C;                                                        // [KN_C] 2^e_j
  __shared__ double tbl[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nq = (n + KN_Q - 1) / KN_Q;
  const int64_t qb = nq - 1 - (qoff + (int64_t)qstride * blockIdx.x);  // longest sweeps first
  const int64_t q0 = qb * KN_Q;
  const int64_t qe = q0 + KN_Q < n ? q0 + KN_Q : n;
  const int ntile = (int)((qe - 1 + KN_C - 1) / KN_C);  // candidates j < i <= min(q0 + 127, n - 1)
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  if (threadIdx.x == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 32 * EW);
    fence_mbar_init();
  }
  if (warp == 1) tc_alloc<512>(tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tbase;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmC);
      int64_t it = 0;
      for (int t = 0; t < ntile; ++t)
        for (int kb = 0; kb < kbmax; ++kb, ++it) {
          const int s = (int)(it % ST);
          if (it >= ST) mbar_wait(&empty[s], (uint32_t)(((it / ST) - 1) & 1));
          uint8_t* a = st + s * OZ_STAGE_BYTES;
          mbar_expect_tx(&full[s], OZ_STAGE_BYTES);
          tma_load_4d(a, &tmQ, 0, 0, 0, (int)(qb * kbmax + kb), &full[s]);
          tma_load_4d(a + OZ_A_BYTES, &tmC, 0, (t & 1) * KN_C, 0, (t >> 1) * kbmax + kb, &full[s]);
        }
    }
  } else if (warp == 1) {
    int64_t it = 0;
    for (int t = 0; t < ntile; ++t) {
      if (t > 0) mbar_wait(tempty, (uint32_t)((t - 1) & 1));
      tc_fence_after();
      for (int kb = 0; kb < kbmax; ++kb, ++it) {
        const int s = (int)(it % ST);
        mbar_wait(&full[s], (uint32_t)((it / ST) & 1));
        tc_fence_after();
        if (lane == 0) {
          oz_issue_stage(tmem, smem_u32(st + s * OZ_STAGE_BYTES), kb == 0);
          tc_commit(&empty[s]);
          if (kb + 1 == kbmax) tc_commit(tfull);
        }
        __syncwarp();
      }
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter
    const int r = q * 32 + lane, et = threadIdx.x - 64;  // query row of the block; epilogue thread
    const int hh = (warp - 2) >> 2;                       // which CW candidates of every tile
    const int64_t i = q0 + r;
    const int d = DD > 0 ? DD : p.d;  // d = 2 as a compile-time constant: coordinates in registers
    double xq[VIF_MAX_D];
#pragma unroll
    for (int k = 0; k < VIF_MAX_D; ++k)
      xq[k] = (k < d && i < n) ? X[i * d + k] * (fam_scale<FAM>() * p.inv_ls[k]) : 0.0;
    const double isq = i < n ? isd[i] : 0.0;
    const bool dgq = i < n && deg[i] != 0;
    const double eq = i < n ? ldexp(1.0, erow[i] - 14) : 0.0;
    const double inv_fs2 = 1.0 / (fam_scale<FAM>() * fam_scale<FAM>());
    double* v = lv + (hh * KN_Q + r) * mv;
    int* ix = li + (hh * KN_Q + r) * mv;
    int k = 0;
    double thr = -INFINITY;
    for (int t = 0; t < ntile; ++t) {
      const int64_t c0 = (int64_t)t * KN_C;
      asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");  // the previous tile's candidates no longer read
      for (int e = et; e < KN_C * d; e += 32 * EW) {
        const int c = e / d, kk = e % d;
        xc[c * VIF_MAX_D + kk] = c0 + c < n ? X[(c0 + c) * d + kk] * (fam_scale<FAM>() * p.inv_ls[kk]) : 0.0;
      }
      if (et < KN_C) {
        const int64_t j = c0 + et;
        isc[et] = j < n ? isd[j] : 0.0;
        esc[et] = j < n ? ldexp(1.0, erow[j]) : 0.0;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");  // xc, isc, esc of this tile visible
      mbar_wait(tfull, (uint32_t)(t & 1));
      tc_fence_after();
#pragma unroll 1
      for (int h = hh * (CW / 16); h < (hh + 1) * (CW / 16); ++h) {
        double g[16];
        oz_drain16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * 16), g);
        if (h + 1 == (hh + 1) * (CW / 16)) {
          tc_fence_before();
          mbar_arrive(tempty);  // TMEM read: the MMA warp may start the next tile
        }
        // the 16 scores as independent chains (ILP)
        double sc[16];
        {
          double t2[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const double d0 = xq[0] - xc[(h * 16 + jj) * VIF_MAX_D];
            t2[jj] = d0 * d0;
          }
          for (int kk = 1; kk < d; ++kk)
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const double dk = xq[kk] - xc[(h * 16 + jj) * VIF_MAX_D + kk];
              t2[jj] = fma(dk, dk, t2[jj]);
            }
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const int c = h * 16 + jj;
            double cv;
            if (FAM == FAM_GAUSS) {
              cv = sig2_exp_neg(t2[jj], tbl);
            } else {
              const double tt = sqrt_fast(t2[jj]);
              const double E = sig2_exp_neg(tt, tbl);
              cv = FAM == FAM_M12 ? E : (FAM == FAM_M32 ? fma(E, tt, E) : fma(E, fma(t2[jj], 1.0 / 3.0, tt), E));
            }
            const double uu = g[jj] * eq * esc[c];
            sc[jj] = dgq ? -t2[jj] * inv_fs2 : (isc[c] == 0.0 ? 0.0 : fabs(cv - uu) * isq * isc[c]);
          }
        }
        // candidates that can enter the list at the current threshold (it only rises): usually none once the
        // list is full; the rest in increasing index order, unrolled so the scores stay in registers
        unsigned msk = 0;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int64_t j = c0 + h * 16 + jj;
          if (j < i && i < n && (k < mv || sc[jj] > thr)) msk |= 1u << jj;
        }
        if (msk) {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const double scj = sc[jj];
            if (((msk >> jj) & 1u) && (k < mv || scj > thr)) {
              int pos = k < mv ? k : mv - 1;
              while (pos > 0 && scj > v[pos - 1]) {
                v[pos] = v[pos - 1];
                ix[pos] = ix[pos - 1];
                --pos;
              }
              v[pos] = scj;
              ix[pos] = (int)(c0 + h * 16 + jj);
              if (k < mv) ++k;
              thr = k < mv ? -INFINITY : v[mv - 1];
            }
          }
        }
      }
    }
    if constexpr (NH == 1) {
      if (i < n)
        for (int kk = 0; kk < mv; ++kk) out[i * mv + kk] = kk < k ? ix[kk] : -1;
    } else {
      // two partial lists per query (candidates 0..31 and 32..63 of every tile), each sorted by (score desc,
      // index asc): merged by the first half's thread, equal scores taking the smaller index
      __shared__ int kcnt[2][KN_Q];
      kcnt[hh][r] = k;
      asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
      if (hh == 0 && i < n) {
        const double* va = lv + r * mv;
        const int* xa = li + r * mv;
        const double* vb = lv + (KN_Q + r) * mv;
        const int* xb = li + (KN_Q + r) * mv;
        const int ka = kcnt[0][r], kb2 = kcnt[1][r];
        int pa = 0, pb = 0;
        for (int kk = 0; kk < mv; ++kk) {
          int o = -1;
          if (pa < ka && pb < kb2) {
            const bool ta = va[pa] > vb[pb] || (va[pa] == vb[pb] && xa[pa] < xb[pb]);
            o = ta ? xa[pa++] : xb[pb++];
          } else if (pa < ka) {
            o = xa[pa++];
          } else if (pb < kb2) {
            o = xb[pb++];
          }
          out[i * mv + kk] = o;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tc_free<512>(tmem);
}

bool knn_i8_supported(int mv, int64_t n) { return mv >= 1 && mv <= KN_MAXMV && n >= 2; }

size_t knn_i8_ws_bytes(int mk, int64_t n) {
  return (size_t)OZ_S * (size_t)((n + OZ_BM - 1) / OZ_BM * OZ_BM) * (size_t)k1_kb(mk) * OZ_BK;
}

// U (n x mk, ldu; rows in the processing order) -> per-row digit slices in ws, exponents in erow (n ints), then the
// search; isd / deg as knn_kernel's resvar pass writes them (launch_knn_resvar)
cudaError_t launch_knn_i8(const double* U, int64_t ldu, int mk, const double* X, int64_t n, const CovParams& p,
                          const double* isd, const int* deg, int mv, int32_t* out, int8_t* ws, int* erow, int sms,
                          cudaStream_t s, int qoff, int qstride) {
  if (!knn_i8_supported(mv, n) || mk < 1) return cudaErrorInvalidValue;
  const int kb = k1_kb(mk), KP = kb * OZ_BK;
  const int64_t nposp = (n + OZ_BM - 1) / OZ_BM * OZ_BM;
  const int nb = (int)std::min<int64_t>((n + 7) / 8, (int64_t)sms * 8);
  const bool reg = KP <= 512 && (ldu & 1) == 0 && (reinterpret_cast<uintptr_t>(U) & 15) == 0;
  if (reg && KP <= 256)
    oz_rowslice_reg_kernel<2><<<nb, 256, 0, s>>>(U, ldu, n, mk, KP, ws, erow);
  else if (reg)
    oz_rowslice_reg_kernel<4><<<nb, 256, 0, s>>>(U, ldu, n, mk, KP, ws, erow);
  else
    oz_rowslice_kernel<<<nb, 256, 0, s>>>(U, ldu, n, mk, KP, ws, erow);
  // rows n .. nposp - 1 of the last block hold stale digits: their queries and candidates are masked
  CUtensorMap tq, tc;
  cudaError_t e = make_tmap_i8_slices(&tq, ws, (uint64_t)kb * (nposp / OZ_BM), (uint64_t)OZ_BM, OZ_S, OZ_BM);
  if (e != cudaSuccess) return e;
  e = make_tmap_i8_slices(&tc, ws, (uint64_t)kb * (nposp / OZ_BM), (uint64_t)OZ_BM, OZ_S, KN_C);
  if (e != cudaSuccess) return e;
  const int64_t nq = (n + KN_Q - 1) / KN_Q;
  if (qoff >= nq) return cudaGetLastError();
  const unsigned grid = (unsigned)((nq - qoff + qstride - 1) / qstride);
  // 8 epilogue warps (two per TMEM lane quarter, each scoring half of every tile into its own partial lists) and
  // a 2-stage ring when their lists fit beside it; else 4 epilogue warps and 3 stages (VIF_KNN_EW=4 forces it)
  static const char* ew_env = getenv("VIF_KNN_EW");
  const bool wide = knn_i8_smem(mv, 8, 2) <= 227 * 1024 && !(ew_env && ew_env[0] == '4');
  auto go = [&](auto kern, int ew, int stg) -> cudaError_t {
    const size_t smem = knn_i8_smem(mv, ew, stg);
    cudaError_t e1 = smem_optin(kern, smem);
    if (e1 != cudaSuccess) return e1;
    kern<<<grid, 64 + 32 * ew, smem, s>>>(tq, tc, kb, erow, X, n, p, isd, deg, mv, out, qoff, qstride);
    return cudaGetLastError();
  };
#define VIF_KNNI8(F)                                                                               \
  (wide ? (p.d == 2 ? go(knn_i8_kernel<F, 8, 2, 2>, 8, 2) : go(knn_i8_kernel<F, 8, 2>, 8, 2))      \
        : (p.d == 2 ? go(knn_i8_kernel<F, 4, KN_STAGES, 2>, 4, KN_STAGES)                          \
                    : go(knn_i8_kernel<F, 4, KN_STAGES>, 4, KN_STAGES)))
  switch (p.family) {
    case FAM_M12: return VIF_KNNI8(FAM_M12);
    case FAM_M32: return VIF_KNNI8(FAM_M32);
    case FAM_M52: return VIF_KNNI8(FAM_M52);
    default: return VIF_KNNI8(FAM_GAUSS);
  }
#undef VIF_KNNI8
}

}  // namespace vif
