// k_syrk.cu -- K4: G = [W r]^T [W r] over the rank's rows ("M"; whitened, reading c4).
//
// Tall-skinny FP64 DMMA SYRK.  The output is the (ld x ld) lower triangle in 64 x 64 tiles (ld = 512 at
// m = 500 -> 36 tiles); the rows are split into contiguous slabs (multiples of SK rows) and the grid of
// (tile, split) items is sized to ONE wave of two CTAs per SM: every tile of a split reads the same rows at
// about the same time, so
// each row of W leaves HBM about once and is served to the other tiles from L2.  Every CTA writes its
// partial tile; a deterministic reduction sums the splits in a fixed order.
//
// Tile movement (Blackwell TMA): a producer warp streams the two 64-column slabs of W for the tile
// (one for a diagonal tile) through an SS-stage shared-memory ring with cp.async.bulk.tensor (boxes of
// 16 columns x SK rows, SWIZZLE_128B) completing on per-stage "full" mbarriers; four consumer warps
// (2 x 2 sub-tiles of 32 x 32) wait on "full", run the DMMAs and release the stage on its "empty"
// mbarrier.  No CTA-wide barrier in the main loop.
//
// Fragments.  With k = the row of W, both DMMA operands are "column c of the slab, row k": lane l of a
// mma.m8n8k4 fragment holds (c0 + l/4, k(l%4)).  Within an 8-row group the k-slots are permuted
// (rows {0,4,1,5} for the first k-step, {2,6,3,7} for the second -- the contraction is
// order-independent and both operands use the same order), so that under the 128-B swizzle the 32
// lanes of a fragment load cover every bank exactly twice (two wavefronts, conflict-free).
#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

#include <stdlib.h>

#include <algorithm>

namespace vif {

namespace {
constexpr int ST = 64;          // output tile
constexpr int SK = 32;          // rows per stage
constexpr int SS = 3;           // stages
constexpr int SYRK_CTAS_PER_SM = 2;
constexpr int BOXB = SK * 128;  // bytes of one 16-column box
constexpr int SLAB = 4 * BOXB;  // one 64-column slab per stage
constexpr int NCONS = 4;        // consumer warps
constexpr size_t SYRK_SMEM = (size_t)SS * 2 * SLAB + 1024 /* alignment */ + 2 * SS * 8;
}  // namespace

__device__ __forceinline__ void tile_ij(int t, int& I, int& J) {
  int i = 0;
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  I = i;
  J = t - i * (i + 1) / 2;
}

// ntc = 0: the SYRK (lower tiles of W^T W, tmW = tmB = W).  ntc > 0: the general C = A^T B over the same rows
// (tmW = A, tmB = B; every tile of an nt1 x ntc grid, so row splits each, no diagonal shortcut).
__global__ void __launch_bounds__(32 * (NCONS + 1), SYRK_CTAS_PER_SM)
    syrk_tma_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmB, int64_t nrows,
                    int nt1, int ntc, int sd, int so, int64_t rps_d, int64_t rps_o, double* __restrict__ Gpart) {
  extern __shared__ uint8_t syrk_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(syrk_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + SS * 2 * SLAB);
  uint64_t* empty = full + SS;
  // work items: the nt1 diagonal tiles x sd row splits first, then the off-diagonal tiles x so splits
  int I, J, split;
  int64_t rps;
  if (ntc > 0) {
    const int t = blockIdx.x / so;
    split = blockIdx.x % so;
    I = t / ntc;
    J = t % ntc;
    rps = rps_o;
  } else if ((int)blockIdx.x < nt1 * sd) {
    I = J = blockIdx.x / sd;
    split = blockIdx.x % sd;
    rps = rps_d;
  } else {
    const int o = blockIdx.x - nt1 * sd;
    const int to = o / so;  // off-diagonal tile number in row-major order of the strict lower triangle
    split = o % so;
    int i = 1;
    while (i * (i + 1) / 2 <= to) ++i;
    I = i;
    J = to - i * (i - 1) / 2;
    rps = rps_o;
  }
  const bool diag = ntc == 0 && I == J;
  const int64_t r0 = (int64_t)split * rps;
  int64_t r1 = r0 + rps;
  if (r1 > nrows) r1 = nrows;
  const int nkt = r0 < r1 ? (int)((r1 - r0 + SK - 1) / SK) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < SS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NCONS) {
    // ---------------- producer: one elected lane issues the TMA boxes of every stage ----------------
    if (lane == 0) {
      tma_prefetch_desc(&tmW);
      if (ntc > 0) tma_prefetch_desc(&tmB);
      const uint32_t bytes = diag ? SLAB : 2 * SLAB;
      for (int kt = 0; kt < nkt; ++kt) {
        const int s = kt % SS;
        if (kt >= SS) mbar_wait(&empty[s], ((kt / SS) + 1) & 1);
        mbar_expect_tx(&full[s], bytes);
        uint8_t* a = sm + s * 2 * SLAB;
        const int row = (int)(r0 + (int64_t)kt * SK);
#pragma unroll
        for (int b = 0; b < 4; ++b) tma_load_2d(a + b * BOXB, &tmW, I * ST + 16 * b, row, &full[s]);
        if (!diag) {
#pragma unroll
          for (int b = 0; b < 4; ++b)
            tma_load_2d(a + SLAB + b * BOXB, ntc > 0 ? &tmB : &tmW, J * ST + 16 * b, row, &full[s]);
        }
      }
    }
    return;
  }

  // ---------------- consumers: 2 x 2 warps of 32 x 32 ----------------
  const int wm = warp >> 1, wn = warp & 1;
  const bool active = !(diag && wn > wm);  // 32 x 32 sub-tile above the diagonal: nothing to compute
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // per-lane byte offsets of the fragments inside a stage: fragment q of the warp's 32 columns lives in
  // box (2 w + q / 2), columns (q & 1) * 8 + lane / 4; the k-slot t = lane % 4 of k-step h in an 8-row
  // group g reads row 8 g + 2 h + (t >> 1) + 4 (t & 1)
  const int tq = lane & 3, cl = lane >> 2;
  const int rsel = (tq >> 1) + ((tq & 1) << 2);  // row within the 8-row group for h = 0 (h = 1: + 2)
  uint32_t offA[4], offB[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    offA[q] = (uint32_t)((2 * wm + (q >> 1)) * BOXB) + swz_off(rsel, (q & 1) * 8 + cl);
    offB[q] = (uint32_t)((diag ? 0 : SLAB) + (2 * wn + (q >> 1)) * BOXB) + swz_off(rsel, (q & 1) * 8 + cl);
  }
  // rows 8 g + rsel + 2 h: the swizzle term depends on (row & 7) = rsel + 2h, so the h = 1 offset is
  // recomputed (not a constant shift)
  uint32_t offA1[4], offB1[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    offA1[q] = (uint32_t)((2 * wm + (q >> 1)) * BOXB) + swz_off(rsel + 2, (q & 1) * 8 + cl);
    offB1[q] = (uint32_t)((diag ? 0 : SLAB) + (2 * wn + (q >> 1)) * BOXB) + swz_off(rsel + 2, (q & 1) * 8 + cl);
  }

  const uint32_t sbase = smem_u32(sm);
  for (int kt = 0; kt < nkt; ++kt) {
    const int s = kt % SS;
    mbar_wait(&full[s], (kt / SS) & 1);
    if (active) {
      const uint32_t st = sbase + s * 2 * SLAB;
#pragma unroll
      for (int g = 0; g < SK / 8; ++g) {
        double af[4], bf[4], af1[4], bf1[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          af[q] = lds_f64(st + g * 1024 + offA[q]);
          bf[q] = lds_f64(st + g * 1024 + offB[q]);
          af1[q] = lds_f64(st + g * 1024 + offA1[q]);
          bf1[q] = lds_f64(st + g * 1024 + offB1[q]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af1[a], bf1[b]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  double* out = Gpart + (size_t)blockIdx.x * ST * ST;
  const int fr = lane >> 2, fcc = (lane & 3) * 2;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = wm * 32 + a * 8 + fr, c = wn * 32 + b * 8 + fcc;
      *reinterpret_cast<double2*>(out + r * ST + c) = make_double2(acc[a][b][0], acc[a][b][1]);
    }
}

// G[a][b] (a >= b tile-wise) = sum over the tile's work items in order, launch by launch (rounds)
__global__ void syrk_reduce_kernel(const double* __restrict__ Gpart, int nt1, int sd, int so, int nlaunch,
                                   int ncols, double* __restrict__ G, int ldg) {
  const int ntiles = nt1 * (nt1 + 1) / 2;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)ntiles * ST * ST) return;
  const int t = (int)(e / (ST * ST));
  const int rc = (int)(e % (ST * ST));
  int I, J;
  tile_ij(t, I, J);
  const int a = I * ST + rc / ST, b = J * ST + rc % ST;
  if (a >= ncols || b >= ncols) return;
  const int items = nt1 * sd + (ntiles - nt1) * so;
  const int first = I == J ? I * sd : nt1 * sd + (t - I) * so;  // t - I = off-diagonal tiles before t
  const int cnt = I == J ? sd : so;
  double s = 0.0;
  for (int l = 0; l < nlaunch; ++l)
    for (int k = 0; k < cnt; ++k) s += Gpart[((size_t)l * items + first + k) * ST * ST + rc];
  G[(size_t)a * ldg + b] = s;
}

int syrk_ntiles(int ncols) {
  const int nt1 = (ncols + ST - 1) / ST;
  return nt1 * (nt1 + 1) / 2;
}

// Split plan: `so` row splits per off-diagonal tile and sd(so) per diagonal tile (equal DMMA work per CTA),
// the largest so whose CTAs all fit one wave of SYRK_CTAS_PER_SM per SM; never fewer than 4 SK rows per split.
// The same number of splits for diagonal and off-diagonal tiles (measured at config 3, profiles/r02_notes.md:
// 8.35 ms; skipping the upper 8 x 8 blocks of the diagonal sub-tiles 8.79 ms; fewer, longer diagonal splits
// for equal work per CTA 10.5 ms -- the per-warp DMMA stream, not the CTA's total, sets the time)
static int syrk_diag_splits(int so) { return so; }

static int syrk_items(int ncols, int so) {
  const int nt1 = (ncols + ST - 1) / ST;
  return nt1 * syrk_diag_splits(so) + (nt1 * (nt1 - 1) / 2) * so;
}

int syrk_nsplit(int ncols, int64_t nrows, int num_sms) {
  // one wave if possible: the largest so whose items all fit (ld = 512: 36 tiles x 8 splits = 288 CTAs); else
  // the plan with the smallest makespan ~ waves x the per-CTA rows (so <= 64)
  const int64_t slots = (int64_t)SYRK_CTAS_PER_SM * num_sms;
  const int64_t max_by_rows = std::max<int64_t>(1, (nrows + 4 * SK - 1) / (4 * SK));
  if (syrk_items(ncols, 1) <= slots) {
    int best = 1;
    for (int so = 2; so <= 256 && so <= max_by_rows && syrk_items(ncols, so) <= slots; ++so) best = so;
    return best;
  }
  int best = 1;
  double best_cost = 1e300;
  for (int so = 1; so <= 64 && so <= max_by_rows; ++so) {
    const int64_t items = syrk_items(ncols, so);
    const double waves = (double)((items + slots - 1) / slots);
    const double cost = waves / so;
    if (cost < best_cost * (1.0 - 1e-9)) {
      best_cost = cost;
      best = so;
    }
  }
  return best;
}

size_t syrk_part_doubles(int ncols, int nsplit) { return (size_t)syrk_items(ncols, nsplit) * ST * ST; }

// partials only (the reduction over splits, and over rounds, is launch_syrk_reduce)
cudaError_t launch_syrk_part(const double* W, int64_t ldw, int64_t nrows, int ncols, int nsplit, double* Gpart,
                             cudaStream_t s) {
  const int nt1 = (ncols + ST - 1) / ST;
  const int so = nsplit, sd = syrk_diag_splits(so);
  if (nrows <= 0) return cudaMemsetAsync(Gpart, 0, syrk_part_doubles(ncols, nsplit) * sizeof(double), s);
  auto rps_of = [&](int ns) {
    int64_t r = (nrows + ns - 1) / ns;
    return (r + SK - 1) / SK * SK;  // stages never straddle two splits
  };
  CUtensorMap tm;
  cudaError_t e = make_tmap_f64(&tm, W, (uint64_t)nrows, (uint64_t)ncols, (uint64_t)ldw, SK);
  if (e != cudaSuccess) return e;
  e = smem_optin(syrk_tma_kernel, SYRK_SMEM);
  if (e != cudaSuccess) return e;
  syrk_tma_kernel<<<syrk_items(ncols, so), 32 * (NCONS + 1), SYRK_SMEM, s>>>(tm, tm, nrows, nt1, 0, sd, so, rps_of(sd),
                                                                             rps_of(so), Gpart);
  return cudaGetLastError();
}

cudaError_t launch_syrk_reduce(const double* Gpart, int ncols, int nsplit, int nlaunch, double* G, int ldg,
                               cudaStream_t s) {
  const int nt1 = (ncols + ST - 1) / ST;
  const int64_t tot = (int64_t)syrk_ntiles(ncols) * ST * ST;
  syrk_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(Gpart, nt1, syrk_diag_splits(nsplit), nsplit,
                                                                   nlaunch, ncols, G, ldg);
  return cudaGetLastError();
}

// C (M x N, ldc) = A^T B, A: nrows x M (lda), B: nrows x N (ldb): the tall-skinny contraction over rows
__global__ void gemm_tt_reduce_kernel(const double* __restrict__ part, int ntc, int so, int M, int N,
                                      double* __restrict__ C, int64_t ldc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nt1 = (M + ST - 1) / ST;
  if (e >= (int64_t)nt1 * ntc * ST * ST) return;
  const int t = (int)(e / (ST * ST)), rc = (int)(e % (ST * ST));
  const int a = (t / ntc) * ST + rc / ST, b = (t % ntc) * ST + rc % ST;
  if (a >= M || b >= N) return;
  double acc = 0.0;
  for (int k = 0; k < so; ++k) acc += part[((size_t)t * so + k) * ST * ST + rc];
  C[(size_t)a * ldc + b] = acc;
}

int gemm_tt_nsplit(int M, int N, int64_t nrows, int num_sms) {
  const int tiles = ((M + ST - 1) / ST) * ((N + ST - 1) / ST);
  const int64_t slots = (int64_t)SYRK_CTAS_PER_SM * num_sms;
  const int64_t max_by_rows = std::max<int64_t>(1, (nrows + 4 * SK - 1) / (4 * SK));
  int64_t so = std::max<int64_t>(1, slots / tiles);
  if (so > max_by_rows) so = max_by_rows;
  return (int)so;
}

size_t gemm_tt_part_doubles(int M, int N, int nsplit) {
  return (size_t)((M + ST - 1) / ST) * ((N + ST - 1) / ST) * nsplit * ST * ST;
}

cudaError_t launch_gemm_tt(const double* A, int64_t lda, int M, const double* B, int64_t ldb, int N, int64_t nrows,
                           int nsplit, double* part, double* C, int64_t ldc, cudaStream_t s) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const int nt1 = (M + ST - 1) / ST, ntc = (N + ST - 1) / ST;
  const int so = nsplit;
  if (nrows <= 0) {
    for (int a = 0; a < M; ++a) {
      cudaError_t e = cudaMemsetAsync(C + (size_t)a * ldc, 0, (size_t)N * sizeof(double), s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  int64_t rps = (nrows + so - 1) / so;
  rps = (rps + SK - 1) / SK * SK;
  CUtensorMap ta, tb;
  cudaError_t e = make_tmap_f64(&ta, A, (uint64_t)nrows, (uint64_t)M, (uint64_t)lda, SK);
  if (e != cudaSuccess) return e;
  e = make_tmap_f64(&tb, B, (uint64_t)nrows, (uint64_t)N, (uint64_t)ldb, SK);
  if (e != cudaSuccess) return e;
  e = smem_optin(syrk_tma_kernel, SYRK_SMEM);
  if (e != cudaSuccess) return e;
  syrk_tma_kernel<<<nt1 * ntc * so, 32 * (NCONS + 1), SYRK_SMEM, s>>>(ta, tb, nrows, nt1, ntc, so, so, rps, rps, part);
  const int64_t tot = (int64_t)nt1 * ntc * ST * ST;
  gemm_tt_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(part, ntc, so, M, N, C, ldc);
  return cudaGetLastError();
}

cudaError_t launch_syrk(const double* W, int64_t ldw, int64_t nrows, int ncols, int nsplit, double* Gpart,
                        double* G, int ldg, cudaStream_t s) {
  cudaError_t e = launch_syrk_part(W, ldw, nrows, ncols, nsplit, Gpart, s);
  if (e != cudaSuccess) return e;
  return launch_syrk_reduce(Gpart, ncols, nsplit, 1, G, ldg, s);
}

}  // namespace vif
