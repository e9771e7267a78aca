// k_syrk.cu -- K4: G = [W r]^T [W r] over the rank's rows ("M"; whitened, reading c4).
//
// Tall-skinny FP64 DMMA SYRK.  The output is the (ld x ld) lower triangle in 64 x 64 tiles (ld = 512 at
// m = 500 -> 36 tiles); the rows are split into `nsplit` contiguous slabs (multiples of SK rows) and the
// grid is tiles x splits, sized to ONE wave of two CTAs per SM: every tile of a split reads the same
// rows at the same time, so each row of W leaves HBM about once and is served to the other tiles from
// L2.  Every CTA writes its partial tile; a deterministic reduction sums the splits in a fixed order.
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

__global__ void __launch_bounds__(32 * (NCONS + 1), SYRK_CTAS_PER_SM)
    syrk_tma_kernel(const __grid_constant__ CUtensorMap tmW, int64_t nrows, int ntiles, int64_t rows_per_split,
                    double* __restrict__ Gpart) {
  extern __shared__ uint8_t syrk_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(syrk_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + SS * 2 * SLAB);
  uint64_t* empty = full + SS;
  const int t = blockIdx.x % ntiles;
  const int split = blockIdx.x / ntiles;
  int I, J;
  tile_ij(t, I, J);
  const bool diag = I == J;
  const int64_t r0 = (int64_t)split * rows_per_split;
  int64_t r1 = r0 + rows_per_split;
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
          for (int b = 0; b < 4; ++b) tma_load_2d(a + SLAB + b * BOXB, &tmW, J * ST + 16 * b, row, &full[s]);
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

// G[a][b] (a >= b tile-wise) = sum over splits in order
__global__ void syrk_reduce_kernel(const double* __restrict__ Gpart, int ntiles, int nsplit, int ncols,
                                   double* __restrict__ G, int ldg) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)ntiles * ST * ST) return;
  const int t = (int)(e / (ST * ST));
  const int rc = (int)(e % (ST * ST));
  int I, J;
  tile_ij(t, I, J);
  const int a = I * ST + rc / ST, b = J * ST + rc % ST;
  if (a >= ncols || b >= ncols) return;
  double s = 0.0;
  for (int sp = 0; sp < nsplit; ++sp) s += Gpart[((size_t)sp * ntiles + t) * ST * ST + rc];
  G[(size_t)a * ldg + b] = s;
}

int syrk_ntiles(int ncols) {
  const int nt1 = (ncols + ST - 1) / ST;
  return nt1 * (nt1 + 1) / 2;
}

// Split count: the smallest with a last wave >= 97% full (time ~ waves / nsplit), else the best up to 64;
// never fewer than SK rows per split.
int syrk_nsplit(int ncols, int64_t nrows, int num_sms) {
  const int nt = syrk_ntiles(ncols);
  const int64_t slots = (int64_t)SYRK_CTAS_PER_SM * num_sms;
  const int64_t max_by_rows = (nrows + 4 * SK - 1) / (4 * SK);
  int64_t best = 1;
  double best_cost = 1e300;
  for (int64_t ns = 1; ns <= 64; ++ns) {
    const int64_t waves = (nt * ns + slots - 1) / slots;
    const double cost = (double)waves / (double)ns;
    const double fill = (double)(nt * ns) / (double)(waves * slots);
    if (cost < best_cost - 1e-12) {
      best_cost = cost;
      best = ns;
    }
    if (fill >= 0.97) {
      best = ns;
      break;
    }
  }
  if (best > max_by_rows) best = max_by_rows;
  if (best < 1) best = 1;
  return (int)best;
}

size_t syrk_part_doubles(int ncols, int nsplit) { return (size_t)syrk_ntiles(ncols) * nsplit * ST * ST; }

// partials only (the reduction over splits, and over rounds, is launch_syrk_reduce)
cudaError_t launch_syrk_part(const double* W, int64_t ldw, int64_t nrows, int ncols, int nsplit, double* Gpart,
                             cudaStream_t s) {
  const int nt = syrk_ntiles(ncols);
  if (nrows <= 0) return cudaMemsetAsync(Gpart, 0, syrk_part_doubles(ncols, nsplit) * sizeof(double), s);
  int64_t rps = (nrows + nsplit - 1) / nsplit;
  rps = (rps + SK - 1) / SK * SK;  // stages never straddle two splits
  CUtensorMap tm;
  cudaError_t e = make_tmap_f64(&tm, W, (uint64_t)nrows, (uint64_t)ncols, (uint64_t)ldw, SK);
  if (e != cudaSuccess) return e;
  e = smem_optin(syrk_tma_kernel, SYRK_SMEM);
  if (e != cudaSuccess) return e;
  syrk_tma_kernel<<<nt * nsplit, 32 * (NCONS + 1), SYRK_SMEM, s>>>(tm, nrows, nt, rps, Gpart);
  return cudaGetLastError();
}

cudaError_t launch_syrk_reduce(const double* Gpart, int ntiles, int nsplit_total, int ncols, double* G, int ldg,
                               cudaStream_t s) {
  const int64_t tot = (int64_t)ntiles * ST * ST;
  syrk_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(Gpart, ntiles, nsplit_total, ncols, G, ldg);
  return cudaGetLastError();
}

cudaError_t launch_syrk(const double* W, int64_t ldw, int64_t nrows, int ncols, int nsplit, double* Gpart,
                        double* G, int ldg, cudaStream_t s) {
  cudaError_t e = launch_syrk_part(W, ldw, nrows, ncols, nsplit, Gpart, s);
  if (e != cudaSuccess) return e;
  return launch_syrk_reduce(Gpart, syrk_ntiles(ncols), nsplit, ncols, G, ldg, s);
}

}  // namespace vif
