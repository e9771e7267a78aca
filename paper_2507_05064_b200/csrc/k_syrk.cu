// k_syrk.cu -- K4: G = [W r]^T [W r] over the rank's rows ("M"; whitened, reading c4).
//
// Tall-skinny FP64 DMMA SYRK: the output is the (ld x ld) lower triangle in 64 x 64 tiles
// (ld = 512 at m = 500 -> 36 tiles); rows are split into `nsplit` slabs so that
// tiles x splits fills the 148 SMs several times over; every CTA writes its partial tile and a
// deterministic reduction sums the splits in a fixed order (no atomics).
// The operands are row slabs of W (k = the row index), so both fragments are read from a
// [row][col] shared tile: lane l loads W[k0 + l%4][c0 + l/4].  Rows padded to 72 doubles
// (576 B = 64 mod 128 B): the 4 rows x 64 B a warp touches land on distinct banks.
#include "common.cuh"
#include "kernels.h"

namespace vif {

namespace {
// SK = 16: a 55 KB ring, four CTAs (16 warps) per SM
constexpr int ST = 64, SK = 16, SS = 3, SPAD = 72;
constexpr int SMINB = 4;
}

__device__ __forceinline__ void tile_ij(int t, int& I, int& J) {
  int i = 0;
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  I = i;
  J = t - i * (i + 1) / 2;
}

__global__ void __launch_bounds__(128, SMINB) syrk_kernel(const double* __restrict__ W, int64_t ldw, int64_t nrows,
                                                   int ncols, int ntiles, int64_t rows_per_split,
                                                   double* __restrict__ Gpart) {
  extern __shared__ __align__(16) double ssm[];
  double* As = ssm;                      // [SS][SK][SPAD]
  double* Bs = ssm + SS * SK * SPAD;     // [SS][SK][SPAD]
  const int t = blockIdx.x % ntiles;
  const int split = blockIdx.x / ntiles;
  int I, J;
  tile_ij(t, I, J);
  const bool diag = I == J;
  const int64_t r0 = (int64_t)split * rows_per_split;
  int64_t r1 = r0 + rows_per_split;
  if (r1 > nrows) r1 = nrows;
  const int nkt = r0 < r1 ? (int)((r1 - r0 + SK - 1) / SK) : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 1, wn = warp & 1;
  const int a0 = I * ST, b0 = J * ST;

  auto load_stage = [&](int st, int kt) {
    const int64_t k0 = r0 + (int64_t)kt * SK;
    double* as = As + st * SK * SPAD;
    double* bs = Bs + st * SK * SPAD;
#pragma unroll
    for (int j = 0; j < SK * 32 / 128; ++j) {  // SK rows x 32 chunks of 16 B
      const int e = tid + j * 128;
      const int r = e >> 5, c2 = (e & 31) * 2;
      const int64_t gr = k0 + r;
      const bool okr = gr < r1;
      {
        const bool ok = okr && a0 + c2 < ncols;
        cp_async16(as + r * SPAD + c2, ok ? W + gr * ldw + a0 + c2 : W, ok);
      }
      if (!diag) {
        const bool ok = okr && b0 + c2 < ncols;
        cp_async16(bs + r * SPAD + c2, ok ? W + gr * ldw + b0 + c2 : W, ok);
      }
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < SS - 1; ++s) {
    if (s < nkt) load_stage(s, s);
    cp_async_commit();
  }
  const int fk = lane & 3, fc = lane >> 2;
  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<SS - 2>();
    __syncthreads();
    {
      const int nk = kt + SS - 1;
      if (nk < nkt) load_stage(nk % SS, nk);
      cp_async_commit();
    }
    if (diag && wn > wm) continue;  // 32x32 sub-tile above the diagonal: nothing to compute
    const double* as = As + (kt % SS) * SK * SPAD + fk * SPAD + wm * 32 + fc;
    const double* bs = (diag ? As : Bs) + (kt % SS) * SK * SPAD + fk * SPAD + wn * 32 + fc;
#pragma unroll
    for (int kk = 0; kk < SK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) af[q] = as[kk * SPAD + q * 8];
#pragma unroll
      for (int q = 0; q < 4; ++q) bf[q] = bs[kk * SPAD + q * 8];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  cp_async_wait<0>();
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

int syrk_nsplit(int ncols, int64_t nrows, int num_sms) {
  const int nt = syrk_ntiles(ncols);
  const int64_t slots = (int64_t)SMINB * num_sms;      // CTAs resident at once
  const int64_t base = (4 * slots + nt - 1) / nt;      // >= ~4 waves
  const int64_t max_by_rows = (nrows + 255) / 256;     // at least 256 rows per split
  // pick the split count in [base, 2 base] whose last wave is fullest (no half-empty tail wave)
  int64_t best = base;
  double best_eff = 0.0;
  for (int64_t ns = base; ns <= 2 * base; ++ns) {
    const int64_t ctas = nt * ns;
    const double eff = (double)ctas / (double)(slots * ((ctas + slots - 1) / slots));
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = ns;
    }
    if (eff > 0.995) break;
  }
  int64_t ns = best;
  if (ns > max_by_rows) ns = max_by_rows;
  if (ns < 1) ns = 1;
  return (int)ns;
}

size_t syrk_part_doubles(int ncols, int nsplit) { return (size_t)syrk_ntiles(ncols) * nsplit * ST * ST; }

cudaError_t launch_syrk(const double* W, int64_t ldw, int64_t nrows, int ncols, int nsplit, double* Gpart,
                        double* G, int ldg, cudaStream_t s) {
  const int nt = syrk_ntiles(ncols);
  const int64_t rps = nrows > 0 ? (nrows + nsplit - 1) / nsplit : 0;
  const size_t smem = (size_t)2 * SS * SK * SPAD * sizeof(double);
  {
    cudaError_t e = smem_optin(syrk_kernel, smem);
    if (e != cudaSuccess) return e;
  }
  syrk_kernel<<<nt * nsplit, 128, smem, s>>>(W, ldw, nrows, ncols, nt, rps, Gpart);
  const int64_t tot = (int64_t)nt * ST * ST;
  syrk_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(Gpart, nt, nsplit, ncols, G, ldg);
  return cudaGetLastError();
}

// per-round SYRK partials only (the reduction over all rounds' splits is launch_syrk_reduce)
cudaError_t launch_syrk_part(const double* W, int64_t ldw, int64_t nrows, int ncols, int nsplit, double* Gpart,
                             cudaStream_t s) {
  const int nt = syrk_ntiles(ncols);
  const int64_t rps = nrows > 0 ? (nrows + nsplit - 1) / nsplit : 0;
  const size_t smem = (size_t)2 * SS * SK * SPAD * sizeof(double);
  {
    cudaError_t e = smem_optin(syrk_kernel, smem);
    if (e != cudaSuccess) return e;
  }
  syrk_kernel<<<nt * nsplit, 128, smem, s>>>(W, ldw, nrows, ncols, nt, rps, Gpart);
  return cudaGetLastError();
}

cudaError_t launch_syrk_reduce(const double* Gpart, int ntiles, int nsplit_total, int ncols, double* G, int ldg,
                               cudaStream_t s) {
  const int64_t tot = (int64_t)ntiles * ST * ST;
  syrk_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(Gpart, ntiles, nsplit_total, ncols, G, ldg);
  return cudaGetLastError();
}

}  // namespace vif
