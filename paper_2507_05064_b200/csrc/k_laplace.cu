// k_laplace.cu -- kernels of the VIF-Laplace iterative path (Sect. 3).
//
// Vectors are row-major n x ncol (ncol = 1 for the Newton solves, ell for the SLQ probes), rows by
// point index (the Vecchia order).  The latent factor B (unit lower triangular, B[i, N(i)] = -A_i),
// D and the whitened U come from the VIF factor with the error variance removed.
//
//   la_level_*    dependency levels of B / B^T (once per neighbour structure): sync-free, warp w
//                 takes rows w, w + W, ... in order, waits (flag polls) on the ready flags of the
//                 rows it depends on and publishes its own with a release store;
//   la_trsv_lvl   x = B^{-1} (s o v), y = B^{-T} u: level-scheduled cooperative solves (one grid
//                 barrier per level, rows bucketed and their entries stored in level order);
//   la_tsgemm     C = U^T diag(rs) V        tall-skinny split-row contraction (m x ncol), two-stage
//                                           deterministic reduction;
//   la_coldot ... per-column dot products (two-stage, fixed order), CG vector updates, FITC rows,
//                 the Newton step and the SLQ quadrature e_1^T log(T) e_1 (implicit QL on T).
//
// Static row assignment over resident warps makes the level pass deadlock-free: the smallest
// unfinished row (in solve order) always has its dependencies done.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace vif {

namespace {

// Flag polls are relaxed gpu-scope loads: ld.acquire.gpu compiles to LDG.STRONG + CCTL.IVALL, an L1
// invalidation per poll (ncu: 426M of them in one multi-column solve, 20x slower).  The data a flag
// guards is read with __ldcg (LDG.STRONG.GPU, L2) only after the poll loop has observed the flag: the
// load's issue is control-dependent on the flag value, and the writer's st.release.gpu made the row
// visible at L2 before the flag.
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int LA_THREADS = 256;
constexpr int LA_WARPS = LA_THREADS / 32;

// ------------------------------------------------------------------ transposed structure of B
__global__ void la_count_kernel(const int32_t* __restrict__ nbr, int64_t n, int mv, int* __restrict__ cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * mv; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = nbr[e];
    if (j >= 0) atomicAdd(cnt + j, 1);
  }
}

// exclusive scan of cnt (n) into ptr (n + 1); one block of 1024 threads, contiguous chunks
__global__ void __launch_bounds__(1024) la_scan_kernel(const int* __restrict__ cnt, int64_t n, int* __restrict__ ptr) {
  __shared__ int part[1024];
  const int t = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t b0 = t * per, b1 = b0 + per < n ? b0 + per : n;
  int s = 0;
  for (int64_t i = b0; i < b1; ++i) s += cnt[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int acc = 0;
    for (int k = 0; k < 1024; ++k) {
      const int v = part[k];
      part[k] = acc;
      acc += v;
    }
    ptr[n] = acc;
  }
  __syncthreads();
  int acc = part[t];
  for (int64_t i = b0; i < b1; ++i) {
    ptr[i] = acc;
    acc += cnt[i];
  }
}

__global__ void la_fill_kernel(const int32_t* __restrict__ nbr, int64_t n, int mv, const int* __restrict__ ptr,
                               int* __restrict__ cursor, int* __restrict__ tpos) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * mv; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = nbr[e];
    if (j >= 0) tpos[ptr[j] + atomicAdd(cursor + j, 1)] = (int)e;
  }
}

// sort each children list by entry index (= by child row): a deterministic gather order
__global__ void la_sort_kernel(int64_t n, const int* __restrict__ ptr, int* __restrict__ tpos) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int a = ptr[j], b = ptr[j + 1];
    for (int k = a + 1; k < b; ++k) {
      const int v = tpos[k];
      int q = k - 1;
      while (q >= a && tpos[q] > v) {
        tpos[q + 1] = tpos[q];
        --q;
      }
      tpos[q + 1] = v;
    }
  }
}

// ------------------------------------------------------------------ flag waits (level pass)
// A row waits (relaxed polls with back-off, see ld_relaxed) on the ready flags of the rows it depends on.
__device__ __forceinline__ void la_wait(const int* f, int epoch) {
  if (ld_relaxed(f) == epoch) return;
  unsigned ns = 8;
  while (ld_relaxed(f) != epoch) {
    __nanosleep(ns);
    ns = ns < 256 ? 2 * ns : 256;
  }
}

// The level-scheduled kernels read rows written in earlier levels with plain (weak) loads: grid.sync()
// orders them (and invalidates L1), and weak loads, unlike the strong __ldcg ones, may be reordered, so
// the unrolled loop below issues all of a chunk's gathers before the first FMA needs one.
// acc{0,1} += sum over the cnt (<= 32) entries (jl, bl) held by lanes 0..cnt-1 of b * x[j, c{0,1}]
__device__ __forceinline__ void la_gather_cols_weak(const double* x, int ncol, int c0, int jl, double bl, int cnt,
                                                    double& acc0, double& acc1) {
  const int c1 = c0 + 32;
  const int r0 = c0 < ncol ? c0 : ncol - 1, r1 = c1 < ncol ? c1 : ncol - 1;
  const bool ok = jl >= 0;  // selects, not branches: the shuffles below need a converged warp
  jl = ok ? jl : 0;
  bl = ok ? bl : 0.0;
  // the valid entries are a prefix of the lanes (neighbour lists are -1 padded at the end only; children
  // lists have no padding), so slot q is used iff q < lim
  const int lim = min(cnt, __popc(__ballot_sync(0xffffffffu, ok)));
  double x0[32], x1[32], bb[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    const int j = __shfl_sync(0xffffffffu, jl, q);
    const double bq = __shfl_sync(0xffffffffu, bl, q);
    bb[q] = q < lim ? bq : 0.0;
    // an unused slot loads row 0 (a safe address) and discards it: 0 x (a not yet written row) could be NaN
    const double* xr = x + (int64_t)j * ncol;
    const double a0 = xr[r0], a1 = xr[r1];
    x0[q] = q < lim ? a0 : 0.0;
    x1[q] = q < lim ? a1 : 0.0;
  }
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    acc0 = fma(bb[q], x0[q], acc0);
    acc1 = fma(bb[q], x1[q], acc1);
  }
}

// transposed values: trow[k] = tpos[k] / mv, tval[k] = Bc[tpos[k]]
__global__ void la_tvals_kernel(const int* __restrict__ tpos, int64_t nnz, int mv, const double* __restrict__ Bc,
                                int* __restrict__ trow, double* __restrict__ tval) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int e = tpos[k];
    trow[k] = e / mv;
    tval[k] = Bc[e];
  }
}

// ------------------------------------------------------------------ level-scheduled triangular solves
// Levels of the dependency DAG (once per neighbour structure): forward lev_i = 1 + max_{j in N(i)} lev_j,
// backward levb_j = 1 + max_{children i} levb_i, computed by the same sync-free scheme as above.
__global__ void __launch_bounds__(LA_THREADS) la_level_fwd_kernel(const int32_t* __restrict__ nbr, int mv, int64_t n,
                                                                  int* lev, int* flags, int epoch) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * LA_WARPS;
  for (int64_t i = (int64_t)blockIdx.x * LA_WARPS + (threadIdx.x >> 5); i < n; i += nw) {
    int l = 0;
    for (int p = lane; p < mv; p += 32) {
      const int j = nbr[i * mv + p];
      if (j >= 0) {
        la_wait(flags + j, epoch);
        l = max(l, __ldcg(lev + j) + 1);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l = max(l, __shfl_xor_sync(0xffffffffu, l, o));
    if (lane == 0) {
      __stcg(lev + i, l);
      st_release(flags + i, epoch);
    }
  }
}

__global__ void __launch_bounds__(LA_THREADS) la_level_bwd_kernel(const int* __restrict__ tptr,
                                                                  const int* __restrict__ trow, int64_t n, int* lev,
                                                                  int* flags, int epoch) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * LA_WARPS;
  for (int64_t t = (int64_t)blockIdx.x * LA_WARPS + (threadIdx.x >> 5); t < n; t += nw) {
    const int64_t j = n - 1 - t;
    int l = 0;
    for (int k = tptr[j] + lane; k < tptr[j + 1]; k += 32) {
      const int i = trow[k];
      la_wait(flags + i, epoch);
      l = max(l, __ldcg(lev + i) + 1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l = max(l, __shfl_xor_sync(0xffffffffu, l, o));
    if (lane == 0) {
      __stcg(lev + j, l);
      st_release(flags + j, epoch);
    }
  }
}

__global__ void la_max_kernel(const int* __restrict__ a, int64_t n, int* __restrict__ out) {
  int m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, a[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// bucket rows by level: order[lptr[L] .. lptr[L+1]) = rows of level L (any order inside a level)
__global__ void la_bucket_count_kernel(const int* __restrict__ key, int64_t n, int* __restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + key[i], 1);
}
__global__ void la_bucket_fill_kernel(const int* __restrict__ key, int64_t n, const int* __restrict__ ptr,
                                      int* __restrict__ cursor, int* __restrict__ order) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int L = key[i];
    order[ptr[L] + atomicAdd(cursor + L, 1)] = (int)i;
  }
}

// long rows (B^T rows of early points: up to hundreds of children): lanes over entries, 16 columns at
// a time in registers, summed over the lanes through shared memory; out of line so that it does not
// change the register allocation of the short-row path
__device__ __noinline__ void la_long_row(const double* x, int ncol, const int32_t* __restrict__ ecol,
                                         const double* __restrict__ eval, int k0, int k1, int lane,
                                         double (*red)[17], double* colsum, double& acc0, double& acc1) {
  for (int cb = 0; cb < ncol; cb += 16) {
    double a16[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) a16[c] = 0.0;
    const int cm = ncol - cb < 16 ? ncol - cb : 16;
    for (int k = k0 + lane; k < k1; k += 32) {
      const int j = ecol[k];
      const double b = j >= 0 ? eval[k] : 0.0;
      const double* xr = x + (int64_t)(j >= 0 ? j : 0) * ncol + cb;
      // a padding entry (j < 0) must not touch x: 0 x (a not yet written row) could be NaN
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const double xv = xr[c < cm ? c : 0];
        a16[c] = j >= 0 ? fma(b, xv, a16[c]) : a16[c];
      }
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) red[lane][c] = a16[c];
    __syncwarp();
    if (lane < cm) {
      double t = 0.0;
      for (int l = 0; l < 32; ++l) t += red[l][lane];
      colsum[cb + lane] = t;
    }
    __syncwarp();
  }
  acc0 = lane < ncol ? colsum[lane] : 0.0;
  acc1 = lane + 32 < ncol ? colsum[lane + 32] : 0.0;
  __syncwarp();
}

// Entries in level order, so that a row's entries are addressed by its level-sorted position q (no
// dependent load through the row index): forward ecol/eval[q*mv + p] = nbr/B[order[q]*mv + p];
// backward eptr2[q] = scan of children counts in order, ecol2/eval2 = trow/tval segments.
__global__ void la_reorder_fwd_kernel(const int* __restrict__ order, const int32_t* __restrict__ nbr,
                                      const double* __restrict__ Bc, int64_t n, int mv, int32_t* __restrict__ ecol,
                                      double* __restrict__ eval) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * mv; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / mv, p = e % mv;
    const int64_t src = (int64_t)order[q] * mv + p;
    ecol[e] = nbr[src];
    eval[e] = Bc[src];
  }
}
__global__ void la_seglen_kernel(const int* __restrict__ order, const int* __restrict__ tptr, int64_t n,
                                 int* __restrict__ cnt) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int r = order[q];
    cnt[q] = tptr[r + 1] - tptr[r];
  }
}
__global__ void la_reorder_bwd_kernel(const int* __restrict__ order, const int* __restrict__ tptr,
                                      const int* __restrict__ trow, const double* __restrict__ tval,
                                      const int* __restrict__ eptr2, int64_t n, int32_t* __restrict__ ecol,
                                      double* __restrict__ eval) {
  const int lane = threadIdx.x & 31;
  for (int64_t q = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); q < n;
       q += (int64_t)gridDim.x * (blockDim.x / 32)) {
    const int r = order[q];
    const int a = tptr[r], len = tptr[r + 1] - a, o = eptr2[q];
    for (int k = lane; k < len; k += 32) {
      ecol[o + k] = trow[a + k];
      eval[o + k] = tval[a + k];
    }
  }
}

// One cooperative kernel per solve: level by level (grid.sync between levels), a warp per row.
// Row r: out_r = s_r v_r - sum_k val[k] out[col[k]] over its entries k (forward: k = r*mv + p with
// col = N(r)_p, val = B[r,p], entries with col < 0 skipped; backward: k in [tptr[r], tptr[r+1]),
// col = trow, val = tval).  Reads of other rows go to L2 (__ldcg; rows written in earlier levels).
// A warp's first row of the next level does not depend on the current level: its index, its first 32
// entries and its right-hand side are loaded before the barrier, so after it only the gathers of
// x remain on the row's dependency chain.
struct LaRowPre {
  int64_t r;
  int k0, k1, jl;
  double bl, sr, v0, v1, w2r, u0, u1;
};

template <bool FWD>
__device__ __forceinline__ bool la_row_load(int q, int qend, const int* __restrict__ order,
                                            const int32_t* __restrict__ ecol, const double* __restrict__ eval,
                                            const int* __restrict__ eptr, int mv, int ncol,
                                            const double* __restrict__ v, const double* __restrict__ s,
                                            const double* __restrict__ v2, const double* __restrict__ w2, int lane,
                                            LaRowPre& o) {
  if (q >= qend) return false;
  o.r = order[q];
  o.k0 = FWD ? q * mv : eptr[q];
  o.k1 = FWD ? o.k0 + mv : eptr[q + 1];
  const int k = o.k0 + lane;
  o.jl = k < o.k1 ? ecol[k] : -1;
  o.bl = k < o.k1 ? eval[k] : 0.0;
  o.sr = s ? s[o.r] : 1.0;
  const int c0 = ncol == 1 ? 0 : lane, c1 = lane + 32;
  o.v0 = c0 < ncol ? v[o.r * ncol + c0] : 0.0;
  o.v1 = c1 < ncol ? v[o.r * ncol + c1] : 0.0;
  o.w2r = o.u0 = o.u1 = 0.0;
  if (v2 && w2) {  // only with out2 (the caller passes v2 = v even without the W^{-1} term)
    o.w2r = w2[o.r];
    o.u0 = c0 < ncol ? v2[o.r * ncol + c0] : 0.0;
    o.u1 = c1 < ncol ? v2[o.r * ncol + c1] : 0.0;
  }
  return true;
}

template <bool FWD>
__global__ void __launch_bounds__(LA_THREADS) la_trsv_lvl_kernel(
    const int* __restrict__ order, const int* __restrict__ lptr, int nlev, const int32_t* __restrict__ ecol,
    const double* __restrict__ eval, const int* __restrict__ eptr, int mv, int ncol, const double* __restrict__ v,
    const double* __restrict__ s, double* x, const double* __restrict__ v2, const double* __restrict__ w2,
    double* __restrict__ out2, int long_min, unsigned long long* dbg) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sm_red[LA_WARPS][32][17];
  __shared__ double sm_col[LA_WARPS][64];
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * LA_WARPS;
  const int w0 = blockIdx.x * LA_WARPS + (threadIdx.x >> 5);
  LaRowPre pre;
  bool have = la_row_load<FWD>(lptr[0] + w0, lptr[1], order, ecol, eval, eptr, mv, ncol, v, s, v2, w2, lane, pre);
  for (int L = 0; L < nlev; ++L) {
    const int b = lptr[L + 1];
    int q = lptr[L] + w0;
    while (have) {
      const LaRowPre& o = pre;
      const int64_t r = o.r;
      if (ncol == 1) {
        double acc = 0.0;
        if (o.jl >= 0) acc = o.bl * x[o.jl];
        for (int k = o.k0 + 32 + lane; k < o.k1; k += 32) {
          const int j = ecol[k];
          if (j >= 0) acc = fma(eval[k], x[j], acc);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) {
          const double xr = o.sr * o.v0 - acc;
          __stcg(x + r, xr);
          if (out2) out2[r] = xr + o.w2r * o.u0;
        }
      } else {
        double acc0 = 0.0, acc1 = 0.0;
        if (o.k1 - o.k0 <= long_min) {
          la_gather_cols_weak(x, ncol, lane, o.jl, o.bl, o.k1 - o.k0 < 32 ? o.k1 - o.k0 : 32, acc0, acc1);
          for (int kb = o.k0 + 32; kb < o.k1; kb += 32) {
            const int k = kb + lane;
            const int jl = k < o.k1 ? ecol[k] : -1;
            const double bl = k < o.k1 ? eval[k] : 0.0;
            la_gather_cols_weak(x, ncol, lane, jl, bl, o.k1 - kb < 32 ? o.k1 - kb : 32, acc0, acc1);
          }
        } else {
          la_long_row(x, ncol, ecol, eval, o.k0, o.k1, lane, sm_red[threadIdx.x >> 5], sm_col[threadIdx.x >> 5],
                      acc0, acc1);
        }
        const int c1 = lane + 32;
        if (lane < ncol) {
          const double xr = o.sr * o.v0 - acc0;
          __stcg(x + r * ncol + lane, xr);
          if (out2) out2[r * ncol + lane] = xr + o.w2r * o.u0;
        }
        if (c1 < ncol) {
          const double xr = o.sr * o.v1 - acc1;
          __stcg(x + r * ncol + c1, xr);
          if (out2) out2[r * ncol + c1] = xr + o.w2r * o.u1;
        }
      }
      q += nw;
      have = la_row_load<FWD>(q, b, order, ecol, eval, eptr, mv, ncol, v, s, v2, w2, lane, pre);
    }
    // the first row of the next level: prefetched before the barrier
    if (L + 1 < nlev)
      have = la_row_load<FWD>(lptr[L + 1] + w0, lptr[L + 2], order, ecol, eval, eptr, mv, ncol, v, s, v2, w2, lane,
                              pre);
    grid.sync();
    if (dbg && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      dbg[L] = t;
    }
  }
}

// ------------------------------------------------------------------ C = U^T diag(rs) V (split rows)
// grid (nsplit, ceil(mk / 64)); thread (kk = t % 64, g = t / 64): k = k0 + kk, rows r = r0 + g + 4 q;
// part[split][c][k] (ncol x mk per split)
constexpr int TS_K = 64, TS_R = 32;
template <int NC>
__global__ void __launch_bounds__(256) la_tsgemm_kernel(const double* __restrict__ U, int64_t ldu, int mk, int64_t n,
                                                        const double* __restrict__ V, int ncol,
                                                        const int64_t* __restrict__ vrow,
                                                        const double* __restrict__ rs, int64_t rows_per,
                                                        double* __restrict__ part) {
  __shared__ double vs[TS_R][NC + 1];
  constexpr int CH = NC > 8 ? 8 : NC;  // columns per reduction round
  __shared__ double red[4][TS_K][CH + 1];
  const int t = threadIdx.x, kk = t & (TS_K - 1), g = t >> 6;
  const int k = blockIdx.y * TS_K + kk;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < n ? r0 + rows_per : n;
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  for (int64_t rb = r0; rb < r1; rb += TS_R) {
    __syncthreads();
    for (int e = t; e < TS_R * NC; e += 256) {
      const int rr = e / NC, c = e % NC;
      const int64_t r = rb + rr;
      double val = 0.0;
      if (r < r1 && c < ncol) {
        const int64_t src = vrow ? vrow[r] : r;
        val = V[src * ncol + c];
        if (rs) val *= rs[src];
      }
      vs[rr][c] = val;
    }
    __syncthreads();
    if (k < mk) {
      for (int rr = g; rr < TS_R && rb + rr < r1; rr += 4) {
        const double u = U[(rb + rr) * ldu + k];
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] = fma(u, vs[rr][c], acc[c]);
      }
    }
  }
  // reduce over the 4 row groups, CH columns at a time
#pragma unroll
  for (int c0 = 0; c0 < NC; c0 += CH) {
    __syncthreads();
#pragma unroll
    for (int c = 0; c < CH; ++c) red[g][kk][c] = acc[c0 + c];
    __syncthreads();
    for (int e = t; e < TS_K * CH; e += 256) {
      const int k2 = e % TS_K, c = e / TS_K;
      const int kg = blockIdx.y * TS_K + k2;
      if (kg < mk && c0 + c < ncol) {
        const double sum = red[0][k2][c] + red[1][k2][c] + red[2][k2][c] + red[3][k2][c];
        part[((size_t)blockIdx.x * ncol + c0 + c) * mk + kg] = sum;
      }
    }
  }
}

// The same contraction on the FP64 tensor cores for 8 < ncol <= 64: a CTA owns 64 columns of U (k) x
// 64 columns of V and a row range; per stage 16 rows of U (cp.async) and of diag(rs) V (registers,
// loaded one stage ahead) in shared memory; warp w computes C rows 8w..8w+7 with 8 DMMA 8x8x4 tiles
// per 4 rows (A = U^T fragment, B = V fragment; pad 4 doubles: two wavefronts per fragment load).
constexpr int TD_R = 16, TD_K = 64, TD_N = 64, TD_PAD = 4;
__global__ void __launch_bounds__(256) la_tsgemm_dmma_kernel(const double* __restrict__ U, int64_t ldu, int mk,
                                                             int64_t n, const double* __restrict__ V, int ncol,
                                                             int64_t ldv, const double* __restrict__ rs,
                                                             int64_t rows_per, double* __restrict__ part) {
  __shared__ __align__(16) double Us[2][TD_R][TD_K + TD_PAD];
  __shared__ __align__(16) double Vs[2][TD_R][TD_N + TD_PAD];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int k0 = blockIdx.y * TD_K;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < n ? r0 + rows_per : n;
  const int nst = (int)((r1 - r0 + TD_R - 1) / TD_R);
  auto load_u = [&](int b, int64_t rb) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int e = t + 256 * i;
      const int rr = e >> 5, c2 = (e & 31) * 2;
      const int64_t r = rb + rr;
      const bool ok = r < r1 && k0 + c2 < mk;
      cp_async16(&Us[b][rr][c2], ok ? U + r * ldu + k0 + c2 : U, ok);
    }
    cp_async_commit();
  };
  double vreg[4];
  auto load_v = [&](int64_t rb) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = t + 256 * i;
      const int rr = e >> 6, c = e & 63;
      const int64_t r = rb + rr;
      double val = 0.0;
      if (r < r1 && c < ncol) {
        val = V[r * ldv + c];
        if (rs) val *= rs[r];
      }
      vreg[i] = val;
    }
  };
  auto store_v = [&](int b) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = t + 256 * i;
      Vs[b][e >> 6][e & 63] = vreg[i];
    }
  };
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  if (nst > 0) {
    load_u(0, r0);
    load_v(r0);
    store_v(0);
  }
  for (int st = 0; st < nst; ++st) {
    const int b = st & 1;
    const bool more = st + 1 < nst;
    if (more) {
      load_u(b ^ 1, r0 + (int64_t)(st + 1) * TD_R);
      load_v(r0 + (int64_t)(st + 1) * TD_R);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int k4 = 0; k4 < TD_R / 4; ++k4) {
      const int rr = 4 * k4 + (lane & 3);
      const double a = Us[b][rr][8 * w + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma884(acc[j][0], acc[j][1], a, Vs[b][rr][8 * j + (lane >> 2)]);
    }
    __syncthreads();
    if (more) store_v(b ^ 1);
  }
  const int k = k0 + 8 * w + (lane >> 2);
  if (k < mk) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * j + 2 * (lane & 3) + e;
        if (c < ncol) part[((size_t)blockIdx.x * ncol + c) * mk + k] = acc[j][e];
      }
    }
  }
}

// out[r] (+)= alpha sum_k U[r][k] c[k] for one right-hand side (the DMMA gemm_tn would compute a
// 64-column tile for one useful column): a warp per row, 16-byte loads, c in shared memory.
__global__ void __launch_bounds__(256) la_gemv_kernel(const double* __restrict__ U, int64_t ldu, int64_t n, int mk,
                                                      const double* __restrict__ c, double alpha, int accum,
                                                      double* __restrict__ out) {
  extern __shared__ double cs[];
  for (int k = threadIdx.x; k < mk; k += blockDim.x) cs[k] = c[k];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); r < n; r += nw) {
    const double2* u2 = reinterpret_cast<const double2*>(U + r * ldu);
    double acc = 0.0;
    for (int k2 = lane; 2 * k2 < mk; k2 += 32) {
      const double2 u = __ldg(u2 + k2);
      acc = fma(u.x, cs[2 * k2], acc);
      acc = fma(u.y, cs[2 * k2 + 1], acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[r] = alpha * acc + (accum ? out[r] : 0.0);
  }
}

// Ct[c][k] = alpha sum_s part[s][c][k]: a warp per output, lanes over the splits (fixed order:
// lane-strided partial sums, then a fixed shuffle tree)
__global__ void la_tsreduce_kernel(const double* __restrict__ part, int nsplit, int ncol, int mk, double* __restrict__ Ct,
                                   double alpha) {
  const int64_t tot = (int64_t)ncol * mk;
  const int lane = threadIdx.x & 31;
  for (int64_t e = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); e < tot;
       e += (int64_t)gridDim.x * (blockDim.x / 32)) {
    double s = 0.0;
    for (int q = lane; q < nsplit; q += 32) s += part[(size_t)q * tot + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) Ct[e] = alpha * s;
  }
}

// ------------------------------------------------------------------ reductions
// OP 0: sum_i a[i,c] b[i,c] (per column c);  OP 1: sum_i y_i b_i - log(1 + e^{b_i}) (ncol = 1, a = y, b = b);
// OP 2: sum_i log a_i (ncol = 1)
template <int OP>
__global__ void __launch_bounds__(256) la_reduce_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                        int64_t n, int ncol, int64_t rows_per,
                                                        double* __restrict__ part) {
  __shared__ double sm[256];
  const int t = threadIdx.x;
  const int used = (256 / ncol) * ncol;  // threads in use: thread t always sees column t % ncol
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < n ? r0 + rows_per : n;
  double s = 0.0;
  if (t < used) {
    const int64_t e0 = r0 * ncol, e1 = r1 * ncol;
    for (int64_t e = e0 + t; e < e1; e += used) {
      if (OP == 0) {
        s = fma(a[e], b[e], s);
      } else if (OP == 1) {
        const double bb = b[e];
        s += a[e] * bb - (fmax(bb, 0.0) + log1p(exp(-fabs(bb))));
      } else {
        s += log(a[e]);
      }
    }
  }
  sm[t] = s;
  __syncthreads();
  if (t < ncol) {
    double acc = 0.0;
    for (int q = t; q < used; q += ncol) acc += sm[q];
    part[(size_t)blockIdx.x * ncol + t] = acc;
  }
}

__global__ void la_reduce_final_kernel(const double* __restrict__ part, int nsplit, int ncol, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  double s = 0.0;
  for (int q = 0; q < nsplit; ++q) s += part[(size_t)q * ncol + c];
  out[c] = s;
}

// ------------------------------------------------------------------ elementwise
// Newton step inputs at b: pi = sigma(b), W = pi (1 - pi), winv = 1/W, v = W b + (y - pi)
__global__ void la_newton_prep_kernel(const double* __restrict__ y, const double* __restrict__ b, int64_t n,
                                      double* __restrict__ W, double* __restrict__ winv, double* __restrict__ v,
                                      double* __restrict__ x0) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double bi = b[i];
    const double pi = 1.0 / (1.0 + exp(-bi));
    const double w = pi * (1.0 - pi);
    W[i] = w;
    winv[i] = 1.0 / w;
    v[i] = w * bi + (y[i] - pi);
    if (x0) x0[i] = w * bi;
  }
}

// after the solve: b = x / W = winv x, a = v - x   (P:265 via pcls2)
__global__ void la_newton_update_kernel(const double* __restrict__ x, const double* __restrict__ v,
                                        const double* __restrict__ winv, int64_t n, double* __restrict__ b,
                                        double* __restrict__ a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    b[i] = winv[i] * x[i];
    a[i] = v[i] - x[i];
  }
}

// FITC rows: DV_i = sigma_1^2 - ||u_i||^2 + 1/W_i, dvinv = 1/DV, S_i = u_i / sqrt(DV_i) (App. FITC)
__global__ void la_fitc_rows_kernel(const double* __restrict__ U, int64_t ldu, int mk, int ld, int64_t n,
                                    const double* __restrict__ unorm2, double sigma2, const double* __restrict__ winv,
                                    double* __restrict__ DV, double* __restrict__ dvinv, double* __restrict__ S) {
  const int64_t i = blockIdx.x;
  if (i >= n) return;
  const double dv = sigma2 - unorm2[i] + winv[i];
  const double r = 1.0 / sqrt(dv);
  if (threadIdx.x == 0) {
    DV[i] = dv;
    dvinv[i] = 1.0 / dv;
  }
  for (int k = threadIdx.x; k < ld; k += blockDim.x) S[i * ld + k] = k < mk ? U[i * ldu + k] * r : 0.0;
}

__global__ void la_rownorm2_kernel(const double* __restrict__ U, int64_t ldu, int mk, int64_t n,
                                   double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  double s = 0.0;
  for (int k = lane; k < mk; k += 32) {
    const double u = U[i * ldu + k];
    s = fma(u, u, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[i] = s;
}

// out[i,c] = alpha_row(i) * in[i,c]  (alpha_row = r[i] or sqrt(r[i]))
__global__ void la_rowscale_kernel(const double* __restrict__ in, const double* __restrict__ r, int use_sqrt,
                                   int64_t n, int ncol, double* __restrict__ out) {
  const int64_t tot = n * ncol;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const double s = r[e / ncol];
    out[e] = (use_sqrt ? sqrt(s) : s) * in[e];
  }
}

// out = (a - b) * r_row  (FITC solve tail: P^{-1} w = D_V^{-1} (w - U M_V^{-1} U^T D_V^{-1} w))
__global__ void la_sub_rowscale_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                       const double* __restrict__ r, int64_t n, int ncol, double* __restrict__ out) {
  const int64_t tot = n * ncol;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = (a[e] - b[e]) * r[e / ncol];
}

// CG: r = b - r (in place: r holds A x0), used for a warm start
__global__ void la_residual_kernel(const double* __restrict__ b, int64_t tot, double* __restrict__ r) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x)
    r[e] = b[e] - r[e];
}

// CG step 1: alpha_c = rz_c / pq_c on active columns (0 otherwise), recorded in hist_a[it][c]
__global__ void la_cg_alpha_kernel(const double* __restrict__ rz, const double* __restrict__ pq,
                                   const int* __restrict__ active, int ncol, double* __restrict__ alpha,
                                   double* __restrict__ hist_a) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const double a = active[c] ? rz[c] / pq[c] : 0.0;
  alpha[c] = a;
  if (hist_a) hist_a[c] = a;
}

// CG step 2: x += alpha p, r -= alpha q
__global__ void la_cg_xr_kernel(const double* __restrict__ alpha, const double* __restrict__ p,
                                const double* __restrict__ q, int64_t n, int ncol, double* __restrict__ x,
                                double* __restrict__ r) {
  const int64_t tot = n * ncol;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const double a = alpha[e % ncol];
    x[e] = fma(a, p[e], x[e]);
    r[e] = fma(-a, q[e], r[e]);
  }
}

// CG step 3: beta_c = rz_new_c / rz_c (active), rz = rz_new; recorded in hist_b[it][c]
__global__ void la_cg_beta_kernel(const double* __restrict__ rz_new, double* __restrict__ rz,
                                  const int* __restrict__ active, int ncol, double* __restrict__ beta,
                                  double* __restrict__ hist_b) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const double b = active[c] ? rz_new[c] / rz[c] : 0.0;
  beta[c] = b;
  if (hist_b) hist_b[c] = b;
  if (active[c]) rz[c] = rz_new[c];
}

// CG step 4: p = z + beta p on active columns
__global__ void la_cg_p_kernel(const double* __restrict__ beta, const int* __restrict__ active,
                               const double* __restrict__ z, int64_t n, int ncol, double* __restrict__ p) {
  const int64_t tot = n * ncol;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % ncol);
    if (active[c]) p[e] = fma(beta[c], p[e], z[e]);
  }
}

__global__ void la_transpose_kernel(const double* __restrict__ in, int rows, int cols, int ldin,
                                    double* __restrict__ out, int ldout) {
  const int64_t tot = (int64_t)rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / cols), c = (int)(e % cols);
    out[(int64_t)c * ldout + r] = in[(int64_t)r * ldin + c];
  }
}

// sum_j log L_jj of an in-place Cholesky factor (lower part of A)
__global__ void la_logdiag_kernel(const double* __restrict__ A, int m, int lda, double* __restrict__ out) {
  __shared__ double sm[256];
  double s = 0.0;
  for (int j = threadIdx.x; j < m; j += blockDim.x) s += log(A[(size_t)j * lda + j]);
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = 2.0 * sm[0];
}

// s_i = (b_i + sum_p B[i,p] b_{N(i)_p}) / sqrt(D_i)  (D^{-1/2} B b, for b^T Sigma_dagger^{-1} b)
__global__ void la_bapply_kernel(const int32_t* __restrict__ nbr, const double* __restrict__ Bc, int mv, int64_t n,
                                 const double* __restrict__ D, const double* __restrict__ b, double* __restrict__ s) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = b[i];
    for (int p = 0; p < mv; ++p) {
      const int j = nbr[i * mv + p];
      if (j >= 0) acc = fma(Bc[i * mv + p], b[j], acc);
    }
    s[i] = acc / sqrt(D[i]);
  }
}

// ---- Sigma_dagger^{-1} v = B^T D^{-1/2} [s - W_U M^{-1} W_U^T s], s = D^{-1/2} B v (Woodbury),
// the (W + Sigma_dagger^{-1}) operator of (pcls1): sparse products with B and B^T, no solves.
// s[i, c] = D_i^{-1/2} (v[i, c] + sum_p B[i,p] v[N(i)_p, c])
__global__ void la_bapply_cols_kernel(const int32_t* __restrict__ nbr, const double* __restrict__ Bc, int mv,
                                      int64_t n, int ncol, const double* __restrict__ D, const double* __restrict__ v,
                                      double* __restrict__ s) {
  const int64_t tot = n * ncol;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ncol;
    const int c = (int)(e % ncol);
    double acc = v[e];
    for (int p = 0; p < mv; ++p) {
      const int j = nbr[i * mv + p];
      if (j >= 0) acc = fma(Bc[i * mv + p], v[(int64_t)j * ncol + c], acc);
    }
    s[e] = acc * rsqrt(D[i]);
  }
}

// z[i, c] = D_i^{-1/2} (s[i, c] - Y[ipos[i], c])  (Y rows by processing position)
__global__ void la_woodbury_mid_kernel(const double* __restrict__ s, const double* __restrict__ Y,
                                       const int* __restrict__ ipos, const double* __restrict__ D, int64_t n, int ncol,
                                       double* __restrict__ z) {
  const int64_t tot = n * ncol;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ncol;
    const int c = (int)(e % ncol);
    const double y = Y ? Y[(int64_t)ipos[i] * ncol + c] : 0.0;
    z[e] = (s[e] - y) * rsqrt(D[i]);
  }
}

// out[j, c] = z[j, c] + sum_{children} tval[k] z[trow[k], c]  (+ w_j v[j, c] with w = 1/winv)
__global__ void la_btapply_cols_kernel(const int* __restrict__ tptr, const int* __restrict__ trow,
                                       const double* __restrict__ tval, int64_t n, int ncol,
                                       const double* __restrict__ z, const double* __restrict__ winv,
                                       const double* __restrict__ v, double* __restrict__ out) {
  const int64_t tot = n * ncol;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / ncol;
    const int c = (int)(e % ncol);
    double acc = z[e];
    for (int k = tptr[j]; k < tptr[j + 1]; ++k) acc = fma(tval[k], z[(int64_t)trow[k] * ncol + c], acc);
    if (winv) acc += v[e] / winv[j];
    out[e] = acc;
  }
}

// inverse of the processing order: ipos[order[p]] = p
__global__ void la_invorder_kernel(const int64_t* __restrict__ order, int64_t n, int* __restrict__ ipos) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    ipos[order[p]] = (int)p;
}

// fin[0] = log p(y|b~), fin[1] = s.s, fin[2] = z.z, fin[3] = log det W, fin[4] = sum log D_V,
// fin[5] = log det M_V; slq[c] = e1^T log(T_c) e1.  out = (nll, -log p, quad, logdet, logdet_W, logdet_P)
// with L = -log p + quad / 2 + logdet / 2 and logdet from slq_v2
__global__ void la_finish_kernel(const double* __restrict__ fin, const double* __restrict__ slq, int64_t n, int ell,
                                 double* __restrict__ out) {
  const double quad = fin[1] - fin[2];
  const double ldP = fin[4] + fin[5];
  double ssum = 0.0;
  for (int c = 0; c < ell; ++c) ssum += slq[c];
  const double logdet = ell > 0 ? fin[3] + (double)n / ell * ssum + ldP : 0.0;
  out[0] = -fin[0] + 0.5 * quad + 0.5 * logdet;
  out[1] = -fin[0];
  out[2] = quad;
  out[3] = logdet;
  out[4] = fin[3];
  out[5] = ldP;
}

// ------------------------------------------------------------------ SLQ quadrature
// One thread per probe c: T (k x k tridiagonal) from the CG coefficients:
//   T_jj = 1/alpha_j + beta_{j-1}/alpha_{j-1},  T_{j,j+1} = sqrt(beta_j)/alpha_j
// eigen-decomposition by the implicit QL iteration with Wilkinson shifts, tracking only the first
// row of the eigenvector matrix; e_1^T log(T) e_1 = sum_k q_{1k}^2 log(lambda_k).
// d, e, q: per-probe scratch of kmax doubles each.
__global__ void la_slq_kernel(const double* __restrict__ hist_a, const double* __restrict__ hist_b,
                              const int* __restrict__ iters, int ncol, int kmax, double* __restrict__ scratch,
                              double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const int k = iters[c];
  double* d = scratch + (size_t)c * 3 * kmax;
  double* e = d + kmax;
  double* q = e + kmax;
  for (int j = 0; j < k; ++j) {
    const double aj = hist_a[(size_t)j * ncol + c];
    d[j] = 1.0 / aj + (j > 0 ? hist_b[(size_t)(j - 1) * ncol + c] / hist_a[(size_t)(j - 1) * ncol + c] : 0.0);
    e[j] = j + 1 < k ? sqrt(hist_b[(size_t)j * ncol + c]) / aj : 0.0;
    q[j] = j == 0 ? 1.0 : 0.0;
  }
  // implicit QL (symmetric tridiagonal): e[j] couples d[j], d[j+1]
  for (int l = 0; l < k; ++l) {
    for (int it = 0; it < 60; ++it) {
      int mm = l;
      for (; mm < k - 1; ++mm) {
        const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(e[mm]) <= 1e-16 * dd) break;
      }
      if (mm == l) break;
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = hypot(g, 1.0);
      g = d[mm] - d[l] + e[l] / (g + (g >= 0.0 ? r : -r));
      double s = 1.0, cc = 1.0, p = 0.0;
      int i = mm - 1;
      bool early = false;
      for (; i >= l; --i) {
        double f = s * e[i];
        const double b = cc * e[i];
        r = hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= p;
          e[mm] = 0.0;
          early = true;
          break;
        }
        s = f / r;
        cc = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0 * cc * b;
        p = s * r;
        d[i + 1] = g + p;
        g = cc * r - b;
        // first-row rotation of the eigenvector matrix (columns i, i+1)
        f = q[i + 1];
        q[i + 1] = s * q[i] + cc * f;
        q[i] = cc * q[i] - s * f;
      }
      if (early) continue;
      d[l] -= p;
      e[l] = g;
      e[mm] = 0.0;
    }
  }
  double sum = 0.0;
  for (int j = 0; j < k; ++j) sum += q[j] * q[j] * log(d[j]);
  out[c] = sum;
}

}  // namespace

// ============================================================================ launchers
static unsigned grid_for(int64_t work, int per = 256) {
  int64_t g = (work + per - 1) / per;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (unsigned)g;
}

cudaError_t launch_la_transpose_struct(const int32_t* nbr, int64_t n, int mv, int* cnt, int* cursor, int* tptr,
                                       int* tpos, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(cnt, 0, (size_t)n * sizeof(int), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(cursor, 0, (size_t)n * sizeof(int), s);
  if (e != cudaSuccess) return e;
  if (mv > 0) la_count_kernel<<<grid_for(n * mv), 256, 0, s>>>(nbr, n, mv, cnt);
  la_scan_kernel<<<1, 1024, 0, s>>>(cnt, n, tptr);
  if (mv > 0) {
    la_fill_kernel<<<grid_for(n * mv), 256, 0, s>>>(nbr, n, mv, tptr, cursor, tpos);
    la_sort_kernel<<<grid_for(n), 256, 0, s>>>(n, tptr, tpos);
  }
  return cudaGetLastError();
}

cudaError_t launch_la_tvals(const int* tpos, int64_t nnz, int mv, const double* Bc, int* trow, double* tval,
                            cudaStream_t s) {
  if (nnz == 0) return cudaSuccess;
  la_tvals_kernel<<<grid_for(nnz), 256, 0, s>>>(tpos, nnz, mv, Bc, trow, tval);
  return cudaGetLastError();
}

int la_ts_nsplit(int64_t n) {
  int64_t ns = (n + 511) / 512;  // >= 4 x 148 CTAs with the k tiles: the contraction is HBM-bound
  if (ns > 592) ns = 592;
  if (ns < 1) ns = 1;
  return (int)ns;
}

cudaError_t launch_la_tsgemm(const double* U, int64_t ldu, int mk, int64_t n, const double* V, int ncol,
                             const int64_t* vrow, const double* rs, double* part, double* Ct, double alpha,
                             cudaStream_t s) {
  if (mk == 0) return cudaSuccess;
  const int ns = la_ts_nsplit(n);
  const int64_t rows_per = (n + ns - 1) / ns;
  dim3 grid(ns, (mk + TS_K - 1) / TS_K);
  if (ncol <= 1)
    la_tsgemm_kernel<1><<<grid, 256, 0, s>>>(U, ldu, mk, n, V, ncol, vrow, rs, rows_per, part);
  else if (ncol <= 8)
    la_tsgemm_kernel<8><<<grid, 256, 0, s>>>(U, ldu, mk, n, V, ncol, vrow, rs, rows_per, part);
  else if (ncol <= 64 && !vrow)
    la_tsgemm_dmma_kernel<<<grid, 256, 0, s>>>(U, ldu, mk, n, V, ncol, ncol, rs, rows_per, part);
  else if (ncol <= 16)
    la_tsgemm_kernel<16><<<grid, 256, 0, s>>>(U, ldu, mk, n, V, ncol, vrow, rs, rows_per, part);
  else if (ncol <= 32)
    la_tsgemm_kernel<32><<<grid, 256, 0, s>>>(U, ldu, mk, n, V, ncol, vrow, rs, rows_per, part);
  else if (ncol <= 64)
    la_tsgemm_kernel<64><<<grid, 256, 0, s>>>(U, ldu, mk, n, V, ncol, vrow, rs, rows_per, part);
  else
    return cudaErrorInvalidValue;
  la_tsreduce_kernel<<<grid_for((int64_t)ncol * mk * 32), 256, 0, s>>>(part, ns, ncol, mk, Ct, alpha);
  return cudaGetLastError();
}

int la_red_nsplit(int64_t n) {
  int64_t ns = (n + 511) / 512;  // up to 4 CTAs per SM: a dot over n x ell is a bandwidth pass
  if (ns > 592) ns = 592;
  if (ns < 1) ns = 1;
  return (int)ns;
}

cudaError_t launch_la_reduce(int op, const double* a, const double* b, int64_t n, int ncol, double* part,
                             double* out, cudaStream_t s) {
  if (ncol < 1 || ncol > 256) return cudaErrorInvalidValue;
  const int ns = la_red_nsplit(n);
  const int64_t rows_per = (n + ns - 1) / ns;
  switch (op) {
    case 0: la_reduce_kernel<0><<<ns, 256, 0, s>>>(a, b, n, ncol, rows_per, part); break;
    case 1: la_reduce_kernel<1><<<ns, 256, 0, s>>>(a, b, n, 1, rows_per, part); break;
    default: la_reduce_kernel<2><<<ns, 256, 0, s>>>(a, b, n, 1, rows_per, part); break;
  }
  la_reduce_final_kernel<<<(ncol + 255) / 256, 256, 0, s>>>(part, ns, op == 0 ? ncol : 1, out);
  return cudaGetLastError();
}

cudaError_t launch_la_newton_prep(const double* y, const double* b, int64_t n, double* W, double* winv, double* v,
                                  double* x0, cudaStream_t s) {
  la_newton_prep_kernel<<<grid_for(n), 256, 0, s>>>(y, b, n, W, winv, v, x0);
  return cudaGetLastError();
}

cudaError_t launch_la_newton_update(const double* x, const double* v, const double* winv, int64_t n, double* b,
                                    double* a, cudaStream_t s) {
  la_newton_update_kernel<<<grid_for(n), 256, 0, s>>>(x, v, winv, n, b, a);
  return cudaGetLastError();
}

cudaError_t launch_la_fitc_rows(const double* U, int64_t ldu, int mk, int ld, int64_t n, const double* unorm2,
                                double sigma2, const double* winv, double* DV, double* dvinv, double* S,
                                cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  la_fitc_rows_kernel<<<(unsigned)n, 128, 0, s>>>(U, ldu, mk, ld, n, unorm2, sigma2, winv, DV, dvinv, S);
  return cudaGetLastError();
}

cudaError_t launch_la_rownorm2(const double* U, int64_t ldu, int mk, int64_t n, double* out, cudaStream_t s) {
  la_rownorm2_kernel<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(U, ldu, mk, n, out);
  return cudaGetLastError();
}

cudaError_t launch_la_rowscale(const double* in, const double* r, int use_sqrt, int64_t n, int ncol, double* out,
                               cudaStream_t s) {
  la_rowscale_kernel<<<grid_for(n * ncol), 256, 0, s>>>(in, r, use_sqrt, n, ncol, out);
  return cudaGetLastError();
}

cudaError_t launch_la_sub_rowscale(const double* a, const double* b, const double* r, int64_t n, int ncol, double* out,
                                   cudaStream_t s) {
  la_sub_rowscale_kernel<<<grid_for(n * ncol), 256, 0, s>>>(a, b, r, n, ncol, out);
  return cudaGetLastError();
}

cudaError_t launch_la_residual(const double* b, int64_t tot, double* r, cudaStream_t s) {
  la_residual_kernel<<<grid_for(tot), 256, 0, s>>>(b, tot, r);
  return cudaGetLastError();
}

cudaError_t launch_la_cg_alpha(const double* rz, const double* pq, const int* active, int ncol, double* alpha,
                               double* hist_a, cudaStream_t s) {
  la_cg_alpha_kernel<<<(ncol + 127) / 128, 128, 0, s>>>(rz, pq, active, ncol, alpha, hist_a);
  return cudaGetLastError();
}

cudaError_t launch_la_cg_xr(const double* alpha, const double* p, const double* q, int64_t n, int ncol, double* x,
                            double* r, cudaStream_t s) {
  la_cg_xr_kernel<<<grid_for(n * ncol), 256, 0, s>>>(alpha, p, q, n, ncol, x, r);
  return cudaGetLastError();
}

cudaError_t launch_la_cg_beta(const double* rz_new, double* rz, const int* active, int ncol, double* beta,
                              double* hist_b, cudaStream_t s) {
  la_cg_beta_kernel<<<(ncol + 127) / 128, 128, 0, s>>>(rz_new, rz, active, ncol, beta, hist_b);
  return cudaGetLastError();
}

cudaError_t launch_la_cg_p(const double* beta, const int* active, const double* z, int64_t n, int ncol, double* p,
                           cudaStream_t s) {
  la_cg_p_kernel<<<grid_for(n * ncol), 256, 0, s>>>(beta, active, z, n, ncol, p);
  return cudaGetLastError();
}

cudaError_t launch_la_transpose(const double* in, int rows, int cols, int ldin, double* out, int ldout, cudaStream_t s) {
  la_transpose_kernel<<<grid_for((int64_t)rows * cols), 256, 0, s>>>(in, rows, cols, ldin, out, ldout);
  return cudaGetLastError();
}

cudaError_t launch_la_logdiag(const double* A, int m, int lda, double* out, cudaStream_t s) {
  la_logdiag_kernel<<<1, 256, 0, s>>>(A, m, lda, out);
  return cudaGetLastError();
}

cudaError_t launch_la_slq(const double* hist_a, const double* hist_b, const int* iters, int ncol, int kmax,
                          double* scratch, double* out, cudaStream_t s) {
  la_slq_kernel<<<(ncol + 31) / 32, 32, 0, s>>>(hist_a, hist_b, iters, ncol, kmax, scratch, out);
  return cudaGetLastError();
}

cudaError_t launch_la_gemv(const double* U, int64_t ldu, int64_t n, int mk, const double* c, double alpha, int accum,
                           double* out, cudaStream_t s) {
  if (mk == 0 || n == 0) return cudaSuccess;
  if (mk & 1) return cudaErrorInvalidValue;  // mk is a multiple of 8
  int64_t blocks = (n + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  la_gemv_kernel<<<(unsigned)blocks, 256, mk * sizeof(double), s>>>(U, ldu, n, mk, c, alpha, accum, out);
  return cudaGetLastError();
}

cudaError_t launch_la_bapply_cols(const int32_t* nbr, const double* Bc, int mv, int64_t n, int ncol, const double* D,
                                  const double* v, double* s, cudaStream_t st) {
  la_bapply_cols_kernel<<<grid_for(n * ncol), 256, 0, st>>>(nbr, Bc, mv, n, ncol, D, v, s);
  return cudaGetLastError();
}
cudaError_t launch_la_woodbury_mid(const double* s, const double* Y, const int* ipos, const double* D, int64_t n,
                                   int ncol, double* z, cudaStream_t st) {
  la_woodbury_mid_kernel<<<grid_for(n * ncol), 256, 0, st>>>(s, Y, ipos, D, n, ncol, z);
  return cudaGetLastError();
}
cudaError_t launch_la_btapply_cols(const int* tptr, const int* trow, const double* tval, int64_t n, int ncol,
                                   const double* z, const double* winv, const double* v, double* out, cudaStream_t st) {
  la_btapply_cols_kernel<<<grid_for(n * ncol), 256, 0, st>>>(tptr, trow, tval, n, ncol, z, winv, v, out);
  return cudaGetLastError();
}
cudaError_t launch_la_invorder(const int64_t* order, int64_t n, int* ipos, cudaStream_t st) {
  la_invorder_kernel<<<grid_for(n), 256, 0, st>>>(order, n, ipos);
  return cudaGetLastError();
}

cudaError_t launch_la_bapply(const int32_t* nbr, const double* Bc, int mv, int64_t n, const double* D, const double* b,
                             double* s, cudaStream_t st) {
  la_bapply_kernel<<<grid_for(n), 256, 0, st>>>(nbr, Bc, mv, n, D, b, s);
  return cudaGetLastError();
}

cudaError_t launch_la_finish(const double* fin, const double* slq, int64_t n, int ell, double* out, cudaStream_t s) {
  la_finish_kernel<<<1, 1, 0, s>>>(fin, slq, n, ell, out);
  return cudaGetLastError();
}

cudaError_t launch_la_levels(const int32_t* nbr, int mv, int64_t n, const int* tptr, const int* trow, int* lev_f,
                             int* lev_b, int* flags, int epoch_f, int epoch_b, int* nlev_dev, cudaStream_t s) {
  // static row assignment over resident warps (deadlock-free only if every warp is resident): at most
  // the occupancy, capped at two blocks per SM
  static int cached = 0;
  if (!cached) {
    int per_sm = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, la_level_fwd_kernel, LA_THREADS, 0);
    int per_sm_b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_b, la_level_bwd_kernel, LA_THREADS, 0);
    per_sm = std::min(std::min(per_sm, per_sm_b), 2);
    cached = sms * std::max(per_sm, 1);
  }
  int64_t blocks = cached;
  const int64_t need = (n + LA_WARPS - 1) / LA_WARPS;
  if (blocks > need) blocks = need;
  la_level_fwd_kernel<<<(unsigned)blocks, LA_THREADS, 0, s>>>(nbr, mv, n, lev_f, flags, epoch_f);
  la_level_bwd_kernel<<<(unsigned)blocks, LA_THREADS, 0, s>>>(tptr, trow, n, lev_b, flags, epoch_b);
  cudaError_t e = cudaMemsetAsync(nlev_dev, 0, 2 * sizeof(int), s);
  if (e != cudaSuccess) return e;
  la_max_kernel<<<grid_for(n), 256, 0, s>>>(lev_f, n, nlev_dev);
  la_max_kernel<<<grid_for(n), 256, 0, s>>>(lev_b, n, nlev_dev + 1);
  return cudaGetLastError();
}

cudaError_t launch_la_reorder(const int* order_f, const int32_t* nbr, const double* Bc, int64_t n, int mv,
                              int32_t* ecol_f, double* eval_f, const int* order_b, const int* tptr, const int* trow,
                              const double* tval, int* cnt, int* eptr_b, int32_t* ecol_b, double* eval_b,
                              cudaStream_t s) {
  if (mv > 0) la_reorder_fwd_kernel<<<grid_for(n * mv), 256, 0, s>>>(order_f, nbr, Bc, n, mv, ecol_f, eval_f);
  la_seglen_kernel<<<grid_for(n), 256, 0, s>>>(order_b, tptr, n, cnt);
  la_scan_kernel<<<1, 1024, 0, s>>>(cnt, n, eptr_b);
  la_reorder_bwd_kernel<<<grid_for(n * 32), 256, 0, s>>>(order_b, tptr, trow, tval, eptr_b, n, ecol_b, eval_b);
  return cudaGetLastError();
}

cudaError_t launch_la_bucket(const int* key, int64_t n, int nkeys, int* cnt, int* cursor, int* ptr, int* order,
                             cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(cnt, 0, (size_t)nkeys * sizeof(int), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(cursor, 0, (size_t)nkeys * sizeof(int), s);
  if (e != cudaSuccess) return e;
  la_bucket_count_kernel<<<grid_for(n), 256, 0, s>>>(key, n, cnt);
  la_scan_kernel<<<1, 1024, 0, s>>>(cnt, nkeys, ptr);
  la_bucket_fill_kernel<<<grid_for(n), 256, 0, s>>>(key, n, ptr, cursor, order);
  return cudaGetLastError();
}

static int la_lvl_blocks(const void* fn) {
  static int cached[2] = {0, 0};
  const int idx = fn == (const void*)la_trsv_lvl_kernel<true> ? 0 : 1;
  if (!cached[idx]) {
    int per_sm = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, LA_THREADS, 0);
    static const char* cap_env = getenv("VIF_LA_LVL_BPS");
    const int cap = cap_env ? atoi(cap_env) : 1;
    if (per_sm < 1) per_sm = 1;
    if (cap > 0 && per_sm > cap) per_sm = cap;
    cached[idx] = sms * per_sm;
    static const char* ctas_env = getenv("VIF_LA_LVL_CTAS");  // experiment: fewer CTAs, cheaper barrier
    if (ctas_env && atoi(ctas_env) > 0 && atoi(ctas_env) < cached[idx]) cached[idx] = atoi(ctas_env);
  }
  return cached[idx];
}

cudaError_t launch_la_trsv_lvl(bool fwd, const int* order, const int* lptr, int nlev, const int32_t* ecol,
                               const double* eval, const int* eptr, int mv, int ncol, const double* v,
                               const double* scale, double* x, const double* v2, const double* w2, double* out2,
                               cudaStream_t s) {
  if (ncol > 64) return cudaErrorInvalidValue;
  const void* fn = fwd ? (const void*)la_trsv_lvl_kernel<true> : (const void*)la_trsv_lvl_kernel<false>;
  const int grid = la_lvl_blocks(fn);
  static const char* dbg_env = getenv("VIF_LA_DEBUG");
  static unsigned long long* dbg = nullptr;
  if (dbg_env && !dbg) cudaMalloc(&dbg, 1 << 20);
  unsigned long long* dbgp = dbg_env ? dbg : nullptr;
  static const char* lm_env = getenv("VIF_LA_LONG");
  // rows with more entries take the lanes-over-entries path; measured (n = 100k B^T): it pays for
  // ncol <= 8 (2.9 vs 3.6 ms at ncol 2), chunks of 32 entries win from ncol 16 on (4.7 vs 9.6 ms at 50)
  int long_min = lm_env ? atoi(lm_env) : (ncol <= 8 ? 32 : 1 << 30);
  void* args[] = {(void*)&order, (void*)&lptr, (void*)&nlev, (void*)&ecol, (void*)&eval, (void*)&eptr, (void*)&mv,
                  (void*)&ncol, (void*)&v, (void*)&scale, (void*)&x, (void*)&v2, (void*)&w2, (void*)&out2,
                  (void*)&long_min, (void*)&dbgp};
  cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(LA_THREADS), args, 0, s);
  if (dbg_env && e == cudaSuccess && nlev > 1 && nlev < 100000) {  // per-level durations (debug)
    static int calls = 0;
    if (++calls % 3 == 0) {
      std::vector<unsigned long long> t(nlev);
      std::vector<int> lp(nlev + 1);
      cudaMemcpyAsync(t.data(), dbg, nlev * 8, cudaMemcpyDeviceToHost, s);
      cudaMemcpyAsync(lp.data(), lptr, (nlev + 1) * 4, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      std::vector<std::pair<double, int>> d;
      for (int L = 1; L < nlev; ++L) d.push_back({(t[L] - t[L - 1]) * 1e-3, L});
      std::sort(d.begin(), d.end());
      double tot = (t[nlev - 1] - t[0]) * 1e-3;
      fprintf(stderr, "[la dbg] fwd=%d ncol=%d nlev=%d total_us=%.1f median_us=%.2f\n", (int)fwd, ncol, nlev, tot,
              d[d.size() / 2].first);
      for (int q = (int)d.size() - 1; q >= 0 && q >= (int)d.size() - 6; --q)
        fprintf(stderr, "   level %d: %.1f us, %d rows\n", d[q].second, d[q].first, lp[d[q].second + 1] - lp[d[q].second]);
    }
  }
  return e;
}

}  // namespace vif
