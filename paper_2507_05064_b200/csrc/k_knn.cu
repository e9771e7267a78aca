// k_knn.cu -- correlation-distance neighbour sets on the GPU.
//
// N(i) = the m_v predecessors j < i with the smallest d_c(i,j) = sqrt(1 - |rho_c(i,j)| /
// sqrt(rho_c(i,i) rho_c(j,j))), rho_c = k - u_i.u_j (no nugget), ranked by (d_c, index)
// (reading c6); readings c5 and c7 as in the oracle (degenerate candidates score 0, degenerate queries
// rank by scaled Euclidean distance).  Exact brute force, the B200 way: a CTA owns 64 consecutive
// queries (rows of U, already in Vecchia order) and sweeps the candidate tiles of 64 predecessors;
// per tile the 64 x 64 block u_Q u_C^T is a DMMA GEMM over the m whitened columns with both operands
// streamed by cp.async (contiguous rows: no gather), the epilogue turns it into scores in shared
// memory, and one thread per query merges the tile into its sorted top-m_v list (a threshold test
// skips almost every candidate once the list is full).  The paper's cover tree (Alg. 3-4) returns the
// same sets; exhaustive search costs n^2 m / 2 FMA (2.5e14 at n = 1M, m = 500).
#include "common.cuh"
#include "kernels.h"

namespace vif {

namespace {

constexpr int KQ = 64, KBK = 16, KST = 2, KPAD = KBK + 8, KMAXMV = 47;  // rows padded to 24 doubles (64 mod 128 B)

// residual variance rd_i = sigma_1^2 - |u_i|^2, its 1/sqrt and degeneracy (c7)
__global__ void resvar_kernel(const double* __restrict__ U, int ldu, int m, int64_t n, double sigma2,
                              double* __restrict__ isd, int* __restrict__ deg) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (i >= n) return;
  double s = 0.0;
  for (int k = lane; k < m; k += 32) {
    const double u = U[i * (int64_t)ldu + k];
    s = fma(u, u, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const double rd = sigma2 - s;
    const bool dg = rd < 1e-7 * sigma2;
    deg[i] = dg;
    isd[i] = dg ? 0.0 : 1.0 / sqrt(rd);
  }
}

template <int FAM>
__global__ void __launch_bounds__(256, 2) knn_kernel(const double* __restrict__ U, int64_t ldu, int mk,
                                                    const double* __restrict__ X, int64_t n, CovParams p,
                                                    const double* __restrict__ isd, const int* __restrict__ deg,
                                                    int mv, int32_t* __restrict__ out, int qoff, int qstride) {
  extern __shared__ __align__(16) double ksm[];
  double* As = ksm;                              // [KST][KQ][KPAD]
  double* Bs = As + KST * KQ * KPAD;             // [KST][KQ][KPAD]
  double* Sc = As;                               // [KQ][KQ + 1] scores, aliased on the idle A/B stages
  double* lv = Bs + KST * KQ * KPAD;             // [KQ][mv] list scores
  int* li = reinterpret_cast<int*>(lv + KQ * mv);  // [KQ][mv] list indices
  __shared__ double xq[KQ][VIF_MAX_D], xc[KQ][VIF_MAX_D];
  __shared__ double isq[KQ], isc[KQ];
  __shared__ int dgq[KQ], cnt[KQ];
  __shared__ double tbl[64];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps of 32 x 16
  const int64_t nq = (n + KQ - 1) / KQ;
  // query blocks of this rank: kb = nq - 1 - (qoff + qstride * blockIdx.x), largest (longest) first; the
  // cyclic assignment balances the triangular work over the ranks
  const int64_t q0 = (nq - 1 - (qoff + (int64_t)qstride * blockIdx.x)) * KQ;
  exp_table_init(tbl, p.sigma2, tid);
  for (int e = tid; e < KQ * p.d; e += blockDim.x) {
    const int r = e / p.d, k = e % p.d;
    xq[r][k] = q0 + r < n ? X[(q0 + r) * p.d + k] * (fam_scale<FAM>() * p.inv_ls[k]) : 0.0;
  }
  if (tid < KQ) {
    isq[tid] = q0 + tid < n ? isd[q0 + tid] : 0.0;
    dgq[tid] = q0 + tid < n ? deg[q0 + tid] : 0;
    cnt[tid] = 0;
  }
  const double inv_fs2 = 1.0 / (fam_scale<FAM>() * fam_scale<FAM>());
  const int fr = lane >> 2, fk = (lane & 3) * 2;
  const int nkt = (mk + KBK - 1) / KBK;
  for (int64_t c0 = 0; c0 <= q0; c0 += KQ) {
    __syncthreads();  // previous tile's merge done (Sc, xc reused)
    for (int e = tid; e < KQ * p.d; e += blockDim.x) {
      const int r = e / p.d, k = e % p.d;
      xc[r][k] = c0 + r < n ? X[(c0 + r) * p.d + k] * (fam_scale<FAM>() * p.inv_ls[k]) : 0.0;
    }
    if (tid < KQ) isc[tid] = c0 + tid < n ? isd[c0 + tid] : 0.0;
    // ---- Gram tile u_Q u_C^T over the mk whitened columns (DMMA, 3-stage cp.async) ----
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    auto load_stage = [&](int st, int kt) {
      const int k0 = kt * KBK;
      double* as = As + st * KQ * KPAD;
      double* bs = Bs + st * KQ * KPAD;
#pragma unroll
      for (int j = 0; j < KQ * (KBK / 2) / 256; ++j) {
        const int e = tid + j * 256;
        const int r = e / (KBK / 2), c2 = (e % (KBK / 2)) * 2;
        const bool okq = q0 + r < n && k0 + c2 < mk, okc = c0 + r < n && k0 + c2 < mk;
        cp_async16(as + r * KPAD + c2, okq ? U + (q0 + r) * ldu + k0 + c2 : U, okq);
        cp_async16(bs + r * KPAD + c2, okc ? U + (c0 + r) * ldu + k0 + c2 : U, okc);
      }
    };
#pragma unroll
    for (int st = 0; st < KST - 1; ++st) {
      if (st < nkt) load_stage(st, st);
      cp_async_commit();
    }
    for (int kt = 0; kt < nkt; ++kt) {
      cp_async_wait<KST - 2>();
      __syncthreads();
      {
        const int nk = kt + KST - 1;
        if (nk < nkt) load_stage(nk % KST, nk);
        cp_async_commit();
      }
      const double* as = As + (kt % KST) * KQ * KPAD + (wm * 32 + fr) * KPAD + fk;
      const double* bs = Bs + (kt % KST) * KQ * KPAD + (wn * 16 + fr) * KPAD + fk;
#pragma unroll
      for (int kk = 0; kk < KBK; kk += 8) {
        double2 af[4], bf[2];
#pragma unroll
        for (int a = 0; a < 4; ++a) af[a] = *reinterpret_cast<const double2*>(as + a * 8 * KPAD + kk);
#pragma unroll
        for (int b = 0; b < 2; ++b) bf[b] = *reinterpret_cast<const double2*>(bs + b * 8 * KPAD + kk);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            dmma884(acc[a][b][0], acc[a][b][1], af[a].x, bf[b].x);
            dmma884(acc[a][b][0], acc[a][b][1], af[a].y, bf[b].y);
          }
      }
    }
    cp_async_wait<0>();
    __syncthreads();  // xc / isc visible
    // ---- scores ----
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wm * 32 + a * 8 + fr, c = wn * 16 + b * 8 + fk + h;
          const int64_t i = q0 + r, j = c0 + c;
          double sc = -INFINITY;
          if (j < i && i < n) {
            if (dgq[r]) {
              double d2 = 0.0;
              for (int k = 0; k < p.d; ++k) {
                const double t = xq[r][k] - xc[c][k];
                d2 = fma(t, t, d2);
              }
              sc = -d2 * inv_fs2;  // scaled Euclidean distance (x / lambda)
            } else if (isc[c] == 0.0) {
              sc = 0.0;
            } else {
              sc = fabs(cov_fast<FAM>(xq[r], xc[c], p.d, tbl) - acc[a][b][h]) * isq[r] * isc[c];
            }
          }
          Sc[r * (KQ + 1) + c] = sc;
        }
    __syncthreads();
    // ---- merge: one thread per query, candidates in increasing index order ----
    if (tid < KQ) {
      double* v = lv + tid * mv;
      int* ix = li + tid * mv;
      int k = cnt[tid];
      double thr = k < mv ? -INFINITY : v[mv - 1];
      for (int c = 0; c < KQ; ++c) {
        const double s = Sc[tid * (KQ + 1) + c];
        if (s == -INFINITY) continue;
        if (k < mv || s > thr) {
          int pos = k < mv ? k : mv - 1;
          while (pos > 0 && s > v[pos - 1]) {
            v[pos] = v[pos - 1];
            ix[pos] = ix[pos - 1];
            --pos;
          }
          v[pos] = s;
          ix[pos] = (int)(c0 + c);
          if (k < mv) ++k;
          thr = k < mv ? -INFINITY : v[mv - 1];
        }
      }
      cnt[tid] = k;
    }
  }
  __syncthreads();
  if (tid < KQ && q0 + tid < n)
    for (int k = 0; k < mv; ++k) out[(q0 + tid) * mv + k] = k < cnt[tid] ? li[tid * mv + k] : -1;
}

}  // namespace

static_assert(2 * KST * KQ * KPAD >= KQ * (KQ + 1), "score tile must fit in the staging buffers");

cudaError_t launch_knn_resvar(const double* U, int64_t ldu, int m, int64_t n, const CovParams& p, double* isd,
                              int* deg, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  resvar_kernel<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(U, (int)ldu, m, n, p.sigma2, isd, deg);
  return cudaGetLastError();
}

size_t knn_smem_bytes(int mv) {
  return sizeof(double) * ((size_t)2 * KST * KQ * KPAD + (size_t)KQ * mv) + sizeof(int) * (size_t)KQ * mv;
}

cudaError_t launch_knn(const double* U, int64_t ldu, int m, int mk, const double* X, int64_t n, const CovParams& p,
                       double* isd, int* deg, int mv, int32_t* out, cudaStream_t s, int qoff, int qstride) {
  if (n == 0 || mv == 0) return cudaSuccess;
  if (mv > KMAXMV) return cudaErrorInvalidValue;
  resvar_kernel<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(U, (int)ldu, m, n, p.sigma2, isd, deg);
  const size_t smem = knn_smem_bytes(mv);
  const int64_t nq = (n + KQ - 1) / KQ;
  if (qoff >= nq) return cudaGetLastError();
  const unsigned grid = (unsigned)((nq - qoff + qstride - 1) / qstride);
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, 256, smem, s>>>(U, ldu, mk, X, n, p, isd, deg, mv, out, qoff, qstride);
    return cudaGetLastError();
  };
  switch (p.family) {
    case FAM_M12: return go(knn_kernel<FAM_M12>);
    case FAM_M32: return go(knn_kernel<FAM_M32>);
    case FAM_M52: return go(knn_kernel<FAM_M52>);
    default: return go(knn_kernel<FAM_GAUSS>);
  }
}

}  // namespace vif
