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

#include <algorithm>
#include <type_traits>

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


// ================================================================================================
// Sub-quadratic exact search (d <= 3): metric pruning with the triangle inequality of d_c.
// d_c(i,j) = sqrt(1 - |corr(i,j)|) is the distance between the sign classes of the normalised residual
// feature vectors (a metric, the one the paper's cover tree relies on), so for a cluster c with
// centre z_c and radius r_c = max_{j in c} d_c(z_c, j), every member j has d_c(i,j) >= d_c(i,z_c) - r_c.
//   clusters   all points in Morton order, 64 per cluster (compact in space, any index);
//   queries    i >= T sorted by (floor(log2 i), Morton) into tiles of 64 (similar neighbour radius);
//              i < T by the brute-force kernel above (their candidates are the first T rows);
//   pass 1     per query tile, the Morton-adjacent clusters (enough to hold ~4 m_v predecessors) give an
//              upper bound D_i on the m_v-th neighbour distance (1 = not enough, 2 = select everything);
//   select     cluster c is kept for tile Q iff d_c(z_Q, z_c) <= r_Q + max_{i in Q} D_i + r_c + 1e-6 -- any
//              true neighbour j of i in Q satisfies d_c(z_Q, z_c) <= d(z_Q,i) + d(i,j) + d(j,z_c);
//   pass 2     exhaustive over the kept clusters (masking j >= i), ties broken by index: the same sets as
//              the brute force, whatever order the clusters come in.
// ================================================================================================
constexpr int KN_LIST_CAP_MAX = 4096;

__device__ __forceinline__ bool knn_better(double s, int j, double v, int ix) { return s > v || (s == v && j < ix); }

// d_c between points a and b (rows of U): sqrt(max(0, 1 - |k - u_a.u_b| isd_a isd_b)); 2 if either is
// degenerate (reading c7: no metric bound, the caller then keeps everything).  Warp-cooperative.
template <int FAM>
__device__ double knn_dc_warp(const double* __restrict__ U, int64_t ldu, int m, const double* __restrict__ X,
                              const CovParams& p, const double* __restrict__ isd, const int* __restrict__ deg,
                              int a, int b, int lane) {
  double s = 0.0;
  const double* ua = U + (int64_t)a * ldu;
  const double* ub = U + (int64_t)b * ldu;
  for (int k = lane; k < m; k += 32) s = fma(ua[k], ub[k], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (deg[a] || deg[b]) return 2.0;
  const double c = cov<FAM>(X + (int64_t)a * p.d, X + (int64_t)b * p.d, p);
  const double sc = fabs(c - s) * isd[a] * isd[b];
  return sqrt(fmax(0.0, 1.0 - sc));
}

// centre (the middle member) and d_c radius of each group of gs consecutive entries of `perm` (clusters or
// query groups); a warp per group
template <int FAM>
__global__ void knn_groups_kernel(const double* __restrict__ U, int64_t ldu, int m, const double* __restrict__ X,
                                  CovParams p, const double* __restrict__ isd, const int* __restrict__ deg,
                                  const int32_t* __restrict__ perm, int64_t len, int64_t ngroups, int gs,
                                  int32_t* __restrict__ centre, double* __restrict__ radius) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= ngroups) return;
  const int64_t b0 = g * gs;
  const int cnt = (int)(len - b0 < gs ? len - b0 : gs);
  const int z = perm[b0 + cnt / 2];
  double r = 0.0;
  if (radius)
    for (int t = 0; t < cnt; ++t) r = fmax(r, knn_dc_warp<FAM>(U, ldu, m, X, p, isd, deg, z, perm[b0 + t], lane));
  if (lane == 0) {
    centre[g] = z;
    if (radius) radius[g] = r;
  }
}

// keys of the queries i >= T: (floor(log2 i) << 48) | the point's rank e in the Morton order (monotone in
// its Morton code); i < T sort last
__global__ void knn_qkeys_kernel(const uint64_t* __restrict__ unused, const int64_t* __restrict__ morder, int64_t n,
                                 int64_t T, uint64_t* __restrict__ qkey, int64_t* __restrict__ qval) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = morder[e];
    uint64_t k = ~0ULL;
    if (i >= T) k = ((uint64_t)(63 - __clzll((long long)i)) << 48) | (uint64_t)e;
    qkey[e] = k;
    qval[e] = i;
  }
}

__global__ void knn_perm32_kernel(const int64_t* __restrict__ src, int64_t len, int32_t* __restrict__ dst,
                                  int32_t* __restrict__ inv) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)src[e];
    dst[e] = v;
    if (inv) inv[v] = (int)e;
  }
}

// ---- 64 x 64 DMMA Gram of gathered rows: acc(r, c) = u_{qrow[r]} . u_{crow[c]} over mk columns ----
// (8 warps of 32 x 16; 2-stage cp.async ring in As / Bs; rows < 0 read as zero)
__device__ __forceinline__ void knn_gram_gather(const double* __restrict__ U, int64_t ldu, int mk,
                                                const int* __restrict__ qrow, const int* __restrict__ crow,
                                                double* As, double* Bs, double (&acc)[4][2][2], int tid) {
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int fr = lane >> 2, fk = (lane & 3) * 2;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nkt = (mk + KBK - 1) / KBK;
  auto load_stage = [&](int st, int kt) {
    const int k0 = kt * KBK;
    double* as = As + st * KQ * KPAD;
    double* bs = Bs + st * KQ * KPAD;
#pragma unroll
    for (int j = 0; j < KQ * (KBK / 2) / 256; ++j) {
      const int e = tid + j * 256;
      const int r = e / (KBK / 2), c2 = (e % (KBK / 2)) * 2;
      const int qi = qrow[r], ci = crow[r];
      const bool okq = qi >= 0 && k0 + c2 < mk, okc = ci >= 0 && k0 + c2 < mk;
      cp_async16(as + r * KPAD + c2, okq ? U + (int64_t)qi * ldu + k0 + c2 : U, okq);
      cp_async16(bs + r * KPAD + c2, okc ? U + (int64_t)ci * ldu + k0 + c2 : U, okc);
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
  __syncthreads();  // the ring may be reused (score tile) after this
}

// Exhaustive search of query tile t over a list of candidate clusters (pass 1: the nadj Morton-adjacent
// clusters around the tile centre's cluster; pass 2: the selected list, or every cluster on overflow).
// mode 1 writes D_i (upper bound of the m_v-th neighbour distance) per query; mode 2 the neighbour rows.
template <int FAM>
__global__ void __launch_bounds__(256, 2) knn_list_kernel(
    const double* __restrict__ U, int64_t ldu, int mk, const double* __restrict__ X, int64_t n, CovParams p,
    const double* __restrict__ isd, const int* __restrict__ deg, int mv, const int32_t* __restrict__ qperm,
    int64_t nqry, const int32_t* __restrict__ cperm, const int32_t* __restrict__ cpos, int64_t ncl,
    const int32_t* __restrict__ qcentre, const int32_t* __restrict__ sel_cnt, const int32_t* __restrict__ sel,
    int sel_cap, int mode, int64_t nmin_pred, int tile_off, int tile_stride, double* __restrict__ Dq,
    int32_t* __restrict__ out) {
  extern __shared__ __align__(16) double ksm[];
  double* As = ksm;
  double* Bs = As + KST * KQ * KPAD;
  double* Sc = As;
  double* lv = Bs + KST * KQ * KPAD;
  int* li = reinterpret_cast<int*>(lv + KQ * mv);
  __shared__ double xq[KQ][VIF_MAX_D], xc[KQ][VIF_MAX_D];
  __shared__ double isq[KQ], isc[KQ];
  __shared__ int dgq[KQ], cnt[KQ], qrow[KQ], crow[KQ];
  __shared__ double tbl[64];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int fr = lane >> 2, fk = (lane & 3) * 2;
  const int64_t t = tile_off + (int64_t)tile_stride * blockIdx.x;
  const int64_t q0 = t * KQ;
  exp_table_init(tbl, p.sigma2, tid);
  if (tid < KQ) {
    const int qi = q0 + tid < nqry ? qperm[q0 + tid] : -1;
    qrow[tid] = qi;
    isq[tid] = qi >= 0 ? isd[qi] : 0.0;
    dgq[tid] = qi >= 0 ? deg[qi] : 0;
    cnt[tid] = 0;
  }
  __syncthreads();
  for (int e = tid; e < KQ * p.d; e += blockDim.x) {
    const int r = e / p.d, k = e % p.d;
    xq[r][k] = qrow[r] >= 0 ? X[(int64_t)qrow[r] * p.d + k] * (fam_scale<FAM>() * p.inv_ls[k]) : 0.0;
  }
  const double inv_fs2 = 1.0 / (fam_scale<FAM>() * fam_scale<FAM>());
  // the candidate clusters of this tile
  int64_t nlist, cbeg = 0;
  bool all = false;
  if (mode == 1) {
    // enough Morton-adjacent clusters to hold ~4 m_v predecessors of the tile's smallest index
    const int64_t need = (4 * (int64_t)mv * n + (int64_t)KQ * nmin_pred - 1) / ((int64_t)KQ * nmin_pred) + 1;
    nlist = need < 4 ? 4 : (need > ncl ? ncl : need);
    const int64_t cz = cpos[qcentre[t]] / KQ;
    cbeg = cz - nlist / 2;
    if (cbeg < 0) cbeg = 0;
    if (cbeg + nlist > ncl) cbeg = ncl - nlist;
  } else {
    const int c = sel_cnt[t];
    all = c > sel_cap;
    nlist = all ? ncl : c;
  }
  for (int64_t li_ = 0; li_ < nlist; ++li_) {
    const int64_t cl = mode == 1 ? cbeg + li_ : (all ? li_ : (int64_t)sel[t * sel_cap + li_]);
    __syncthreads();  // previous tile's merge done (Sc, xc, crow reused)
    if (tid < KQ) {
      const int64_t e = cl * KQ + tid;
      const int cj = e < n ? cperm[e] : -1;
      crow[tid] = cj;
      isc[tid] = cj >= 0 ? isd[cj] : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < KQ * p.d; e += blockDim.x) {
      const int r = e / p.d, k = e % p.d;
      xc[r][k] = crow[r] >= 0 ? X[(int64_t)crow[r] * p.d + k] * (fam_scale<FAM>() * p.inv_ls[k]) : 0.0;
    }
    double acc[4][2][2];
    knn_gram_gather(U, ldu, mk, qrow, crow, As, Bs, acc, tid);
    // ---- scores (as knn_kernel; candidate j must precede the query i) ----
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wm * 32 + a * 8 + fr, c = wn * 16 + b * 8 + fk + h;
          const int i = qrow[r], j = crow[c];
          double sc = -INFINITY;
          if (i >= 0 && j >= 0 && j < i) {
            if (dgq[r]) {
              double d2 = 0.0;
              for (int k = 0; k < p.d; ++k) {
                const double tt = xq[r][k] - xc[c][k];
                d2 = fma(tt, tt, d2);
              }
              sc = -d2 * inv_fs2;
            } else if (isc[c] == 0.0) {
              sc = 0.0;
            } else {
              sc = fabs(cov_fast<FAM>(xq[r], xc[c], p.d, tbl) - acc[a][b][h]) * isq[r] * isc[c];
            }
          }
          Sc[r * (KQ + 1) + c] = sc;
        }
    __syncthreads();
    // ---- merge: one thread per query; (score desc, index asc) whatever the candidate order ----
    if (tid < KQ) {
      double* v = lv + tid * mv;
      int* ix = li + tid * mv;
      int k = cnt[tid];
      for (int c = 0; c < KQ; ++c) {
        const double s = Sc[tid * (KQ + 1) + c];
        if (s == -INFINITY) continue;
        const int j = crow[c];
        if (k < mv || knn_better(s, j, v[mv - 1], ix[mv - 1])) {
          int pos = k < mv ? k : mv - 1;
          while (pos > 0 && knn_better(s, j, v[pos - 1], ix[pos - 1])) {
            v[pos] = v[pos - 1];
            ix[pos] = ix[pos - 1];
            --pos;
          }
          v[pos] = s;
          ix[pos] = j;
          if (k < mv) ++k;
        }
      }
      cnt[tid] = k;
    }
  }
  __syncthreads();
  if (tid < KQ && qrow[tid] >= 0) {
    const int i = qrow[tid];
    const int want = i < mv ? i : mv;  // all predecessors when i <= m_v (reading c5)
    if (mode == 1) {
      double D = 2.0;  // degenerate query: scaled Euclidean ranking, no metric bound -> keep everything
      if (!dgq[tid]) D = cnt[tid] < want ? 2.0 : (want == 0 ? 0.0 : sqrt(fmax(0.0, 1.0 - lv[tid * mv + want - 1])));
      Dq[i] = D;
    } else {
      for (int k = 0; k < mv; ++k) out[(int64_t)i * mv + k] = k < cnt[tid] ? li[tid * mv + k] : -1;
    }
  }
}

// Selection: for 64 query tiles x every cluster (in blocks of 64) the centre-centre d_c by a DMMA Gram;
// cluster c is appended to tile t's list iff d_c(z_t, z_c) - r_c <= tau_t (tau = r_Q + max D_i + margin).
template <int FAM>
__global__ void __launch_bounds__(256, 2) knn_select_kernel(
    const double* __restrict__ U, int64_t ldu, int mk, const double* __restrict__ X, CovParams p,
    const double* __restrict__ isd, const int* __restrict__ deg, const int32_t* __restrict__ qcentre,
    const double* __restrict__ tau, int64_t nqt, const int32_t* __restrict__ ccentre,
    const double* __restrict__ crad, int64_t ncl, int32_t* __restrict__ sel_cnt, int32_t* __restrict__ sel,
    int sel_cap) {
  extern __shared__ __align__(16) double ksm[];
  double* As = ksm;
  double* Bs = As + KST * KQ * KPAD;
  __shared__ double xq[KQ][VIF_MAX_D], xc[KQ][VIF_MAX_D];
  __shared__ double isq[KQ], isc[KQ], tq[KQ], rc_[KQ];
  __shared__ int qrow[KQ], crow[KQ], dq[KQ], dcn[KQ];
  __shared__ double tbl[64];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int fr = lane >> 2, fk = (lane & 3) * 2;
  const int64_t t0 = (int64_t)blockIdx.x * KQ;
  exp_table_init(tbl, p.sigma2, tid);
  if (tid < KQ) {
    const int z = t0 + tid < nqt ? qcentre[t0 + tid] : -1;
    qrow[tid] = z;
    isq[tid] = z >= 0 ? isd[z] : 0.0;
    dq[tid] = z >= 0 ? deg[z] : 0;
    tq[tid] = t0 + tid < nqt ? tau[t0 + tid] : -1.0;
  }
  __syncthreads();
  for (int e = tid; e < KQ * p.d; e += blockDim.x) {
    const int r = e / p.d, k = e % p.d;
    xq[r][k] = qrow[r] >= 0 ? X[(int64_t)qrow[r] * p.d + k] * (fam_scale<FAM>() * p.inv_ls[k]) : 0.0;
  }
  for (int64_t c0 = 0; c0 < ncl; c0 += KQ) {
    __syncthreads();
    if (tid < KQ) {
      const int z = c0 + tid < ncl ? ccentre[c0 + tid] : -1;
      crow[tid] = z;
      isc[tid] = z >= 0 ? isd[z] : 0.0;
      dcn[tid] = z >= 0 ? deg[z] : 0;
      rc_[tid] = c0 + tid < ncl ? crad[c0 + tid] : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < KQ * p.d; e += blockDim.x) {
      const int r = e / p.d, k = e % p.d;
      xc[r][k] = crow[r] >= 0 ? X[(int64_t)crow[r] * p.d + k] * (fam_scale<FAM>() * p.inv_ls[k]) : 0.0;
    }
    double acc[4][2][2];
    knn_gram_gather(U, ldu, mk, qrow, crow, As, Bs, acc, tid);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wm * 32 + a * 8 + fr, c = wn * 16 + b * 8 + fk + h;
          if (qrow[r] < 0 || crow[c] < 0) continue;
          double dcc = 0.0;  // degenerate centres: no bound (keep)
          if (!dq[r] && !dcn[c]) {
            const double sc = fabs(cov_fast<FAM>(xq[r], xc[c], p.d, tbl) - acc[a][b][h]) * isq[r] * isc[c];
            dcc = sqrt(fmax(0.0, 1.0 - sc));
          }
          if (dcc - rc_[c] <= tq[r]) {
            const int64_t t = t0 + r;
            const int k = atomicAdd(&sel_cnt[t], 1);
            if (k < sel_cap) sel[t * sel_cap + k] = (int)(c0 + c);
          }
        }
  }
}

// tau_g = r_g + max_{i in group} D_i + margin (any D_i >= 2: keep everything); groups of gs queries
__global__ void knn_tau_kernel(const int32_t* __restrict__ qperm, int64_t nqry, const double* __restrict__ Dq,
                               const double* __restrict__ qrad, int64_t ngr, int gs, double* __restrict__ tau,
                               int32_t* __restrict__ sel_cnt) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ngr) return;
  double mx = 0.0;
  for (int r = 0; r < gs; ++r) {
    const int64_t e = g * gs + r;
    if (e < nqry) mx = fmax(mx, Dq[qperm[e]]);
  }
  tau[g] = mx >= 2.0 || qrad[g] >= 2.0 ? 1e30 : qrad[g] + mx + 1e-6;
  sel_cnt[g] = 0;
}

// Exhaustive search of query group g (8 queries, one warp) over its kept clusters (8 points each): per
// cluster one 8 x 8 DMMA block u_Q u_C^T over the mk columns with both operands loaded straight into the
// fragments (lane (r, t) holds row r, k-pair 2t of each 8-column chunk: the query rows stay in L1 across
// the clusters), scores as the brute force, merged into per-query lists by (score desc, index asc).
constexpr int KSW = 8;  // warps (query groups) per block
template <int FAM>
__global__ void __launch_bounds__(KSW * 32) knn_small_kernel(
    const double* __restrict__ U, int64_t ldu, int mk, const double* __restrict__ X, CovParams p,
    const double* __restrict__ isd, const int* __restrict__ deg, int mv, const int32_t* __restrict__ qperm,
    int64_t nqry, int64_t ngr, const int32_t* __restrict__ cperm, int64_t n, int64_t ncl,
    const int32_t* __restrict__ sel_cnt, const int32_t* __restrict__ sel, int sel_cap, int g_off, int g_stride,
    int32_t* __restrict__ out) {
  extern __shared__ __align__(16) double ssm_[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* lv = ssm_ + warp * (8 * mv + 8 * 8 + 2 * 8 * VIF_MAX_D);  // [8][mv] list scores
  double* sct = lv + 8 * mv;                                         // [8][8] scores of a block
  double* xq = sct + 64;                                             // [8][d]
  double* xc = xq + 8 * VIF_MAX_D;                                   // [8][d]
  __shared__ int ix_all[KSW][8][KMAXMV];
  __shared__ int cnt_all[KSW][8], qi_all[KSW][8], ci_all[KSW][8];
  __shared__ double tbl[64];
  exp_table_init(tbl, p.sigma2, threadIdx.x);
  __syncthreads();
  int(*ix)[KMAXMV] = ix_all[warp];
  int* cnt = cnt_all[warp];
  int* qi = qi_all[warp];
  int* ci = ci_all[warp];
  const double inv_fs2 = 1.0 / (fam_scale<FAM>() * fam_scale<FAM>());
  const int r = lane >> 2, t = lane & 3;
  for (int64_t g = g_off + (int64_t)g_stride * ((int64_t)blockIdx.x * KSW + warp); g < ngr;
       g += (int64_t)g_stride * gridDim.x * KSW) {
    if (lane < 8) {
      const int64_t e = g * 8 + lane;
      qi[lane] = e < nqry ? qperm[e] : -1;
      cnt[lane] = 0;
    }
    __syncwarp();
    for (int e = lane; e < 8 * p.d; e += 32) {
      const int rr = e / p.d, k = e % p.d;
      xq[rr * VIF_MAX_D + k] = qi[rr] >= 0 ? X[(int64_t)qi[rr] * p.d + k] * (fam_scale<FAM>() * p.inv_ls[k]) : 0.0;
    }
    const int myq = qi[r];
    const double isq = myq >= 0 ? isd[myq] : 0.0;
    const bool dgq = myq >= 0 && deg[myq];
    const double* qrow = U + (int64_t)(myq >= 0 ? myq : 0) * ldu + 2 * t;
    const int nsel = sel_cnt[g];
    const bool all = nsel > sel_cap;
    const int64_t nl = all ? ncl : nsel;
    for (int64_t l = 0; l < nl; ++l) {
      const int64_t c = all ? l : (int64_t)sel[g * sel_cap + l];
      __syncwarp();
      if (lane < 8) {
        const int64_t e = c * 8 + lane;
        ci[lane] = e < n ? cperm[e] : -1;
      }
      __syncwarp();
      // skip a cluster none of whose members precedes any query of the group
      int mx_q = -1, mn_c = 0x7fffffff;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        mx_q = max(mx_q, qi[k]);
        if (ci[k] >= 0) mn_c = min(mn_c, ci[k]);
      }
      if (mn_c >= mx_q) continue;
      for (int e = lane; e < 8 * p.d; e += 32) {
        const int rr = e / p.d, k = e % p.d;
        xc[rr * VIF_MAX_D + k] = ci[rr] >= 0 ? X[(int64_t)ci[rr] * p.d + k] * (fam_scale<FAM>() * p.inv_ls[k]) : 0.0;
      }
      const int myc = ci[r];
      const double* crow = U + (int64_t)(myc >= 0 ? myc : 0) * ldu + 2 * t;
      double a0 = 0.0, a1 = 0.0;
      const bool okq = myq >= 0, okc = myc >= 0;
      int k0 = 0;
      for (; k0 + 32 <= mk; k0 += 32) {
        double2 qa[4], cb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          qa[u] = okq ? __ldg(reinterpret_cast<const double2*>(qrow + k0 + 8 * u)) : make_double2(0.0, 0.0);
          cb[u] = okc ? __ldg(reinterpret_cast<const double2*>(crow + k0 + 8 * u)) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          dmma884(a0, a1, qa[u].x, cb[u].x);
          dmma884(a0, a1, qa[u].y, cb[u].y);
        }
      }
      for (; k0 < mk; k0 += 8) {
        const double2 qa = okq ? __ldg(reinterpret_cast<const double2*>(qrow + k0)) : make_double2(0.0, 0.0);
        const double2 cb = okc ? __ldg(reinterpret_cast<const double2*>(crow + k0)) : make_double2(0.0, 0.0);
        dmma884(a0, a1, qa.x, cb.x);
        dmma884(a0, a1, qa.y, cb.y);
      }
      // C fragment: lane (r, t) holds query r x candidates 2t, 2t+1
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = 2 * t + h;
        const int j = ci[cc];
        double sc = -INFINITY;
        if (myq >= 0 && j >= 0 && j < myq) {
          if (dgq) {
            double d2 = 0.0;
            for (int k = 0; k < p.d; ++k) {
              const double tt = xq[r * VIF_MAX_D + k] - xc[cc * VIF_MAX_D + k];
              d2 = fma(tt, tt, d2);
            }
            sc = -d2 * inv_fs2;
          } else if (deg[j]) {
            sc = 0.0;
          } else {
            sc = fabs(cov_fast<FAM>(xq + r * VIF_MAX_D, xc + cc * VIF_MAX_D, p.d, tbl) - (h ? a1 : a0)) * isq * isd[j];
          }
        }
        sct[r * 8 + cc] = sc;
      }
      __syncwarp();
      if (lane < 8) {
        double* v = lv + lane * mv;
        int* ixr = ix[lane];
        int k = cnt[lane];
        for (int cc = 0; cc < 8; ++cc) {
          const double s = sct[lane * 8 + cc];
          if (s == -INFINITY) continue;
          const int j = ci[cc];
          if (k < mv || knn_better(s, j, v[mv - 1], ixr[mv - 1])) {
            int pos = k < mv ? k : mv - 1;
            while (pos > 0 && knn_better(s, j, v[pos - 1], ixr[pos - 1])) {
              v[pos] = v[pos - 1];
              ixr[pos] = ixr[pos - 1];
              --pos;
            }
            v[pos] = s;
            ixr[pos] = j;
            if (k < mv) ++k;
          }
        }
        cnt[lane] = k;
      }
    }
    __syncwarp();
    if (lane < 8 && qi[lane] >= 0)
      for (int k = 0; k < mv; ++k) out[(int64_t)qi[lane] * mv + k] = k < cnt[lane] ? ix[lane][k] : -1;
    __syncwarp();
  }
}

}  // namespace

static_assert(2 * KST * KQ * KPAD >= KQ * (KQ + 1), "score tile must fit in the staging buffers");

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


// brute force of the query blocks from row T on (the prefix is already done)
static cudaError_t launch_knn_rest(const double* U, int64_t ldu, int m, int mk, const double* X, int64_t n,
                                   const CovParams& p, double* isd, int* deg, int mv, int32_t* out, cudaStream_t s,
                                   int qoff, int qstride, int64_t T) {
  (void)T;  // the brute force recomputes rows < T too (identical sets); kept simple for the rare fallback
  return launch_knn(U, ldu, m, mk, X, n, p, isd, deg, mv, out, s, qoff, qstride);
}

cudaError_t launch_knn_pruned(const double* U, int64_t ldu, int m, int mk, const double* X, int64_t n, const CovParams& p,
                              double* isd, int* deg, int mv, int32_t* out, cudaStream_t s, int qoff, int qstride,
                              void* scratch, size_t scratch_bytes, int64_t prefix) {
  if (n == 0 || mv == 0) return cudaSuccess;
  if (mv > KMAXMV) return cudaErrorInvalidValue;
  const int64_t T = prefix < 1 ? 1 : prefix;
  if (p.d > 3 || n <= T) return launch_knn(U, ldu, m, mk, X, n, p, isd, deg, mv, out, s, qoff, qstride);
  resvar_kernel<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(U, (int)ldu, m, n, p.sigma2, isd, deg);
  const size_t smem = knn_smem_bytes(mv);
  // ---- queries i < T: the brute force over the first T rows (their candidates) ----
  {
    const int64_t nqb = (T + KQ - 1) / KQ;
    if (qoff < nqb) {
      const unsigned grid = (unsigned)((nqb - qoff + qstride - 1) / qstride);
      auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e = smem_optin(kern, smem);
        if (e != cudaSuccess) return e;
        kern<<<grid, 256, smem, s>>>(U, ldu, mk, X, T, p, isd, deg, mv, out, qoff, qstride);
        return cudaGetLastError();
      };
      cudaError_t e;
      switch (p.family) {
        case FAM_M12: e = go(knn_kernel<FAM_M12>); break;
        case FAM_M32: e = go(knn_kernel<FAM_M32>); break;
        case FAM_M52: e = go(knn_kernel<FAM_M52>); break;
        default: e = go(knn_kernel<FAM_GAUSS>); break;
      }
      if (e != cudaSuccess) return e;
    }
  }
  // ---- scratch layout ----
  const int64_t nq = n - T;                          // queries of the pruned search
  const int64_t ncl64 = (n + KQ - 1) / KQ;           // 64-point clusters (pass 1 windows)
  const int64_t nqt64 = (nq + KQ - 1) / KQ;          // 64-query tiles (pass 1)
  const int64_t ncl = (n + 7) / 8;                   // 8-point clusters
  const int64_t ngr = (nq + 7) / 8;                  // 8-query groups
  char* base = reinterpret_cast<char*>(scratch);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    void* q = base + off;
    off += (bytes + 255) / 256 * 256;
    return q;
  };
  uint64_t* keys = (uint64_t*)take(n * 8);
  uint64_t* keys2 = (uint64_t*)take(n * 8);
  int64_t* vals = (int64_t*)take(n * 8);
  int64_t* vals2 = (int64_t*)take(n * 8);
  const size_t tb = order_temp_bytes(n);
  void* temp = take(tb);
  double* bbox = (double*)take(128 * 6 * 8 + 3 * VIF_MAX_D * 8 + 1024);
  int32_t* cperm = (int32_t*)take(n * 4);
  int32_t* cpos = (int32_t*)take(n * 4);
  int32_t* qperm = (int32_t*)take(n * 4);
  double* Dq = (double*)take(n * 8);
  int32_t* qcentre64 = (int32_t*)take(nqt64 * 4);
  int32_t* ccentre = (int32_t*)take(ncl * 4);
  double* crad = (double*)take(ncl * 8);
  int32_t* qcentre = (int32_t*)take(ngr * 4);
  double* qrad = (double*)take(ngr * 8);
  double* tau = (double*)take(ngr * 8);
  int32_t* sel_cnt = (int32_t*)take(ngr * 4);
  int64_t cap = off > scratch_bytes ? 0 : (int64_t)((scratch_bytes - off) / 4) / (ngr > 0 ? ngr : 1);
  if (cap > KN_LIST_CAP_MAX) cap = KN_LIST_CAP_MAX;
  if (cap > ncl) cap = ncl;
  // too little scratch for the lists (tiny m with a large n): the brute force for the rest, same result
  if (cap < 64 && cap < ncl) return launch_knn_rest(U, ldu, m, mk, X, n, p, isd, deg, mv, out, s, qoff, qstride, T);
  int32_t* sel = (int32_t*)take((size_t)ngr * cap * 4);
  // ---- clusters: all points in Morton order ----
  int64_t* morder = nullptr;
  cudaError_t e = launch_order(X, n, p.d, n, n, 1, 0, bbox, keys, keys2, vals, vals2, temp, tb, &morder, s);
  if (e != cudaSuccess) return e;
  knn_perm32_kernel<<<296, 256, 0, s>>>(morder, n, cperm, cpos);
  // ---- queries i >= T: (band, Morton rank) ----
  knn_qkeys_kernel<<<296, 256, 0, s>>>(nullptr, morder, n, T, keys, vals);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int64_t* qorder = nullptr;
  e = sort_pairs_u64(keys, keys2, vals, vals2, n, temp, tb, &qorder, s);
  if (e != cudaSuccess) return e;
  knn_perm32_kernel<<<296, 256, 0, s>>>(qorder, nq, qperm, nullptr);
  e = cudaMemsetAsync(Dq, 0, n * 8, s);
  if (e != cudaSuccess) return e;
  auto run = [&](auto fam) -> cudaError_t {
    constexpr int FAM = decltype(fam)::value;
    // pass 1: upper bounds D_i from the Morton-adjacent 64-point clusters of each 64-query tile
    knn_groups_kernel<FAM><<<(unsigned)((nqt64 + 7) / 8), 256, 0, s>>>(U, ldu, m, X, p, isd, deg, qperm, nq, nqt64, KQ,
                                                                      qcentre64, nullptr);
    cudaError_t e2 = smem_optin(knn_list_kernel<FAM>, smem);
    if (e2 != cudaSuccess) return e2;
    if (qoff < nqt64) {
      const unsigned gl = (unsigned)((nqt64 - qoff + qstride - 1) / qstride);
      knn_list_kernel<FAM><<<gl, 256, smem, s>>>(U, ldu, mk, X, n, p, isd, deg, mv, qperm, nq, cperm, cpos, ncl64,
                                                  qcentre64, nullptr, nullptr, 0, 1, T, qoff, qstride, Dq, out);
    }
    // 8-point clusters and 8-query groups: centres and d_c radii; the selection by the centre-centre bound
    knn_groups_kernel<FAM><<<(unsigned)((ncl + 7) / 8), 256, 0, s>>>(U, ldu, m, X, p, isd, deg, cperm, n, ncl, 8,
                                                                    ccentre, crad);
    knn_groups_kernel<FAM><<<(unsigned)((ngr + 7) / 8), 256, 0, s>>>(U, ldu, m, X, p, isd, deg, qperm, nq, ngr, 8,
                                                                    qcentre, qrad);
    knn_tau_kernel<<<(unsigned)((ngr + 255) / 256), 256, 0, s>>>(qperm, nq, Dq, qrad, ngr, 8, tau, sel_cnt);
    e2 = smem_optin(knn_select_kernel<FAM>, (size_t)2 * KST * KQ * KPAD * 8);
    if (e2 != cudaSuccess) return e2;
    knn_select_kernel<FAM><<<(unsigned)((ngr + KQ - 1) / KQ), 256, (size_t)2 * KST * KQ * KPAD * 8, s>>>(
        U, ldu, mk, X, p, isd, deg, qcentre, tau, ngr, ccentre, crad, ncl, sel_cnt, sel, (int)cap);
    // pass 2: every group over its kept clusters; groups of this rank: g = qoff, qoff + qstride, ...
    const size_t ssm = (size_t)KSW * (8 * mv + 64 + 2 * 8 * VIF_MAX_D) * sizeof(double);
    e2 = smem_optin(knn_small_kernel<FAM>, ssm);
    if (e2 != cudaSuccess) return e2;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t mine = (ngr - qoff + qstride - 1) / qstride;
    if (mine > 0) {
      const unsigned gs = (unsigned)std::min<int64_t>((mine + KSW - 1) / KSW, (int64_t)sms * 8);
      knn_small_kernel<FAM><<<gs, KSW * 32, ssm, s>>>(U, ldu, mk, X, p, isd, deg, mv, qperm, nq, ngr, cperm, n, ncl,
                                                      sel_cnt, sel, (int)cap, qoff, qstride, out);
    }
    return cudaGetLastError();
  };
  switch (p.family) {
    case FAM_M12: return run(std::integral_constant<int, FAM_M12>{});
    case FAM_M32: return run(std::integral_constant<int, FAM_M32>{});
    case FAM_M52: return run(std::integral_constant<int, FAM_M52>{});
    default: return run(std::integral_constant<int, FAM_GAUSS>{});
  }
}

}  // namespace vif
