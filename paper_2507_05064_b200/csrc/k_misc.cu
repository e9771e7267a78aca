// k_misc.cu -- input validation, processing order (Morton sort for L2 reuse of neighbour rows),
// emulated all-reduce, status reset.
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "kernels.h"

namespace vif {

// N(i) subset of {0..i-1}, no duplicates, -1 only as trailing padding (reading c5);
// X, y finite; Z finite.
__global__ void validate_kernel(const double* __restrict__ X, int64_t n, int d, const double* __restrict__ Z, int m,
                                const double* __restrict__ y, const int32_t* __restrict__ nbr, int mv,
                                DevStatus* st) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool bad = !isfinite(y[i]);
    for (int k = 0; k < d; ++k) bad |= !isfinite(X[i * d + k]);
    const int32_t* row = nbr + i * mv;
    bool pad = false;
    for (int k = 0; k < mv; ++k) {
      const int32_t j = row[k];
      if (j < 0) {
        bad |= j != -1;
        pad = true;
      } else {
        bad |= pad || j >= i;
        for (int t = 0; t < k; ++t) bad |= row[t] == j;
      }
    }
    if (bad) atomicMin(&st->bad_input, (unsigned long long)i);
    if (i < m) {
      bool bz = false;
      for (int k = 0; k < d; ++k) bz |= !isfinite(Z[i * d + k]);
      if (bz) atomicExch(&st->bad_z, 1);
    }
  }
  if (m > n) {  // more inducing points than data points
    for (int64_t i = n + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
      bool bz = false;
      for (int k = 0; k < d; ++k) bz |= !isfinite(Z[i * d + k]);
      if (bz) atomicExch(&st->bad_z, 1);
    }
  }
}

cudaError_t launch_validate(const double* X, int64_t n, int d, const double* Z, int m, const double* y,
                            const int32_t* nbr, int mv, DevStatus* st, cudaStream_t s) {
  validate_kernel<<<296, 256, 0, s>>>(X, n, d, Z, m, y, nbr, mv, st);
  return cudaGetLastError();
}

// prediction inputs (reading p1): finite coordinates; each neighbour row holds distinct training
// indices in [0, ntrain), -1 only as trailing padding (the vecchia kernel counts the leading valid
// entries and gathers them unchecked)
__global__ void validate_pred_kernel(const double* __restrict__ Xp, int64_t np, int d, const int32_t* __restrict__ nbrp,
                                     int mv, int64_t ntrain, DevStatus* st) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
    bool bad = false;
    for (int k = 0; k < d; ++k) bad |= !isfinite(Xp[i * d + k]);
    const int32_t* row = nbrp + i * mv;
    bool pad = false;
    for (int k = 0; k < mv; ++k) {
      const int32_t j = row[k];
      if (j < 0) {
        bad |= j != -1;
        pad = true;
      } else {
        bad |= pad || j >= ntrain;
        for (int t = 0; t < k; ++t) bad |= row[t] == j;
      }
    }
    if (bad) atomicMin(&st->bad_input, (unsigned long long)i);
  }
}

cudaError_t launch_validate_pred(const double* Xp, int64_t np, int d, const int32_t* nbrp, int mv, int64_t ntrain,
                                 DevStatus* st, cudaStream_t s) {
  validate_pred_kernel<<<296, 256, 0, s>>>(Xp, np, d, nbrp, mv, ntrain, st);
  return cudaGetLastError();
}

__global__ void reset_status_kernel(DevStatus* st) {
  st->bad_row = ~0ULL;
  st->bad_input = ~0ULL;
  st->km_fail = 0;
  st->m_fail = 0;
  st->bad_z = 0;
}

cudaError_t launch_reset_status(DevStatus* st, cudaStream_t s) {
  reset_status_kernel<<<1, 1, 0, s>>>(st);
  return cudaGetLastError();
}

// ---- processing order: Morton code of the first min(d,3) coordinates (bounding-box normalised) ----
constexpr int BB_BLOCKS = 128;

__global__ void bbox_partial_kernel(const double* __restrict__ X, int64_t n, int d, double* __restrict__ part) {
  const int dd = d < 3 ? d : 3;
  __shared__ double lo[3][256], hi[3][256];
  double l[3] = {1e300, 1e300, 1e300}, h[3] = {-1e300, -1e300, -1e300};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < dd; ++k) {
      const double v = X[i * d + k];
      l[k] = fmin(l[k], v);
      h[k] = fmax(h[k], v);
    }
  for (int k = 0; k < 3; ++k) {
    lo[k][threadIdx.x] = l[k];
    hi[k][threadIdx.x] = h[k];
  }
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int k = 0; k < 3; ++k) {
        lo[k][threadIdx.x] = fmin(lo[k][threadIdx.x], lo[k][threadIdx.x + w]);
        hi[k][threadIdx.x] = fmax(hi[k][threadIdx.x], hi[k][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 3) {
    part[blockIdx.x * 6 + threadIdx.x] = lo[threadIdx.x][0];
    part[blockIdx.x * 6 + 3 + threadIdx.x] = hi[threadIdx.x][0];
  }
}

__device__ __forceinline__ uint64_t spread2(uint64_t x) {  // 31 bits -> even positions
  x &= 0x7fffffffULL;
  x = (x | (x << 16)) & 0x0000FFFF0000FFFFULL;
  x = (x | (x << 8)) & 0x00FF00FF00FF00FFULL;
  x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0FULL;
  x = (x | (x << 2)) & 0x3333333333333333ULL;
  x = (x | (x << 1)) & 0x5555555555555555ULL;
  return x;
}

__device__ __forceinline__ uint64_t spread3(uint64_t x) {  // 21 bits -> every third position
  x &= 0x1fffffULL;
  x = (x | (x << 32)) & 0x1f00000000ffffULL;
  x = (x | (x << 16)) & 0x1f0000ff0000ffULL;
  x = (x | (x << 8)) & 0x100f00f00f00f00fULL;
  x = (x | (x << 4)) & 0x10c30c30c30c30c3ULL;
  x = (x | (x << 2)) & 0x1249249249249249ULL;
  return x;
}

__global__ void morton_kernel(const double* __restrict__ X, int64_t n, int d, int64_t npos, int64_t chunk, int world,
                              int rank, const double* __restrict__ part, uint64_t* __restrict__ keys,
                              int64_t* __restrict__ vals) {
  const int dd = d < 3 ? d : 3;
  __shared__ double lo[3], sc[3];
  if (threadIdx.x < 3) {
    double l = 1e300, h = -1e300;
    for (int b = 0; b < BB_BLOCKS; ++b) {
      l = fmin(l, part[b * 6 + threadIdx.x]);
      h = fmax(h, part[b * 6 + 3 + threadIdx.x]);
    }
    const int bits = dd == 1 ? 48 : (dd == 2 ? 24 : 16);  // 48-bit Morton code; round index above
    const double span = h > l ? h - l : 1.0;
    lo[threadIdx.x] = l;
    sc[threadIdx.x] = (double)((1ULL << bits) - 1) / span;
  }
  __syncthreads();
  for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < npos;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = (pos / chunk) * (int64_t)world * chunk + (int64_t)rank * chunk + pos % chunk;
    uint64_t key = ~0ULL;
    if (i < n) {
      uint64_t c[3] = {0, 0, 0};
      for (int k = 0; k < dd; ++k) {
        double v = (X[i * d + k] - lo[k]) * sc[k];
        v = v < 0 ? 0 : v;
        c[k] = (uint64_t)v;
      }
      if (dd == 1) key = c[0];
      else if (dd == 2) key = spread2(c[0]) | (spread2(c[1]) << 1);
      else key = spread3(c[0]) | (spread3(c[1]) << 1) | (spread3(c[2]) << 2);
      // positions are grouped by round (chunk-cyclic round = pos / chunk), Morton order inside a
      // round, so the Vecchia rows of round r can run as soon as round r of U is gathered
      key = ((uint64_t)(pos / chunk) << 48) | (key & 0xffffffffffffULL);
    }
    keys[pos] = key;
    vals[pos] = i;
  }
}

// ---- d > 3: Morton code over the K = min(d, 8) input dimensions along which the given
// neighbour sets are tightest (ranked by r_k = E[(x_ik - x_{N(i)_1,k})^2] / Var(x_k), the
// neighbours' spread relative to the data's), each scaled by its neighbour spread delta_k so that
// the Morton cells follow the shape of the neighbourhoods.  No hyperparameter enters: the
// neighbour sets carry the (ARD) correlation geometry.  Only the processing order changes (it is a
// permutation of independent rows), so the results do not depend on it beyond summation order. ----
constexpr int OD_MAX = 8;

__global__ void nbr_spread_kernel(const double* __restrict__ X, int64_t n, int d, const int32_t* __restrict__ nbr,
                                  int mv, double* __restrict__ acc) {
  __shared__ double red[3 * VIF_MAX_D];
  for (int t = threadIdx.x; t < 3 * VIF_MAX_D; t += blockDim.x) red[t] = 0.0;
  __syncthreads();
  double a[3 * VIF_MAX_D];
#pragma unroll
  for (int t = 0; t < 3 * VIF_MAX_D; ++t) a[t] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = nbr[i * mv];
#pragma unroll
    for (int k = 0; k < VIF_MAX_D; ++k)
      if (k < d) {
        const double x = X[i * d + k];
        a[3 * k + 1] += x;
        a[3 * k + 2] = fma(x, x, a[3 * k + 2]);
        if (j >= 0) {
          const double df = x - X[(int64_t)j * d + k];
          a[3 * k] = fma(df, df, a[3 * k]);
        }
      }
  }
#pragma unroll
  for (int t = 0; t < 3 * VIF_MAX_D; ++t)
    if (t < 3 * d) {
      double v = a[t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0) atomicAdd(&red[t], v);
    }
  __syncthreads();
  for (int t = threadIdx.x; t < 3 * d; t += blockDim.x) atomicAdd(&acc[t], red[t]);
}

// prm: [0..K) selected dims, [8..8+K) lo, [16..16+K) scale (to 48/K-bit cells), [24] = K (K <= 8)
__global__ void order_dims_kernel(const double* __restrict__ acc, int64_t n, int d, int kmax,
                                  double* __restrict__ prm) {
  if (threadIdx.x != 0) return;
  double r[VIF_MAX_D], sd[VIF_MAX_D], mu[VIF_MAX_D];
  bool used[VIF_MAX_D];
  for (int k = 0; k < d; ++k) {
    mu[k] = acc[3 * k + 1] / (double)n;
    const double var = fmax(acc[3 * k + 2] / (double)n - mu[k] * mu[k], 1e-300);
    sd[k] = sqrt(var);
    r[k] = acc[3 * k] / var;
    used[k] = false;
  }
  const int K = d < kmax ? d : kmax;
  const int bits = 48 / K;
  double width = 0.0;  // widest selected dimension in units of its neighbour spread
  int sel[OD_MAX];
  double dl[OD_MAX];
  for (int t = 0; t < K; ++t) {
    int best = -1;
    for (int k = 0; k < d; ++k)
      if (!used[k] && (best < 0 || r[k] < r[best])) best = k;
    used[best] = true;
    sel[t] = best;
    dl[t] = sqrt(acc[3 * best] / (double)n);
    if (!(dl[t] > 0.0)) dl[t] = sd[best] > 0.0 ? sd[best] : 1.0;
    width = fmax(width, 16.0 * sd[best] / dl[t]);
  }
  for (int t = 0; t < K; ++t) {
    prm[t] = (double)sel[t];
    prm[8 + t] = mu[sel[t]] - 8.0 * sd[sel[t]];
    prm[16 + t] = (double)((1ULL << bits) - 1) / (width * dl[t]);
  }
  prm[24] = (double)K;
}

__global__ void morton_nd_kernel(const double* __restrict__ X, int64_t n, int d, int64_t npos, int64_t chunk,
                                 int world, int rank, const double* __restrict__ prm, uint64_t* __restrict__ keys,
                                 int64_t* __restrict__ vals) {
  const int K = (int)prm[24];
  const int bits = 48 / K;
  const double cmax = (double)((1ULL << bits) - 1);
  for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < npos;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = (pos / chunk) * (int64_t)world * chunk + (int64_t)rank * chunk + pos % chunk;
    uint64_t key = ~0ULL;
    if (i < n) {
      uint64_t c[OD_MAX];
      for (int t = 0; t < K; ++t) {
        const double v = (X[i * d + (int)prm[t]] - prm[8 + t]) * prm[16 + t];
        c[t] = (uint64_t)fmin(fmax(v, 0.0), cmax);
      }
      uint64_t m = 0;
      for (int b = bits - 1; b >= 0; --b)
        for (int t = 0; t < K; ++t) m = (m << 1) | ((c[t] >> b) & 1ULL);
      key = ((uint64_t)(pos / chunk) << 48) | (m & 0xffffffffffffULL);
    }
    keys[pos] = key;
    vals[pos] = i;
  }
}

size_t order_temp_bytes(int64_t npos) { return (size_t)(16u << 20) + (size_t)npos * 4; }

cudaError_t launch_order(const double* X, int64_t n, int d, int64_t npos, int64_t chunk, int world, int rank,
                         double* bbox, uint64_t* keys, uint64_t* keys_alt, int64_t* vals, int64_t* vals_alt,
                         void* temp, size_t temp_bytes, int64_t** order_out, cudaStream_t s, const int32_t* nbr,
                         int mv) {
  static const char* nd_env = getenv("VIF_ORDER_ND");  // 0: the first three coordinates for every d
  const bool nd = d > 3 && nbr != nullptr && mv > 0 && n > 1 && !(nd_env && nd_env[0] == '0');
  if (nd) {
    cudaError_t e = cudaMemsetAsync(bbox, 0, 3 * VIF_MAX_D * sizeof(double), s);
    if (e != cudaSuccess) return e;
    nbr_spread_kernel<<<296, 256, 0, s>>>(X, n, d, nbr, mv, bbox);
    static const char* k_env = getenv("VIF_ORDER_K");  // A/B hook: dimensions in the code (1..8), default 8
    const int kmax = k_env ? (atoi(k_env) < 1 ? 1 : (atoi(k_env) > OD_MAX ? OD_MAX : atoi(k_env))) : OD_MAX;
    order_dims_kernel<<<1, 32, 0, s>>>(bbox, n, d, kmax, bbox + 64);
    morton_nd_kernel<<<296, 256, 0, s>>>(X, n, d, npos, chunk, world, rank, bbox + 64, keys, vals);
  } else {
    bbox_partial_kernel<<<BB_BLOCKS, 256, 0, s>>>(X, n, d, bbox);
    morton_kernel<<<296, 256, 0, s>>>(X, n, d, npos, chunk, world, rank, bbox, keys, vals);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  cub::DoubleBuffer<uint64_t> dk(keys, keys_alt);
  cub::DoubleBuffer<int64_t> dv(vals, vals_alt);
  size_t need = 0;
  e = cub::DeviceRadixSort::SortPairs(nullptr, need, dk, dv, npos, 0, 64, s);
  if (e != cudaSuccess) return e;
  if (need > temp_bytes) return cudaErrorMemoryAllocation;
  e = cub::DeviceRadixSort::SortPairs(temp, need, dk, dv, npos, 0, 64, s);
  if (e != cudaSuccess) return e;
  *order_out = dv.Current();
  return cudaGetLastError();
}

__global__ void sum_buffers_kernel(const double* __restrict__ src, int64_t count, int nbuf, int64_t stride,
                                   double* __restrict__ dst) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nbuf; ++b) s += src[b * stride + e];
    dst[e] = s;
  }
}

cudaError_t launch_sum_buffers(const double* src, int64_t count, int nbuf, int64_t stride, double* dst,
                               cudaStream_t s) {
  sum_buffers_kernel<<<296, 256, 0, s>>>(src, count, nbuf, stride, dst);
  return cudaGetLastError();
}

}  // namespace vif
