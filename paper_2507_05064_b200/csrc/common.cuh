// common.cuh -- device helpers shared by the libvif kernels (product path only).
//
// FP64 on sm_100a: tcgen05 has no .kind::f64, so FP64 tensor work is the warp-level
// DMMA (mma.sync.m8n8k4.f64, SASS DMMA.8x8x4) measured at 37.1 TF/s on B200 (148 SMs x
// 64 FMA/clk x 1.965 GHz), vs 33.9 TF/s for a DFMA loop.  Fragment layout of m8n8k4.f64:
//   A (8x4, row):  lane l holds A[l/4][l%4]
//   B (4x8, col):  lane l holds B[l%4][l/4]
//   C (8x8):       lane l holds C[l/4][2*(l%4) + {0,1}]
// For a Gram block U_R U_S^T both fragments are "row l/4, k l%4" of the two row blocks, so a
// single load serves as A for one tile and as B for another.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <unordered_map>

#ifndef VIF_MAX_D
#define VIF_MAX_D 16
#endif

namespace vif {

// Covariance parameters in kernel-argument form (reading c1: k = sigma2 f(r), r = ||(a-b)/lambda||).
struct CovParams {
  double sigma2;
  double nugget;
  double jitter;
  int32_t d;
  int32_t family;
  double inv_ls[VIF_MAX_D];
};

enum { FAM_M12 = 0, FAM_M32 = 1, FAM_M52 = 2, FAM_GAUSS = 3 };

// 1/sqrt(x) for x > 0: MUFU.RSQ64H seed + two Newton steps (relative error ~1 ulp).  Inline: the
// libdevice sqrt/div/rsqrt carry an out-of-line slow path whose CALL forces register spills in
// the unrolled per-point Cholesky.  x <= 0 gives NaN/inf, which the callers test for.
// One third-order step y (1 + r/2 + 3r^2/8), r = 1 - x y^2, instead of two Newton steps: the seed
// error e (~2^-23) becomes O(e^3), and the dependent FP64 chain is 4 ops instead of 6 (each
// dependent FP64 op waits ~16 cycles per DMMA-issuing warp on the SMSP: tools/dmma_mix.cu).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double r = fma(-x * y, y, 1.0);
  const double p = fma(0.375, r, 0.5);
  return fma(y * r, p, y);
}

__device__ __forceinline__ double sqrt_nr(double x) { return x > 0.0 ? x * rsqrt_nr(x) : 0.0; }

// single-precision approximate square root (MUFU.SQRT, no slow path) for index arithmetic
__device__ __forceinline__ float sqrtf_fast(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// f(r) as a function of r^2 (reading c1)
template <int FAM>
__device__ __forceinline__ double cov_f(double r2) {
  if (FAM == FAM_M12) {
    return exp(-sqrt_nr(r2));
  } else if (FAM == FAM_M32) {
    const double t = 1.7320508075688772 * sqrt_nr(r2);
    return (1.0 + t) * exp(-t);
  } else if (FAM == FAM_M52) {
    const double t = 2.23606797749979 * sqrt_nr(r2);
    return (1.0 + t + (5.0 / 3.0) * r2) * exp(-t);
  } else {
    return exp(-r2);
  }
}

__device__ __forceinline__ double sqdist(const double* __restrict__ a, const double* __restrict__ b,
                                         const CovParams& p) {
  double r2 = 0.0;
#pragma unroll 4
  for (int k = 0; k < p.d; ++k) {
    const double t = (a[k] - b[k]) * p.inv_ls[k];
    r2 = fma(t, t, r2);
  }
  return r2;
}

template <int FAM>
__device__ __forceinline__ double cov(const double* __restrict__ a, const double* __restrict__ b,
                                      const CovParams& p) {
  return p.sigma2 * cov_f<FAM>(sqdist(a, b, p));
}

// ---- fast covariance for the hot loops (same function as cov<FAM>, fewer FP64 instructions) ----
// Every scalar FP64 instruction competes with the DMMAs for the SMSP's FP64 unit, so the kernel
// evaluations of K1a / K2 use: coordinates pre-scaled by fam_scale / lambda_k (t^2 = sum of
// squared differences, t = sqrt(2 nu) r; Gaussian: t = r^2), a 5-op square root, and
// sigma1^2 e^{-t} from a 64-entry shared-memory table tbl[j] = sigma1^2 2^{-j/64}:
//   t = (64 k' + j) ln2 / 64 + rho, |rho| <= ln2 / 128,  e^{-rho} by a degree-5 polynomial
//   (truncation error rho^6 / 720 < 4e-17), 2^{-k'} applied to the exponent field.
// ~20 FP64 instructions per Matern-3/2 evaluation instead of ~37 (libdevice exp + generic sqdist).
template <int FAM>
__host__ __device__ constexpr double fam_scale() {
  return FAM == FAM_M32 ? 1.7320508075688772 : (FAM == FAM_M52 ? 2.23606797749979 : 1.0);
}

// shared-memory table init (threads 0..63 of the block)
__device__ __forceinline__ void exp_table_init(double* tbl, double sigma2, int tid) {
  if (tid < 64) tbl[tid] = sigma2 * exp2(-(double)tid / 64.0);
}

// sqrt(t2) for t2 >= 0: MUFU.RSQ64H seed y, t = a (1 + r/2 + 3 r^2 / 8), a = t2 y, r = 1 - a y
// (third-order correction of the ~2^-23 seed); zero and denormal t2 give 0 (integer test).
__device__ __forceinline__ double sqrt_fast(double t2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t2));
  const double a = t2 * y;
  const double r = fma(-a, y, 1.0);
  const double pp = fma(0.375, r, 0.5);
  const double t = fma(a * r, pp, a);
  return __double2hiint(t2) < 0x00100000 ? 0.0 : t;
}

// sigma1^2 e^{-t} for t >= 0 (tbl as above)
__device__ __forceinline__ double sig2_exp_neg(double t, const double* __restrict__ tbl) {
  t = fmin(t, 1000.0);  // e^{-1000} underflows anyway; keeps k in range
  const double kd = fma(t, 0x1.71547652b82fep+6, 6755399441055744.0);  // round(64 t / ln 2) + 1.5 2^52
  const int k = __double2loint(kd);
  const double kf = kd - 6755399441055744.0;
  double rho = fma(-kf, 0x1.62e42fee00000p-7, t);  // ln2/64 = hi + lo (hi: 21 trailing zero bits, so
  rho = fma(-kf, 0x1.a39ef35793c76p-39, rho);      // kf * hi is exact for k < 2^21)
  double q = fma(rho, -1.0 / 120.0, 1.0 / 24.0);
  q = fma(rho, q, -1.0 / 6.0);
  q = fma(rho, q, 0.5);
  q = fma(rho, q, -1.0);
  q = rho * q;  // e^{-rho} - 1
  const double T = tbl[k & 63];
  const double e = fma(T, q, T);
  const int n = k >> 6;
  const int hi = __double2hiint(e);
  // 2^{-n} on the exponent field; results below the normal range are flushed to 0
  return (((hi >> 20) & 0x7ff) > n + 1) ? __hiloint2double(hi - (n << 20), __double2loint(e)) : 0.0;
}

// k(a, b) from pre-scaled coordinates (a~ = fam_scale * a / lambda)
template <int FAM>
__device__ __forceinline__ double cov_fast(const double* __restrict__ a, const double* __restrict__ b, int d,
                                           const double* __restrict__ tbl) {
  double t2;
  {
    const double d0 = a[0] - b[0];
    t2 = d0 * d0;
    for (int k = 1; k < d; ++k) {
      const double dk = a[k] - b[k];
      t2 = fma(dk, dk, t2);
    }
  }
  if (FAM == FAM_GAUSS) return sig2_exp_neg(t2, tbl);
  const double t = sqrt_fast(t2);
  const double E = sig2_exp_neg(t, tbl);
  if (FAM == FAM_M12) return E;
  if (FAM == FAM_M32) return fma(E, t, E);
  return fma(E, fma(t2, 1.0 / 3.0, t), E);  // (1 + t + t^2/3) E
}

// processing position p of a rank -> global row (rows sharded chunk-cyclically over `world` ranks)
__device__ __forceinline__ int64_t pos_to_row(int64_t p, int64_t chunk, int world, int rank) {
  return (p / chunk) * (int64_t)world * chunk + (int64_t)rank * chunk + p % chunk;
}

// D(8x8) += A(8x4) * B(4x8), FP64 tensor core
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = pred ? 16 : 0;  // src-size 0 => zero-fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---- shared-memory mbarrier helpers (CTA scope) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Opt `fn` into `bytes` of dynamic shared memory (host).  The attribute belongs to the function
// (per device), so the record is keyed on (device, function pointer) -- never a static per call
// site, which would be shared by every kernel a templated launcher passes through it.  Below 40 KB
// nothing is needed (48 KB default minus the static arrays the kernels declare).
inline cudaError_t smem_optin(const void* fn, size_t bytes) {
  if (bytes <= 40 * 1024) return cudaSuccess;
  static std::mutex mu;
  static std::unordered_map<uint64_t, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t key = reinterpret_cast<uint64_t>(fn) ^ ((uint64_t)dev << 56);
  std::lock_guard<std::mutex> lk(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done[key] = bytes;
  return e;
}
template <typename K>
inline cudaError_t smem_optin(K* fn, size_t bytes) {
  return smem_optin(reinterpret_cast<const void*>(fn), bytes);
}

// Device-side status shared by all kernels of one evaluation.
struct DevStatus {
  unsigned long long bad_row;    // min failing point index of a residual block (ULLONG_MAX = none)
  unsigned long long bad_input;  // validation: min offending row (ULLONG_MAX = none)
  int km_fail;                   // Cholesky of K_m failed
  int m_fail;                    // Cholesky of M failed
  int bad_z;                     // non-finite inducing point
  int pad;
};

}  // namespace vif
