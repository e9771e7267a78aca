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

// D(8x8) += A(8x4) * B(4x8), FP64 tensor core
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = pred ? 16 : 0;  // src-size 0 => zero-fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
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
