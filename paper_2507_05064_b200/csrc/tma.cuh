// tma.cuh -- Blackwell tile movement for the FP64 DMMA engines: TMA tensor maps (host), bulk tensor
// copies global -> shared completing on mbarriers (device), and the swizzled fragment addressing.
//
// Tiles of an FP64 row-major matrix are moved as boxes of 16 columns (128 B) x R rows with
// SWIZZLE_128B: inside every 1024-B atom of 8 box rows, the 16-B chunk c of row r lands at chunk
// c ^ (r & 7).  Element (r, c) of a box is therefore at byte
//     r * 128 + (((c >> 1) ^ (r & 7)) << 4) + (c & 1) * 8
// (swz_off).  Boxes that reach past the matrix (columns >= cols, rows >= rows) are zero-filled by
// the TMA unit, which is what the ragged tails of the contractions need.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace vif {

// ------------------------------------------------------------------ host: tensor maps
// 2-D map over a row-major FP64 matrix (rows x cols, leading dimension ld doubles, base 16-B
// aligned, ld * 8 a multiple of 16), box = 16 columns x box_rows rows, SWIZZLE_128B, zero fill.
cudaError_t make_tmap_f64(CUtensorMap* map, const double* base, uint64_t rows, uint64_t cols, uint64_t ld,
                          uint32_t box_rows);

// 4-D map over int8 digit slices stored [nkb][nslice][rows][32] (blocks of 32 k-values, each block holding
// every slice and row contiguously): box = {32 B of k, box_rows rows, all nslice slices, 1 block}, SWIZZLE_32B
// (the K-major tcgen05 operand layout, tc.cuh); one box reads nslice contiguous runs of box_rows x 32 B
cudaError_t make_tmap_i8_slices(CUtensorMap* map, const int8_t* base, uint64_t nkb, uint64_t rows, uint32_t nslice,
                                uint32_t box_rows);

// ------------------------------------------------------------------ device
__device__ __forceinline__ uint32_t swz_off(int r, int c) {
  return (uint32_t)(r * 128 + ((((c >> 1) ^ (r & 7)) & 7) << 4) + (c & 1) * 8);
}

// shared-memory loads by 32-bit shared address (keeps LDS, not generic LD, after address arithmetic)
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ double2 lds_f64x2(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// box (c0 = first column, r0 = first row) of `map` into shared memory `dst`, completing `bytes`
// (announced by mbar_expect_tx) on `bar`
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int r0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(smem_u32(bar))
      : "memory");
}

// the same with an L2 cache hint (createpolicy): EVICT_LAST keeps operands many CTAs re-read resident
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int c0, int r0, uint64_t* bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

}  // namespace vif
