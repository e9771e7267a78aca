// tc_i8_probe.cu -- tcgen05 kind::i8 bring-up on sm_100a: TMA 3-D boxes of int8 digit slices (SWIZZLE_32B,
// K-major), tcgen05.mma into TMEM int32 accumulators laid out by digit level (slice p of A times the
// concatenated slices 0..S-1-p of B lands at columns 64p..), tcgen05.ld epilogue.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tcp tools/tc_i8_probe.cu
//   ./tcp            correctness (one CTA, K = 512) + throughput (148 CTAs, L2-resident operands)
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
      exit(1);                                                                            \
    }                                                                                     \
  } while (0)

constexpr int S = 7;        // digit slices
constexpr int BM = 128;     // rows of A per tile (TMEM lanes)
constexpr int BN = 64;      // rows of B per tile (accumulator columns per level)
constexpr int BK = 32;      // bytes of k per stage (one MMA K)
constexpr int STAGES = 4;
constexpr int A_BYTES = S * BM * BK;  // 28 KB
constexpr int B_BYTES = S * BN * BK;  // 14 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(
          smem_u32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// K-major SWIZZLE_32B operand: rows of 32 B, 8-row atoms of 256 B stacked (SBO = 256 B), version 1
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
  d |= (uint64_t)(256 >> 4) << 32;     // SBO
  d |= (uint64_t)1 << 46;              // version (sm_100)
  d |= (uint64_t)6 << 61;              // SWIZZLE_32B
  return d;
}
// instruction descriptor: s8 x s8 -> s32, K-major both, M x N
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t dtm, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(dtm),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// One CTA per output tile; warps: 0 = TMA producer, 1 = MMA issuer (+ TMEM alloc), 2..5 = epilogue.
// A slices: tensor [S][rowsA][K] int8, B slices: [S][rowsB][K].  out: [S][BM][BN] int32 level sums.
__global__ void __launch_bounds__(192, 1)
    probe_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int nk, int reps,
                 int32_t* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* st = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1), mbar_init(&empty[i], 1);
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tbase;
  const int total = nk * reps;
  if (warp == 0 && lane == 0) {
    for (int it = 0; it < total; ++it) {
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
      uint8_t* a = st + s * STAGE_BYTES;
      mbar_expect_tx(&full[s], STAGE_BYTES);
      const int kb = it % nk;
      tma_3d(a, &tmA, kb * BK, blockIdx.x * 0, 0, &full[s]);
      tma_3d(a + A_BYTES, &tmB, kb * BK, 0, 0, &full[s]);
    }
  } else if (warp == 1) {
    for (int it = 0; it < total; ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t a0 = smem_u32(st + s * STAGE_BYTES), b0 = a0 + A_BYTES;
        const uint32_t acc = (it % nk) > 0 || (it / nk) > 0;  // reps accumulate (throughput mode)
#pragma unroll
        for (int p = 0; p < S; ++p) {
          // A slice p times B slices 0..S-1-p (contiguous in smem) -> level columns 64p ..
          int q0 = 0;
          while (q0 < S - p) {
            const int nq = (S - p - q0) > 4 ? 4 : (S - p - q0);
            // slice 0 of A initialises every level column on the first k block; the rest accumulate
            mma_i8(tmem + (uint32_t)(BN * (p + q0)), desc_sw32(a0 + p * BM * BK), desc_sw32(b0 + q0 * BN * BK),
                   idesc_i8(BM, BN * nq), acc | (p > 0));
            q0 += nq;
          }
        }
        mma_commit(&empty[s]);
        if (it == total - 1) mma_commit(tfull);
      }
      __syncwarp();
    }
  } else if (warp >= 2) {
    mbar_wait(tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    for (int L = 0; L < S; ++L) {
      uint32_t v[32];
      for (int h = 0; h < 2; ++h) {
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(L * BN + h * 32);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%"
            "18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (blockIdx.x == 0)
          for (int j = 0; j < 32; ++j) out[((size_t)L * BM + row) * BN + h * 32 + j] = (int32_t)v[j];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void make_map(CUtensorMap* m, void* base, int K, int rows, int box_rows) {
  static EncodeTiled enc = nullptr;
  if (!enc) {
    void* p;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    enc = (EncodeTiled)p;
  }
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)S};
  cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)K * rows};
  cuuint32_t box[3] = {BK, (cuuint32_t)box_rows, S};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
}

int main(int argc, char** argv) {
  const int K = 512, nk = K / BK;
  std::vector<int8_t> hA((size_t)S * BM * K), hB((size_t)S * BN * K);
  srand(1);
  for (auto& x : hA) x = (int8_t)((rand() % 256) - 128);
  for (auto& x : hB) x = (int8_t)((rand() % 256) - 128);
  int8_t *dA, *dB;
  int32_t* dO;
  CK(cudaMalloc(&dA, hA.size()));
  CK(cudaMalloc(&dB, hB.size()));
  CK(cudaMalloc(&dO, sizeof(int32_t) * S * BM * BN));
  CK(cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice));
  CUtensorMap mA, mB;
  make_map(&mA, dA, K, BM, BM);
  make_map(&mB, dB, K, BN, BN);
  const int smem = STAGES * STAGE_BYTES + 1024;
  CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe_kernel<<<1, 192, smem>>>(mA, mB, nk, 1, dO);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> hO((size_t)S * BM * BN);
  CK(cudaMemcpy(hO.data(), dO, hO.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int L = 0; L < S; ++L)
    for (int i = 0; i < BM; ++i)
      for (int j = 0; j < BN; ++j) {
        long long ref = 0;
        for (int p = 0; p <= L; ++p) {
          const int q = L - p;
          for (int k = 0; k < K; ++k)
            ref += (long long)hA[((size_t)p * BM + i) * K + k] * hB[((size_t)q * BN + j) * K + k];
        }
        const long long got = hO[((size_t)L * BM + i) * BN + j];
        if (got != ref && bad++ < 8) printf("mismatch L=%d i=%d j=%d got %lld ref %lld\n", L, i, j, got, ref);
      }
  printf("correctness: %ld mismatches of %d\n", bad, S * BM * BN);
  // throughput: 148 CTAs x reps passes over the same (L2-resident) K = 512
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int reps = argc > 1 ? atoi(argv[1]) : 200;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int w = 0; w < 2; ++w) {
    CK(cudaEventRecord(e0));
    probe_kernel<<<sms, 192, smem>>>(mA, mB, nk, reps, dO);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
  }
  CK(cudaGetLastError());
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double mac = (double)sms * reps * nk * (S * (S + 1) / 2) * (double)BM * BN * BK;
  printf("throughput: %.3f ms, %.1f int8 TOPS (2 ops/MAC), %.2f fp64-equiv TFLOP/s (28 products)\n", ms,
         2 * mac / ms / 1e9, 2 * mac / ms / 1e9 / (S * (S + 1) / 2));
  return 0;
}
