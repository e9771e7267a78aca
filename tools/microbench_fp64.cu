// Microbenchmarks that decide the FP64 kernel design on sm_100a:
//   DFMA vs DMMA (mma.sync .f64 shapes) throughput, and row-gather bandwidth
//   from HBM vs L2.  Standalone; prints one JSON object per line.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\":\"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = threadIdx.x * 1e-3 + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = fma(acc[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += acc[j];
  if (s == 12345.678) out[0] = s;
}

template <int SHAPE>
__global__ void dmma_kernel(double* out, int iters) {
  // SHAPE 0: m8n8k4, 1: m16n8k4, 2: m16n8k8, 3: m16n8k16
  double a[8], b[4], c[4][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = 1e-3 * (threadIdx.x + j);
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = 1e-3 * (threadIdx.x - j);
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[t][j] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (SHAPE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a[t]), "d"(b[t]));
      } else if (SHAPE == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a[t]), "d"(a[t+1]), "d"(b[t]));
      } else if (SHAPE == 2) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                     : "d"(a[t]), "d"(a[t+1]), "d"(a[t+2]), "d"(a[t+3]), "d"(b[t]), "d"(b[(t+1)&3]));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[t][j];
  if (s == 12345.678) out[0] = s;
}

// gather: each warp copies rows idx[r] (row_len doubles) and sums them (forces reads)
__global__ void gather_kernel(const double* __restrict__ src, const int* __restrict__ idx, int nrows_total,
                              int row_len, double* out) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  double acc = 0;
  for (int r = warp; r < nrows_total; r += nw) {
    const double2* p = reinterpret_cast<const double2*>(src + (size_t)idx[r] * row_len);
    for (int c = lane; c < row_len / 2; c += 32) {
      double2 v = __ldg(p + c);
      acc += v.x + v.y;
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("{\"device\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_per_block_optin\":%zu,\"clock_khz\":%d}\n",
         prop.name, sms, prop.l2CacheSize, (size_t)prop.sharedMemPerBlockOptin, prop.clockRate);
  double* dout;
  CK(cudaMalloc(&dout, 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  // DFMA
  for (int tpb : {256, 512}) {
    int blocks = sms * (2048 / tpb);
    int iters = 20000;
    dfma_kernel<<<blocks, tpb>>>(dout, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      dfma_kernel<<<blocks, tpb>>>(dout, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 16 * iters * (double)blocks * tpb;
    printf("{\"bench\":\"dfma\",\"tpb\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", tpb, best, flops / best / 1e9);
  }
  // DMMA
  auto run_dmma = [&](int shape, const char* name, double fma_per_mma) -> int {
    for (int wpb : {4, 8, 16}) {
      int tpb = wpb * 32;
      int blocks = sms * (32 / wpb);
      int iters = 4000;
      void (*k)(double*, int) = shape == 0 ? dmma_kernel<0> : shape == 1 ? dmma_kernel<1> : shape == 2 ? dmma_kernel<2> : dmma_kernel<3>;
      k<<<blocks, tpb>>>(dout, 10);
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k<<<blocks, tpb>>>(dout, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double flops = 2.0 * fma_per_mma * 4 * iters * (double)blocks * wpb;
      printf("{\"bench\":\"dmma_%s\",\"warps_per_block\":%d,\"blocks\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", name, wpb, blocks, best, flops / best / 1e9);
    }
    return 0;
  };
  if (run_dmma(0, "m8n8k4", 8 * 8 * 4)) return 1;
  if (run_dmma(1, "m16n8k4", 16 * 8 * 4)) return 1;
  if (run_dmma(2, "m16n8k8", 16 * 8 * 8)) return 1;
  if (run_dmma(3, "m16n8k16", 16 * 8 * 16)) return 1;
  // Gather bandwidth
  for (size_t src_rows : {(size_t)1000000, (size_t)12000}) {
    for (int row_len : {512, 208}) {
      size_t bytes = src_rows * row_len * 8;
      double* src; CK(cudaMalloc(&src, bytes));
      CK(cudaMemset(src, 0, bytes));
      int nr = 4000000;
      std::vector<int> h(nr);
      std::mt19937 rng(1);
      for (int i = 0; i < nr; ++i) h[i] = rng() % src_rows;
      int* didx; CK(cudaMalloc(&didx, nr * 4));
      CK(cudaMemcpy(didx, h.data(), nr * 4, cudaMemcpyHostToDevice));
      int blocks = sms * 8;
      gather_kernel<<<blocks, 256>>>(src, didx, nr, row_len, dout);
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        gather_kernel<<<blocks, 256>>>(src, didx, nr, row_len, dout);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double gb = (double)nr * row_len * 8 / 1e9;
      printf("{\"bench\":\"gather\",\"src_MB\":%.0f,\"row_bytes\":%d,\"ms\":%.3f,\"GBps\":%.0f}\n", bytes / 1e6, row_len * 8, best, gb / best * 1e3);
      cudaFree(src); cudaFree(didx);
    }
  }
  return 0;
}
