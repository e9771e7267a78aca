// DMMA.8x8x4 latency / throughput vs independent accumulator chains per warp and warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void chain_kernel(double* out, int iters, long long* cycles) {
  double c[CH][2];
  double a = 1e-3 * threadIdx.x, b = 1e-3 * (threadIdx.x + 1);
#pragma unroll
  for (int j = 0; j < CH; ++j) c[j][0] = c[j][1] = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = t1 - t0;
}
template <int CH>
void run(int warps_per_sm, double* d, long long* cyc) {
  int iters = 2000;
  int sms = 148;
  int blocks = sms, tpb = 32 * warps_per_sm;
  chain_kernel<CH><<<blocks, tpb>>>(d, 10, cyc);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  chain_kernel<CH><<<blocks, tpb>>>(d, iters, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double flops = 2.0 * 256 * CH * (double)iters * blocks * warps_per_sm;
  printf("{\"chains\":%d,\"warps_per_sm\":%d,\"cycles_per_dmma_per_warp\":%.1f,\"tflops\":%.2f}\n", CH, warps_per_sm,
         (double)c / (iters * CH), flops / ms / 1e9);
}
int main() {
  double* d; long long* cyc; cudaMalloc(&d, 64); cudaMalloc(&cyc, 64);
  for (int w : {1, 2, 4, 8, 16}) { run<1>(w, d, cyc); run<2>(w, d, cyc); run<4>(w, d, cyc); run<10>(w, d, cyc); run<16>(w, d, cyc); }
  return 0;
}
