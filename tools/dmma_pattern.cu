// DMMA throughput for the GEMM inner-loop pattern (warp tile 4x4 of 8x8 tiles, fresh fragments each
// k-step from shared memory or registers) vs warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int MODE>  // 0: register fragments rotated; 1: LDS.64 fragments per k-step; 2: LDS.128 k-pair
__global__ void pat_kernel(double* out, int iters) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1e-3 * i;
  __syncthreads();
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0;
  const int lane = threadIdx.x & 31;
  const double* base = sm + (threadIdx.x >> 5) * 128 + lane;
  double ra[4], rb[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) { ra[t] = base[t * 8]; rb[t] = base[t * 8 + 32]; }
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], ra[a], rb[b]);
#pragma unroll
      for (int t = 0; t < 4; ++t) { double x = ra[t]; ra[t] = rb[t]; rb[t] = x; }
    } else if (MODE == 1) {
      double af[4], bf[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) { af[t] = base[(it & 7) * 16 + t * 40]; bf[t] = base[(it & 7) * 16 + t * 40 + 8]; }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    } else {
      double2 af[4], bf[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        af[t] = *reinterpret_cast<const double2*>(sm + ((it & 7) * 64 + t * 48 + 2 * lane) % 4000);
        bf[t] = *reinterpret_cast<const double2*>(sm + ((it & 7) * 64 + t * 48 + 2 * lane + 16) % 4000);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a].x, bf[b].x);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a].y, bf[b].y);
    }
  }
  double s = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) s += acc[a][b][0] + acc[a][b][1];
  if (s == 1.2345) out[0] = s;
}
template <int MODE>
void run(int wps, double* d) {
  int iters = MODE == 2 ? 1000 : 2000;
  int blocks = 148, tpb = 32 * wps;
  pat_kernel<MODE><<<blocks, tpb>>>(d, 10);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  pat_kernel<MODE><<<blocks, tpb>>>(d, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double dm = 16.0 * (MODE == 2 ? 2 : 1) * iters;
  double flops = 2.0 * 256 * dm * blocks * wps;
  printf("{\"mode\":%d,\"warps_per_sm\":%d,\"tflops\":%.2f}\n", MODE, wps, flops / ms / 1e9);
}
int main() {
  double* d; cudaMalloc(&d, 64);
  for (int w : {4, 8, 16}) { run<0>(w, d); run<1>(w, d); run<2>(w, d); }
  return 0;
}
