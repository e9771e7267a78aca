#include <cstdio>
#include <cmath>
#include "/root/repo/paper_2507_05064_b200/csrc/common.cuh"
__global__ void k(const double* x, double* y, int n) { int i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) y[i] = vif::rsqrt_nr(x[i]); }
int main() {
  const int n = 1 << 20; double *hx = new double[n], *hy = new double[n], *dx, *dy;
  for (int i = 0; i < n; ++i) hx[i] = pow(10.0, -12.0 + 24.0 * i / n) * (1.0 + 0.37 * ((i * 7919) % 1000) / 1000.0);
  cudaMalloc(&dx, n * 8); cudaMalloc(&dy, n * 8); cudaMemcpy(dx, hx, n * 8, cudaMemcpyHostToDevice);
  k<<<n / 256, 256>>>(dx, dy, n); cudaMemcpy(hy, dy, n * 8, cudaMemcpyDeviceToHost);
  double worst = 0; for (int i = 0; i < n; ++i) { double r = 1.0 / sqrt(hx[i]); double e = fabs(hy[i] - r) / r; if (e > worst) worst = e; }
  printf("{\"rsqrt_nr_max_rel_err\": %.3e}\n", worst); return 0; }
