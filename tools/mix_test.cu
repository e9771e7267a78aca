// Unit test of the mixed-precision per-point solver (mix_solve in k_vecchia.cuh) on random SPD
// blocks: one warp per matrix; prints max errors against an FP64 LU solve done on the host.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2507_05064_b200/csrc/k_vecchia.cuh"
using namespace vif;

template <int SP>
__global__ void mix_test_kernel(const double* Cs, const int* qs, double* a_out, double* D_out, int* ok_out, int nmat) {
  constexpr int CS = SP + 1;
  __shared__ double C[SP * CS];
  __shared__ double colbuf[2 * SP];
  const int lane = threadIdx.x;
  const int t = blockIdx.x;
  if (t >= nmat) return;
  const int q = qs[t];
  for (int e = lane; e < SP * CS; e += 32) C[e] = 0.0;
  __syncwarp();
  for (int e = lane; e < (q + 1) * (q + 1); e += 32) {
    const int r = e / (q + 1), c = e % (q + 1);
    if (c <= r) C[r * CS + c] = Cs[(size_t)t * SP * SP + r * SP + c];
  }
  __syncwarp();
  double a, Di;
  const bool ok = mix_solve<SP>(C, reinterpret_cast<float*>(colbuf), colbuf + SP, q, lane, a, Di);
  if (lane < SP) a_out[(size_t)t * SP + lane] = a;
  if (lane == 0) { D_out[t] = Di; ok_out[t] = ok; }
}

static void solve(int n, std::vector<double> A, std::vector<double> b, std::vector<double>& x) {
  // Gaussian elimination with partial pivoting, n x n row-major
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int r = k + 1; r < n; ++r) if (fabs(A[r * n + k]) > fabs(A[p * n + k])) p = r;
    for (int c = 0; c < n; ++c) std::swap(A[k * n + c], A[p * n + c]);
    std::swap(b[k], b[p]);
    for (int r = k + 1; r < n; ++r) {
      const double f = A[r * n + k] / A[k * n + k];
      for (int c = k; c < n; ++c) A[r * n + c] -= f * A[k * n + c];
      b[r] -= f * b[k];
    }
  }
  x.assign(n, 0.0);
  for (int k = n - 1; k >= 0; --k) {
    double s = b[k];
    for (int c = k + 1; c < n; ++c) s -= A[k * n + c] * x[c];
    x[k] = s / A[k * n + k];
  }
}

template <int SP>
int run(int nmat) {
  std::vector<double> Cs((size_t)nmat * SP * SP, 0.0);
  std::vector<int> qs(nmat);
  srand(7);
  auto rnd = [] { return (rand() / (double)RAND_MAX) * 2 - 1; };
  for (int t = 0; t < nmat; ++t) {
    const int q = t % SP;  // s = q + 1 <= SP
    qs[t] = q;
    const int s = q + 1, kk = s + 3;
    std::vector<double> G(s * kk);
    for (auto& g : G) g = rnd();
    for (int r = 0; r < s; ++r)
      for (int c = 0; c < s; ++c) {
        double v = 0;
        for (int k = 0; k < kk; ++k) v += G[r * kk + k] * G[c * kk + k];
        Cs[(size_t)t * SP * SP + r * SP + c] = v / kk + (r == c ? 0.05 : 0.0);
      }
  }
  double *dC, *da, *dD; int *dq, *dok;
  cudaMalloc(&dC, Cs.size() * 8); cudaMalloc(&da, (size_t)nmat * SP * 8); cudaMalloc(&dD, nmat * 8);
  cudaMalloc(&dq, nmat * 4); cudaMalloc(&dok, nmat * 4);
  cudaMemcpy(dC, Cs.data(), Cs.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dq, qs.data(), nmat * 4, cudaMemcpyHostToDevice);
  mix_test_kernel<SP><<<nmat, 32>>>(dC, dq, da, dD, dok, nmat);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("SP=%d cuda error %s\n", SP, cudaGetErrorString(e)); return 1; }
  std::vector<double> a((size_t)nmat * SP), D(nmat); std::vector<int> ok(nmat);
  cudaMemcpy(a.data(), da, a.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(D.data(), dD, nmat * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(ok.data(), dok, nmat * 4, cudaMemcpyDeviceToHost);
  double ea = 0, eD = 0; int nok = 0, shown = 0;
  for (int t = 0; t < nmat; ++t) {
    const int q = qs[t];
    std::vector<double> A(q * q), b(q), x;
    for (int r = 0; r < q; ++r) {
      b[r] = Cs[(size_t)t * SP * SP + q * SP + r];
      for (int c = 0; c < q; ++c) A[r * q + c] = Cs[(size_t)t * SP * SP + r * SP + c];
    }
    solve(q, A, b, x);
    double Dr = Cs[(size_t)t * SP * SP + q * SP + q];
    for (int r = 0; r < q; ++r) Dr -= b[r] * x[r];
    double amax = 1e-300, em = 0;
    for (int r = 0; r < q; ++r) { amax = fmax(amax, fabs(x[r])); em = fmax(em, fabs(a[(size_t)t * SP + r] - x[r])); }
    const double er = em / amax, eDr = fabs(D[t] - Dr) / Dr;
    nok += ok[t];
    if (ok[t]) { ea = fmax(ea, er); eD = fmax(eD, eDr); }
    if ((er > 1e-12 || eDr > 1e-12 || !ok[t]) && shown < 5) {
      ++shown;
      printf("  SP=%d t=%d q=%d ok=%d errA=%.3e errD=%.3e D=%.17g Dref=%.17g\n", SP, t, q, ok[t], er, eDr, D[t], Dr);
    }
  }
  printf("SP=%d: %d/%d ok, max rel err A %.3e, D %.3e\n", SP, nok, nmat, ea, eD);
  return 0;
}

int main() {
  run<8>(64);
  run<16>(64);
  run<24>(96);
  run<32>(256);
  return 0;
}
