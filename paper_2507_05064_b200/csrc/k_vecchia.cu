// k_vecchia.cu -- K2 + K3 dispatch by covariance family (kernels in k_vecchia.cuh).
#include "kernels.h"

namespace vif {
cudaError_t launch_vecchia_m12(const VecchiaArgs& a, cudaStream_t s);
cudaError_t launch_vecchia_m32(const VecchiaArgs& a, cudaStream_t s);
cudaError_t launch_vecchia_m52(const VecchiaArgs& a, cudaStream_t s);
cudaError_t launch_vecchia_gauss(const VecchiaArgs& a, cudaStream_t s);

cudaError_t launch_vecchia(const VecchiaArgs& a, cudaStream_t s) {
  if (a.npts == 0) return cudaSuccess;
  switch (a.p.family) {
    case FAM_M12: return launch_vecchia_m12(a, s);
    case FAM_M32: return launch_vecchia_m32(a, s);
    case FAM_M52: return launch_vecchia_m52(a, s);
    default: return launch_vecchia_gauss(a, s);
  }
}
}  // namespace vif
