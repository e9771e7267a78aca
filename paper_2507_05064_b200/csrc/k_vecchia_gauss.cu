// k_vecchia_gauss.cu -- instantiation of the K2+K3 vecchia kernels (k_vecchia.cuh) for FAM_GAUSS
// (one translation unit per covariance family so the build compiles them in parallel).
#include "k_vecchia.cuh"

namespace vif {
cudaError_t launch_vecchia_gauss(const VecchiaArgs& a, cudaStream_t s) { return launch_fam<FAM_GAUSS>(a, s); }
}  // namespace vif
