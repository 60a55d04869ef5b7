// One (real type, n_subbands) instantiation unit of the fused block kernel,
// compiled once per (CB_REAL, CB_P) pair by the build (see build.py).
#include "cbessfm_launch.cuh"

#ifndef CB_REAL
#error "CB_REAL must be float or double"
#endif
#ifndef CB_P
#error "CB_P must be the cluster size (n_subbands)"
#endif

#define CB_CAT2(a, b, c) a##_##b##_##c
#define CB_CAT(a, b, c) CB_CAT2(a, b, c)

namespace cbessfm {
cudaError_t CB_CAT(launch, CB_REAL, CB_P)(const Params<CB_REAL>& prm, int q, int64_t nclusters,
                                          cudaStream_t stream, KernelInfo* info) {
  return launch_q<CB_REAL, CB_P>(prm, q, nclusters, stream, info);
}
}  // namespace cbessfm
