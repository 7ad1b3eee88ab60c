// k_march_cf.cu -- instantiations of the marching level kernels (float, compress).
#include "k_march.cuh"

namespace hb {

void march_launch_cf(const LvArgs& A, const MarchLaunch& L, int cfg, int oid, cudaStream_t s) {
  march_launch_T<float, false>(A, L, cfg, oid, s);
}

}  // namespace hb
