// k_march_cd.cu -- instantiations of the marching level kernels (double, compress).
#include "k_march.cuh"

namespace hb {

void march_launch_cd(const LvArgs& A, const MarchLaunch& L, int cfg, int oid, cudaStream_t s) {
  march_launch_T<double, false>(A, L, cfg, oid, s);
}

}  // namespace hb
