// k_march_dd.cu -- instantiations of the marching level kernels (double, decompress).
#include "k_march.cuh"

namespace hb {

void march_launch_dd(const LvArgs& A, const MarchLaunch& L, int cfg, int oid, cudaStream_t s) {
  march_launch_T<double, true>(A, L, cfg, oid, s);
}

}  // namespace hb
