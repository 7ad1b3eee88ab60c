// k_march_df.cu -- instantiations of the marching level kernels (float, decompress).
#include "k_march.cuh"

namespace hb {

void march_launch_df(const LvArgs& A, const MarchLaunch& L, int cfg, int oid, cudaStream_t s) {
  march_launch_T<float, true>(A, L, cfg, oid, s);
}

}  // namespace hb
