// k_col_cf.cu -- compress / float instantiation of the column level kernel (k_col.cuh).
#include "k_col.cuh"

namespace hb {

template <>
int col_launch<false, float>(const LvArgs& A, unsigned blocks, int cfg, cudaStream_t s) {
  return col_launch_impl<false, float>(A, blocks, cfg, s);
}

}  // namespace hb
