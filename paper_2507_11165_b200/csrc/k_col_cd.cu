// k_col_cd.cu -- compress / double instantiation of the column level kernel (k_col.cuh).
#include "k_col.cuh"

namespace hb {

template <>
int col_launch<false, double>(const LvArgs& A, unsigned blocks, int cfg, cudaStream_t s) {
  return col_launch_impl<false, double>(A, blocks, cfg, s);
}

}  // namespace hb
