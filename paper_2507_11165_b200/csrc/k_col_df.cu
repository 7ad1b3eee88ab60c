// k_col_df.cu -- decompress / float instantiation of the column level kernel (k_col.cuh).
#include "k_col.cuh"

namespace hb {

template <>
int col_launch<true, float>(const LvArgs& A, unsigned blocks, int cfg, cudaStream_t s) {
  return col_launch_impl<true, float>(A, blocks, cfg, s);
}

}  // namespace hb
