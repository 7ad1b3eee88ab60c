// k_col_dd.cu -- decompress / double instantiation of the column level kernel (k_col.cuh).
#include "k_col.cuh"

namespace hb {

template <>
int col_launch<true, double>(const LvArgs& A, unsigned blocks, int cfg, cudaStream_t s) {
  return col_launch_impl<true, double>(A, blocks, cfg, s);
}

}  // namespace hb
