// k_level_c.cu -- compress instantiations of the tiled level kernels (k_level.cuh).
#include "k_level.cuh"

namespace hb {

bool launch_level_tiled_compress(const LevelGeom& g, const void* field, int prec, double* E, uint8_t* seq,
                                 uint32_t* obm, DevState* st, cudaStream_t s) {
  LvArgs A{};
  A.field = field;
  A.E = E;
  A.seq = seq;
  A.obm = obm;
  A.st = st;
  return launch_tiled<false>(g, A, prec, s);
}

}  // namespace hb
