// k_level_c.cu -- compress instantiations of the tiled level kernels (k_level.cuh).
#include "k_col.cuh"

namespace hb {


int launch_level_tiled_compress(const LevelGeom& g, const void* field, int prec, double* E, uint8_t* seq,
                                 uint32_t* obm, DevState* st, cudaStream_t s, int cfg) {
  LvArgs A{};
  A.field = field;
  A.E = E;
  A.seq = seq;
  A.obm = obm;
  A.st = st;
  if (const int n = launch_col<false>(g, A, prec, cfg, s)) return n;
  return launch_tiled<false>(g, A, prec, s) ? 1 : 0;
}

}  // namespace hb
