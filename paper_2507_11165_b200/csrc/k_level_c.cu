// k_level_c.cu -- compress instantiations of the tiled level kernels (k_level.cuh).
#include "k_level.cuh"
#include "k_march_plan.h"

namespace hb {


bool launch_level_tiled_compress(const LevelGeom& g, const void* field, int prec, double* E, uint8_t* seq,
                                 uint32_t* obm, DevState* st, cudaStream_t s, int cfg) {
  LvArgs A{};
  A.field = field;
  A.E = E;
  A.seq = seq;
  A.obm = obm;
  A.st = st;
  MarchLaunch ML;
  if (cfg >= 0 && march_plan(g, &ML)) {
    A.g = g;
    if (prec == 4)
      march_launch_cf(A, ML, cfg, order_id(g), s);
    else
      march_launch_cd(A, ML, cfg, order_id(g), s);
    return true;
  }
  return launch_tiled<false>(g, A, prec, s);
}

}  // namespace hb
