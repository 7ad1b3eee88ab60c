// k_level_d.cu -- decompress instantiations of the tiled level kernels (k_level.cuh).
#include "k_level.cuh"
#include "k_march_plan.h"

namespace hb {


bool launch_level_tiled_decompress(const LevelGeom& g, const uint8_t* seq, const uint64_t* oidx, const double* oval,
                                   const unsigned long long* ocount_dev, double* E, void* out, int prec, DevState* st,
                                   cudaStream_t s, int cfg) {
  LvArgs A{};
  A.E = E;
  A.seq = const_cast<uint8_t*>(seq);
  A.oidx = oidx;
  A.oval = oval;
  A.ocount = ocount_dev;
  A.out = out;
  A.st = st;
  MarchLaunch ML;
  if (cfg >= 0 && march_plan(g, &ML)) {
    A.g = g;
    if (prec == 4)
      march_launch_df(A, ML, cfg, order_id(g), s);
    else
      march_launch_dd(A, ML, cfg, order_id(g), s);
    return true;
  }
  return launch_tiled<true>(g, A, prec, s);
}

}  // namespace hb
