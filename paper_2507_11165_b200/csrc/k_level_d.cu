// k_level_d.cu -- decompress instantiations of the tiled level kernels (k_level.cuh).
#include "k_col.cuh"

namespace hb {


int launch_level_tiled_decompress(const LevelGeom& g, const uint8_t* seq, const uint64_t* oidx, const double* oval,
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
  if (const int n = launch_col<true>(g, A, prec, cfg, s)) return n;
  return launch_tiled<true>(g, A, prec, s) ? 1 : 0;
}

}  // namespace hb
