// k_march_plan.h -- launch plan of the marching level kernels (k_march.cuh)
#pragma once
#include <cstdlib>
#include "hb_kernels.h"

namespace hb {

struct LvArgs;

constexpr int MT = 32;       // column extent in y and z (lattice units)
constexpr int MH = MT / 2;   // odd positions per axis
constexpr int ME = MH + 3;   // even positions incl. the halo [Y0-2, Y0+MT+2]
constexpr int M_THREADS = 256;

// even-plane slot: eee (ME x ME), {y} (MH x ME), {z} (ME x MH), {yz} (MH x MH)
constexpr int SL_EEE = 0, SL_EY = ME * ME, SL_EZ = SL_EY + MH * ME, SL_EYZ = SL_EZ + ME * MH;
constexpr int SL_SIZE = SL_EYZ + MH * MH;
// odd plane: {x} (ME x ME), {xy} (MH x ME), {xz} (ME x MH); {xyz} is never re-read
constexpr int OD_X = 4 * SL_SIZE, OD_XY = OD_X + ME * ME, OD_XZ = OD_XY + MH * ME, OD_END = OD_XZ + ME * MH;
constexpr int M_STAGE = OD_END;  // orig / code staging, one ME*ME area per class of a phase
constexpr int M_SMEM_DOUBLES = M_STAGE + 4 * ME * ME;


struct MarchLaunch {
  unsigned blocks;
  int segp, ncz, ncy;
  size_t smem;
};

// 3D fields with every dim > 1 and enough columns x segments to fill the GPU
inline bool march_plan(const LevelGeom& g, MarchLaunch* L) {
  if (!(g.d[0] > 1 && g.d[1] > 1 && g.d[2] > 1)) return false;
  if (g.d[0] * g.d[1] * g.d[2] >= (1ll << 31) - (1ll << 24)) return false;
  if (!getenv("HB_MARCH")) return false;  // opt-in while it trails the tiled kernel
  const int ncy = (int)((g.D[1] + MT - 1) / MT), ncz = (int)((g.D[2] + MT - 1) / MT);
  const long long ncol = (long long)ncy * ncz;
  long long segp = (g.D[0] * ncol) / (148 * 8);  // aim at ~8 CTAs per SM
  segp = segp < 16 ? 16 : (segp > 128 ? 128 : segp);
  segp &= ~1ll;
  const long long nseg = (g.D[0] + segp - 1) / segp;
  if (ncol * nseg < 148 * 2) return false;  // too little parallelism: tiled kernel
  L->blocks = (unsigned)(ncol * nseg);
  L->segp = (int)segp;
  L->ncz = ncz;
  L->ncy = ncy;
  L->smem = (size_t)M_SMEM_DOUBLES * 8;
  return true;
}

void march_launch_cf(const LvArgs& A, const MarchLaunch& L, int cfg, int oid, cudaStream_t s);
void march_launch_cd(const LvArgs& A, const MarchLaunch& L, int cfg, int oid, cudaStream_t s);
void march_launch_df(const LvArgs& A, const MarchLaunch& L, int cfg, int oid, cudaStream_t s);
void march_launch_dd(const LvArgs& A, const MarchLaunch& L, int cfg, int oid, cudaStream_t s);

}  // namespace hb
