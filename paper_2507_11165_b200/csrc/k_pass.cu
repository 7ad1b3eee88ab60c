// k_pass.cu -- the levels of 3D fields as TMA-fed dependency passes.
//
// A level (predictor.py:264-304) visits the parity classes of its lattice in
// three dependency steps -- multidim {1,2,4} -> {3,5,6} -> {7}; seq1d {b0} ->
// {b1, b0|b1} -> {b2, b0|b2, b1|b2, 7} -- and each step is one launch that
// computes every target of its classes exactly once (no halo recompute, no
// intra-CTA phases).  Reconstructions of classes that a later step reads go
// to dense per-class f64 scratch arrays in HBM.  The level's source lattice
// (class 0) is the E array itself at level 1 (unit stride, even rows) and a
// dense gathered copy otherwise; levels >= 2 also write their targets into E,
// where they form the next level's lattice.
//
// A CTA owns an 8 x 8 x 32 (x, y, z) block of one class.  One elected thread
// issues one TMA box load per interpolation axis (the source class with a
// halo along that axis; out-of-range coordinates are zero-filled by the TMA
// unit and only ever feed unused stencil taps), completing on an mbarrier,
// while every thread loads its 8 originals (compress) or 8 codes
// (decompress) into registers.  Warps = y rows, lanes = z (consecutive in
// memory and in shared memory), each thread walks 8 targets along x.
//
// Reference: predictor.py:181-304 (prediction), :313-329 (quantize),
// :397-411 (replay), ordering.py:68-84 (Eq. 3 slot of every code).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "hb_common.cuh"
#include "hb_interp.cuh"
#include "hb_kernels.h"

namespace hb {

namespace {

constexpr int TY = 8, TZ = 32;
constexpr int TZH = TZ + 4;  // z-source box z0-2 .. z0+TZ+1 (even start, 16-byte multiple)
constexpr int T_THREADS = TY * 32;
// targets per thread along x (per step: 16 was measured slower for every K on
// B200 -- fewer resident blocks outweigh the amortised per-thread setup; the
// three-source step takes 4 so its three tiles leave room for 4 blocks / SM)
constexpr __host__ __device__ int txof(int k) { return k == 3 ? 4 : 8; }
// doubles per source tile slot: the largest of the x / y / z boxes
constexpr __host__ __device__ int cmax(int a, int b) { return a > b ? a : b; }
constexpr __host__ __device__ int slot_of(int tx) {
  return cmax((tx + 3) * TY * TZ, cmax(tx * (TY + 3) * TZ, tx * TY * TZH));
}

struct alignas(64) TMaps {
  CUtensorMap m[6];
};

struct TPassArgs {
  LevelGeom g;
  const void* field;
  double* E;
  uint8_t* seq;
  uint32_t* obm;
  const uint64_t* oidx;
  const double* oval;
  const unsigned long long* ocount;
  void* out;
  DevState* st;
  double* scr;        // class c (1..6) at scr + (c - 1) * cstride, rows padded to even length;
  long long cstride;  // gathered class 0 (when used) at scr + 6 * cstride
  int ncls, nbx;
  int pairs;          // decompress, multidim, even d2: odd-z classes write (z-1, z) output pairs
  int cls[4], axm[4];
  int map[4][3];      // TMA map of the j-th interpolation axis of class k
};

__device__ __forceinline__ int cdim1(const LevelGeom& g, int cls, int a) {
  return ((cls >> a) & 1) ? (int)(g.D[a] >> 1) : (int)((g.D[a] + 1) >> 1);
}

// ---- PTX wrappers: mbarrier + TMA
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"((unsigned)__cvta_generic_to_shared(b))
      : "memory");
}

// code 0 on decompress: the outlier value at linear index `lin`
// (predictor.py:400-405; orphan -> ArchiveError).  Rare, kept out of line.
__device__ __noinline__ double tp_outlier(const uint64_t* oidx, const double* oval, unsigned long long lin,
                                          unsigned long long cnt, bool& bad) {
  unsigned long long a0 = 0, a1 = cnt;
  while (a0 < a1) {
    const unsigned long long mid = (a0 + a1) >> 1;
    if (oidx[mid] < lin)
      a0 = mid + 1;
    else
      a1 = mid;
  }
  if (a0 < cnt && oidx[a0] == lin) return oval[a0];
  bad = true;
  return 0.0;
}

struct Acc {
  unsigned h127, h128, h129;
  bool bad, nf;
};

// shared-memory geometry of the box of an axis-`a` source: strides of the
// local x / y index and of one stencil step along a
struct Tile {
  int sx, sy, st;
};
__device__ __forceinline__ Tile tile_of(int a) {
  Tile t;
  if (a == 0) {
    t.sx = TY * TZ, t.sy = TZ, t.st = TY * TZ;
  } else if (a == 1) {
    t.sx = (TY + 3) * TZ, t.sy = TZ, t.st = TZ;
  } else {
    t.sx = TY * TZH, t.sy = TZH, t.st = 1;
  }
  return t;
}

// One thread: targets (x0 + i, y, z), i < nx.  INT: every stencil complete.
template <typename T, bool DEC, int K, bool LINEAR, bool INT, bool LV1, int TX = txof(K)>
__device__ __forceinline__ void tp_run(const TPassArgs& A, const double* tiles, int CLS, int AXM, int x0, int nx,
                                       int y, int z, int yl, int zl, long long lin, long long slot, const T* o,
                                       const uint8_t* cd, double eb, double two_eb, double inv_two_eb,
                                       unsigned long long ocount, unsigned* shist, Acc& acc) {
  const LevelGeom& g = A.g;
  const int odd0 = CLS & 1, odd1 = (CLS >> 1) & 1, odd2 = (CLS >> 2) & 1;
  const long long P0 = 2ll * x0 + odd0, P1 = 2ll * y + odd1, P2 = 2ll * z + odd2;
  const long long sg = LV1 ? 1 : g.s;
  const int kl0 = (int)g.kl[0], ks0 = (int)g.ks0;
  uint8_t* sq = A.seq + slot;
  // reconstruction destination (class 7 is never re-read)
  const int n1 = cdim1(g, CLS, 1), n2p = (cdim1(g, CLS, 2) + 1) & ~1;
  double* dp = CLS != 7 ? A.scr + (CLS - 1) * A.cstride + ((long long)x0 * n1 + y) * n2p + z : nullptr;
  const int dst0 = n1 * n2p;
  // levels >= 2: the target is also a point of the next level's lattice (E)
  double* ep = !LV1 ? A.E + ((P0 * sg) >> 1) * g.Ed[1] * g.Ed[2] + ((P1 * sg) >> 1) * g.Ed[2] + ((P2 * sg) >> 1)
                            : nullptr;
  const int ke0 = (int)g.ke[0];
  // per-axis shared-memory taps and (boundary) stencil classes
  const double* tb[K];
  int tsx[K], tst[K], sax[K], scls[K];
  {
    int m = AXM;
#pragma unroll
    for (int j = 0; j < K; j++) {
      const int a = __ffs(m) - 1;
      m &= m - 1;
      const Tile t = tile_of(a);
      sax[j] = a;
      tb[j] = tiles + j * slot_of(TX) + yl * t.sy + zl + (a == 2);  // z box starts one below the first tap
      tsx[j] = t.sx;
      tst[j] = t.st;
      scls[j] = (INT || a == 0) ? (LINEAR ? ST_MID : ST_CUBIC) : classify(a == 1 ? P1 : P2, g.D[a], 1, LINEAR);
    }
  }
#pragma unroll
  for (int i = 0; i < TX; i++) {
    if (i >= nx) break;
    double pv[K];
    int ov[K];
    double zpart = 0.0;  // the z-source value at z (the output partner of an odd-z target)
#pragma unroll
    for (int j = 0; j < K; j++) {
      int cls = scls[j];
      if (!INT && sax[j] == 0) cls = classify(P0 + 2 * i, g.D[0], 1, LINEAR);
      const double* q = tb[j] + i * tsx[j];
      const int t = tst[j];
      if (DEC && sax[j] == 2) zpart = q[t];
      const double v0 = (INT && LINEAR) ? 0.0 : q[0], v3 = (INT && LINEAR) ? 0.0 : q[3 * t];
      pv[j] = apply_stencil(INT ? (LINEAR ? ST_MID : ST_CUBIC) : cls, v0, q[t], q[2 * t], v3);
      ov[j] = INT ? (LINEAR ? 2 : 4) : stencil_order(cls);
    }
    const double pred = K == 1 ? pv[0] : combine_axes(K, pv, ov);
    double r;
    if (!DEC) {
      const double ov_ = (double)o[i];
      const int code = quantize_fast<sizeof(T) == 4>(ov_, pred, eb, two_eb, inv_two_eb, &r);
      sq[i * ks0] = (uint8_t)code;
      if (code == 128) {
        acc.h128++;
      } else if (code == 127) {
        acc.h127++;
      } else if (code == 129) {
        acc.h129++;
      } else {
        atomicAdd(&shist[code], 1u);
        if (code == 0) {  // outlier (non-finite originals always land here)
          const unsigned long long li = (unsigned long long)(lin + (long long)i * kl0);
          atomicOr(&A.obm[li >> 5], 1u << (li & 31));
          acc.bad |= !isfinite(ov_);
        }
      }
    } else {
      const int code = cd[i];
      if (code != 0)
        r = dequantize(pred, two_eb, code);
      else
        r = tp_outlier(A.oidx, A.oval, (unsigned long long)(lin + (long long)i * kl0), ocount, acc.bad);
      T* op = reinterpret_cast<T*>(A.out) + lin + (long long)i * kl0;
      if (!LV1) {
        // not an output point yet: the value lives on in E
      } else if (!A.pairs) {
        *op = (T)r;
        acc.nf |= !isfinite(r);
      } else if (odd2) {  // one aligned store covers (z-1, z); the even-z classes write nothing
        if (sizeof(T) == 4)
          *reinterpret_cast<float2*>(op - 1) = make_float2((float)zpart, (float)r);
        else
          *reinterpret_cast<double2*>(op - 1) = make_double2(zpart, r);
        acc.nf |= !isfinite(r) || !isfinite(zpart);
      }
    }
    if (dp) dp[i * dst0] = r;
    if (!LV1) ep[i * ke0] = r;
  }
}

// ---- level 1, multidim, class known at compile time: the hot loop.
// Everything per target that does not depend on the target is hoisted: the
// interpolation axes and their shared-memory tap strides are compile-time
// constants, the originals / codes are in registers, the code byte, the f64
// reconstruction and the output are written through per-thread pointers
// stepped by runtime strides, the rare paths (exact-division fallback of the
// quantizer, outliers, orphan codes) are out of line, and the 127/128/129
// histogram bins are counted branch-free in registers.

// floor(|err| / two_eb + 0.5) by IEEE division (quantize_fast's fallback)
__device__ __noinline__ double q_exact(double ae, double two_eb) {
  return floor(__dadd_rn(__ddiv_rn(ae, two_eb), 0.5));
}

__device__ __noinline__ void note_outlier(uint32_t* obm, unsigned long long li) {
  atomicOr(&obm[li >> 5], 1u << (li & 31));
}

template <bool CAST32>
__device__ __forceinline__ int quantize_lv1(double o, double p, double eb, double two_eb, double inv_two_eb,
                                            double* recon) {
  const double err = __dsub_rn(o, p);
  const double ae = fabs(err);
  const double u = __dadd_rn(__dmul_rn(ae, inv_two_eb), 0.5);
  double f = floor(u);
  const double fr = __dsub_rn(u, f);
  // the reciprocal product decides floor() unless the fraction is within
  // 2^-40 of an integer (hb_interp.cuh: quantize_fast); NaN fails both tests
  if (!(fabs(__dsub_rn(fr, 0.5)) < 0.5 - 0x1p-40) && !(u >= 200.5)) f = q_exact(ae, two_eb);
  const double q = copysign(f, err);
  const double r = __dadd_rn(p, __dmul_rn(two_eb, q));
  const double stored = CAST32 ? (double)__double2float_rn(r) : r;
  const bool ok = (f <= 127.0) && (fabs(__dsub_rn(o, stored)) <= eb);
  *recon = ok ? r : o;
  return ok ? (int)q + 128 : 0;
}

template <typename T, bool DEC, int K, bool LINEAR, bool INT, int TX, int CLS, bool LV1 = true>
__device__ __forceinline__ void tp_run_lv1(const TPassArgs& A, const double* tiles, int x0, int nx, int y, int z,
                                           int yl, int zl, long long lin, long long slot, const T* o,
                                           const uint8_t* cd, double eb, double two_eb, double inv_two_eb,
                                           unsigned long long ocount, unsigned* shist, Acc& acc) {
  const LevelGeom& g = A.g;
  constexpr int odd2 = (CLS >> 2) & 1;
  const long long P0 = 2ll * x0 + (CLS & 1), P1 = 2ll * y + ((CLS >> 1) & 1), P2 = 2ll * z + odd2;
  const int kl0 = (int)g.kl[0], ks0 = (int)g.ks0;
  uint8_t* sq = A.seq + slot;
  const int n1 = cdim1(g, CLS, 1), n2p = (cdim1(g, CLS, 2) + 1) & ~1;
  const int dst0 = n1 * n2p;
  double* dp = CLS != 7 ? A.scr + (CLS - 1) * A.cstride + ((long long)x0 * n1 + y) * n2p + z : nullptr;
  // levels >= 2: the target is also a point of the next level's lattice (E)
  const long long sg = LV1 ? 1 : g.s;
  double* ep = LV1 ? nullptr
                   : A.E + ((P0 * sg) >> 1) * g.Ed[1] * g.Ed[2] + ((P1 * sg) >> 1) * g.Ed[2] + ((P2 * sg) >> 1);
  const long long ke0 = g.ke[0];
  // axes of the class in ascending order, their tiles and tap strides
  constexpr int ax0 = (CLS & 1) ? 0 : ((CLS & 2) ? 1 : 2);
  constexpr int ax1 = K < 2 ? -1 : ((CLS & 1) ? ((CLS & 2) ? 1 : 2) : 2);
  constexpr int ax2 = K < 3 ? -1 : 2;
  constexpr int AX[3] = {ax0, ax1, ax2};
  const double* tb[K];
  int scls[K];
#pragma unroll
  for (int j = 0; j < K; j++) {
    const int a = AX[j];
    const Tile t = tile_of(a);
    tb[j] = tiles + j * slot_of(TX) + yl * t.sy + zl + (a == 2);
    scls[j] = (INT || a == 0) ? (LINEAR ? ST_MID : ST_CUBIC) : classify(a == 1 ? P1 : P2, g.D[a], 1, LINEAR);
  }
  T* op = DEC ? reinterpret_cast<T*>(A.out) + lin : nullptr;
  unsigned h7 = 0, h8 = 0, h9 = 0;
#pragma unroll
  for (int i = 0; i < TX; i++) {
    if (!INT && i >= nx) break;
    double pv[K];
    int ov[K];
    double zpart = 0.0;
#pragma unroll
    for (int j = 0; j < K; j++) {
      const int a = AX[j];
      const Tile t = tile_of(a);
      int c = scls[j];
      if (!INT && a == 0) c = classify(P0 + 2 * i, g.D[0], 1, LINEAR);
      const double* q = tb[j] + i * t.sx;
      if (DEC && a == 2) zpart = q[t.st];
      if (INT) {
        pv[j] = LINEAR ? apply_stencil(ST_MID, 0.0, q[t.st], q[2 * t.st], 0.0)
                       : apply_stencil(ST_CUBIC, q[0], q[t.st], q[2 * t.st], q[3 * t.st]);
        ov[j] = LINEAR ? 2 : 4;
      } else {
        pv[j] = apply_stencil(c, q[0], q[t.st], q[2 * t.st], q[3 * t.st]);
        ov[j] = stencil_order(c);
      }
    }
    const double pred = K == 1 ? pv[0] : (INT ? (K == 2 ? __dmul_rn(__dadd_rn(__dadd_rn(0.0, pv[0]), pv[1]), 0.5)
                                                        : __ddiv_rn(__dadd_rn(__dadd_rn(__dadd_rn(0.0, pv[0]), pv[1]), pv[2]), 3.0))
                                              : combine_axes(K, pv, ov));
    double r;
    if (!DEC) {
      const double ov_ = (double)o[i];
      const int code = quantize_lv1<sizeof(T) == 4>(ov_, pred, eb, two_eb, inv_two_eb, &r);
      sq[(long long)i * ks0] = (uint8_t)code;
      h7 += code == 127;
      h8 += code == 128;
      h9 += code == 129;
      if ((unsigned)(code - 127) > 2u) {
        atomicAdd(&shist[code], 1u);
        if (code == 0) {
          note_outlier(A.obm, (unsigned long long)(lin + (long long)i * kl0));
          acc.bad |= !isfinite(ov_);
        }
      }
    } else {
      const int code = cd[i];
      if (code != 0)
        r = dequantize(pred, two_eb, code);
      else
        r = tp_outlier(A.oidx, A.oval, (unsigned long long)(lin + (long long)i * kl0), ocount, acc.bad);
      T* opi = op + (long long)i * kl0;
      if (!LV1) {
        // not an output point yet: the value lives on in E
      } else if (!A.pairs) {
        *opi = (T)r;
        acc.nf |= !isfinite(r);
      } else if (odd2) {  // one aligned store covers (z-1, z); the even-z classes write nothing
        if (sizeof(T) == 4)
          *reinterpret_cast<float2*>(opi - 1) = make_float2((float)zpart, (float)r);
        else
          *reinterpret_cast<double2*>(opi - 1) = make_double2(zpart, r);
        acc.nf |= !isfinite(r) || !isfinite(zpart);
      }
    }
    if (CLS != 7) dp[(long long)i * dst0] = r;
    if (!LV1) ep[i * ke0] = r;
  }
  acc.h127 += h7;
  acc.h128 += h8;
  acc.h129 += h9;
}

// One CTA's tile of class k.  CLSC >= 0: that class is known at compile time
// and interpolates along all its odd axes (multidim) -- every parity test,
// tap stride and slot term folds; CLSC < 0: class and axes from the arguments
#define AXM_OF(c) (c)  // class-specialised bodies are multidim: every odd axis interpolates

// error bound, its reciprocal and the outlier count of the running launch
__shared__ double sh_eb[3];
__shared__ unsigned long long sh_ocount;

template <bool DEC>
__device__ __forceinline__ void sweep_consts(const TPassArgs& A) {
  sh_eb[0] = A.st->eb;
  sh_eb[1] = A.st->two_eb;
  sh_eb[2] = A.st->inv_two_eb;
  sh_ocount = DEC ? *A.ocount : 0;
}

// SWEEP: called from the persistent level-1 sweep (k_tsweep) -- the block
// coordinates come from the work item, the mbarrier was initialised once and
// completes phase `phase`, the histogram is flushed once per CTA at the end.
// Returns whether the block had work (and so used a barrier phase).
template <typename T, bool DEC, int K, bool LINEAR, bool LV1, int CLSC, int TX, bool SWEEP = false>
__device__ __forceinline__ bool tp_block(const TPassArgs& A, const TMaps& M, int k, int bx, double* tiles,
                                         unsigned* shist, uint64_t& bar, int by = -1, int bz = -1,
                                         unsigned phase = 0) {
  const LevelGeom& g = A.g;
  const int CLS = CLSC >= 0 ? CLSC : A.cls[k], AXM = CLSC >= 0 ? CLSC : A.axm[k];
  const int n0 = cdim1(g, CLS, 0), n1 = cdim1(g, CLS, 1), n2 = cdim1(g, CLS, 2);
  const int x0 = bx * TX, y0 = (SWEEP ? by : (int)blockIdx.y) * TY, z0 = (SWEEP ? bz : (int)blockIdx.x) * TZ;
  if (x0 >= n0 || y0 >= n1 || z0 >= n2) return false;  // block past this class's extent (uniform)
  const int yl = threadIdx.x >> 5, zl = threadIdx.x & 31;
  const int y = y0 + yl, z = z0 + zl;
  const int nx = min(TX, n0 - x0);
  double* s_eb = sh_eb;
  unsigned long long& s_ocount = sh_ocount;
  if (!SWEEP) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      s_eb[0] = A.st->eb;
      s_eb[1] = A.st->two_eb;
      s_eb[2] = A.st->inv_two_eb;  // __ddiv_rn(1.0, two_eb), computed once with eb
      s_ocount = DEC ? *A.ocount : 0;
    }
    if (!DEC)
      for (int i = threadIdx.x; i < 256; i += T_THREADS) shist[i] = 0;
    __syncthreads();
  }  // SWEEP: s_eb / s_ocount were set once at the start of the CTA (sweep_consts)
  if (threadIdx.x == 0) {
    unsigned bytes = 0;
    int m = AXM;
    for (int j = 0; j < K; j++) {
      const int a = __ffs(m) - 1;
      m &= m - 1;
      bytes += (a == 2 ? TX * TY * TZH : (a == 1 ? TX * (TY + 3) * TZ : (TX + 3) * TY * TZ)) * 8;
    }
    mbar_expect_tx(&bar, bytes);
    m = AXM;
    for (int j = 0; j < K; j++) {
      const int a = __ffs(m) - 1;
      m &= m - 1;
      const CUtensorMap* map = &M.m[A.map[k][j]];
      // the innermost start coordinate must be 16-byte aligned: the z box starts at z0 - 2
      tma_load_3d(tiles + j * slot_of(TX), map, z0 - 2 * (a == 2), y0 - (a == 1), x0 - (a == 0), &bar);
    }
  }
  // originals / codes of this thread's run, in flight with the boxes
  const bool live = y < n1 && z < n2;
  const int odd0 = CLS & 1, odd1 = (CLS >> 1) & 1, odd2 = (CLS >> 2) & 1;
  T o[TX];
  uint8_t cd[TX];
  // element index and Eq. 3 slot of the run's first target (ordering.py:68-84)
  long long lin, slot;
  if (LV1 && CLSC >= 0) {
    // level 1, class fixed: both are affine in (x0, y, z) -- with P = 2u + odd
    // and (P + 1) >> 1 = u + odd the Eq. 3 closed form collapses to
    // slot = S0 + x0 * ks0 + y * (2 D2 - [!odd0] ez) + z * (2 - [!odd0 && !odd1])
    const long long d12 = g.d[1] * g.d[2];
    lin = odd0 * d12 + odd1 * g.d[2] + odd2 + (long long)x0 * g.kl[0] + (long long)(y * 2) * g.d[2] + 2 * z;
    const long long s0 = g.prefix + odd0 * d12 + odd1 * g.d[2] + odd2 - odd0 * g.eyez -
                         (odd0 ? 0 : odd1 * g.ez + (odd1 ? 0 : odd2));
    slot = s0 + (long long)x0 * g.ks0 + (long long)y * (2 * g.d[2] - (odd0 ? 0 : g.ez)) +
           (long long)z * (2 - (!odd0 && !odd1));
  } else {
    const long long P0 = 2ll * x0 + odd0, P1 = 2ll * y + odd1, P2 = 2ll * z + odd2;
    const long long sg = LV1 ? 1 : g.s;
    lin = ((P0 * sg) * g.d[1] + P1 * sg) * g.d[2] + P2 * sg;
    slot = g.prefix + (P0 * g.D[1] + P1) * g.D[2] + P2 - ((P0 + 1) >> 1) * g.eyez;
    if (!odd0) {
      slot -= ((P1 + 1) >> 1) * g.ez;
      if (!odd1) slot -= (P2 + 1) >> 1;
    }
  }
  if (live) {
    if (!DEC) {
      const T* fp = reinterpret_cast<const T*>(A.field) + lin;
      const int kl0 = (int)g.kl[0];
#pragma unroll
      for (int i = 0; i < TX; i++)
        if (i < nx) o[i] = __ldg(fp + i * kl0);
    } else {
      const uint8_t* sq = A.seq + slot;
      const int ks0 = (int)g.ks0;
#pragma unroll
      for (int i = 0; i < TX; i++)
        if (i < nx) cd[i] = __ldg(sq + i * ks0);
    }
  }
  // complete stencils for every target of the block along every axis of AXM
  bool full = true;
  {
    const int lo[3] = {x0, y0, z0};
    const int hi[3] = {x0 + nx - 1, min(y0 + TY, n1) - 1, min(z0 + TZ, n2) - 1};
#pragma unroll
    for (int a = 0; a < 3; a++)
      if ((AXM >> a) & 1) {
        const long long Plo = 2ll * lo[a] + 1, Phi = 2ll * hi[a] + 1;
        full &= LINEAR ? (Phi + 1 < g.D[a]) : (Plo >= 3 && Phi + 3 < g.D[a]);
      }
  }
  const double eb = s_eb[0], two_eb = s_eb[1], inv_two_eb = s_eb[2];
  const unsigned long long ocount = s_ocount;
  Acc acc{0u, 0u, 0u, false, false};
  mbar_wait(&bar, phase);
  if constexpr (CLSC >= 0 && (CLSC == AXM_OF(CLSC))) {
    full &= nx == TX;  // the interior loop has no x-extent check
    if (live) {
      if (full)
        tp_run_lv1<T, DEC, K, LINEAR, true, TX, CLSC, LV1>(A, tiles, x0, nx, y, z, yl, zl, lin, slot, o, cd, eb,
                                                           two_eb, inv_two_eb, ocount, shist, acc);
      else
        tp_run_lv1<T, DEC, K, LINEAR, false, TX, CLSC, LV1>(A, tiles, x0, nx, y, z, yl, zl, lin, slot, o, cd, eb,
                                                            two_eb, inv_two_eb, ocount, shist, acc);
    }
  } else if (live) {
    if (full)
      tp_run<T, DEC, K, LINEAR, true, LV1, TX>(A, tiles, CLS, AXM, x0, nx, y, z, yl, zl, lin, slot, o, cd, eb, two_eb, inv_two_eb, ocount,
                                      shist, acc);
    else
      tp_run<T, DEC, K, LINEAR, false, LV1, TX>(A, tiles, CLS, AXM, x0, nx, y, z, yl, zl, lin, slot, o, cd, eb, two_eb, inv_two_eb,
                                       ocount, shist, acc);
  }
  if (DEC && __any_sync(0xffffffffu, acc.nf) && zl == 0) raise_flag(A.st, F_NONFINITE);
  if (__any_sync(0xffffffffu, acc.bad) && zl == 0) raise_flag(A.st, DEC ? F_ORPHAN : F_NONFINITE);
  if (!DEC) {
    const unsigned h7 = __reduce_add_sync(0xffffffffu, acc.h127), h8 = __reduce_add_sync(0xffffffffu, acc.h128),
                   h9 = __reduce_add_sync(0xffffffffu, acc.h129);
    if (zl == 0) {
      if (h7) atomicAdd(&shist[127], h7);
      if (h8) atomicAdd(&shist[128], h8);
      if (h9) atomicAdd(&shist[129], h9);
    }
    if (!SWEEP) {
      __syncthreads();
      for (int i = threadIdx.x; i < 256; i += T_THREADS)
        if (shist[i]) atomicAdd(&A.st->hist[i], (unsigned long long)shist[i]);
    }
  }
  return true;
}

// A dependency step.  C0..C2 >= 0: the step's classes (multidim, all odd
// axes) as compile-time constants, each CTA branching once to its class's
// specialised body; the classes stay in one launch with class-minor block
// order, so the source tiles they share are read from HBM once and from L2
// by the other classes.
template <typename T, bool DEC, int K, bool LINEAR, bool LV1, int C0 = -1, int C1 = -1, int C2 = -1,
          int TX = txof(K)>
__global__ void __launch_bounds__(T_THREADS, C0 >= 0 ? (C1 >= 0 && !DEC ? 3 : 4) : 2) k_tpass(const __grid_constant__ TPassArgs A,
                                                         const __grid_constant__ TMaps M) {
  extern __shared__ __align__(128) double tiles[];
  __shared__ unsigned shist[256];
  __shared__ __align__(8) uint64_t bar;
  // a single compile-time class per launch needs no class index
  const int bx = (C0 >= 0 && C1 < 0) ? (int)blockIdx.z : (int)blockIdx.z / A.ncls;
  const int k = (C0 >= 0 && C1 < 0) ? 0 : (int)blockIdx.z - bx * A.ncls;
  if constexpr (C0 < 0) {
    tp_block<T, DEC, K, LINEAR, LV1, -1, TX>(A, M, k, bx, tiles, shist, bar);
  } else {
    if (k == 0) {
      tp_block<T, DEC, K, LINEAR, LV1, C0, TX>(A, M, k, bx, tiles, shist, bar);
    } else if constexpr (C1 >= 0) {
      if (k == 1) {
        tp_block<T, DEC, K, LINEAR, LV1, C1, TX>(A, M, k, bx, tiles, shist, bar);
      } else if constexpr (C2 >= 0) {
        tp_block<T, DEC, K, LINEAR, LV1, C2, TX>(A, M, k, bx, tiles, shist, bar);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Level 1 (multidim) as ONE persistent sweep along axis 0.
//
// The seven per-class passes above each stream the whole volume, so the f64
// class arrays one step writes are evicted before the next step reads them,
// and the E lattice and both z-parities of every field sector are fetched by
// several launches (4.9x the algorithmic DRAM bytes at 512^3).  Here the
// class lattice is cut into x-slabs of SX planes and the work items (one
// 4 x 8 x 32 block of one class) are handed out by an atomic ticket in stage
// order
//     stage t:  step 1 (classes 1, 2, 4) of slab t,
//               step 2 (classes 3, 5, 6) of slab t - 2,
//               step 3 (class 7)         of slab t - 4,
// so a step reads what the previous step wrote about one stage earlier (a
// few MB per slab: still in L2) and the field rows shared by two classes of a
// slab are read from HBM once.  A step-q item of slab j waits (one thread,
// acquire loads) until step q-1 has finished slabs j-1..j+1 -- its stencils
// reach +-3 lattice points = +-2 class planes, never past the neighbour slab
// (SX >= 2).  Tickets are taken in list order by resident CTAs and every
// dependency points to a smaller ticket, so the sweep cannot deadlock for any
// grid size.  The bodies are the class-specialised blocks of k_tpass
// (tp_block), bit for bit the same arithmetic.
constexpr int SX = 4;     // class planes per slab
constexpr int SKEW = 2;   // stages between dependent steps

struct SweepArgs {
  TPassArgs A[3];  // step q: classes / maps of the step (plan_step)
  int nslab, nby, nbz, nitems;
  int one;         // one item per CTA (grid = nitems) instead of a persistent loop
  int I[3];        // items per slab of step q
  unsigned* ticket;
  unsigned* done;  // [3][nslab] finished items per (step, slab)
};
struct alignas(64) SweepMaps {
  TMaps M[3];
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__host__ __device__ __forceinline__ int stage_items(const SweepArgs& S, int t) {
  return (t < S.nslab ? S.I[0] : 0) + (t >= SKEW && t - SKEW < S.nslab ? S.I[1] : 0) +
         (t >= 2 * SKEW && t - 2 * SKEW < S.nslab ? S.I[2] : 0);
}

template <typename T, bool DEC, bool LINEAR>
__global__ void __launch_bounds__(T_THREADS, 4) k_tsweep(const __grid_constant__ SweepArgs S,
                                                        const __grid_constant__ SweepMaps SM) {
  extern __shared__ __align__(128) double tiles[];
  __shared__ unsigned shist[256];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int s_it;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (!DEC)
    for (int i = threadIdx.x; i < 256; i += T_THREADS) shist[i] = 0;
  unsigned ph = 0;
  int t = 0, tstart = 0;
  // thread 0: the next ticket is fetched while the current item runs, and
  // per step the prefix of predecessor slabs already seen complete is kept
  unsigned nxt = 0;
  int okp[3] = {-1, -1, -1};
  if (threadIdx.x == 0) {
    sweep_consts<DEC>(S.A[0]);
    nxt = atomicAdd(S.ticket, 1u);
  }
  for (int n = 0; !S.one || n < 1; n++) {
    if (threadIdx.x == 0) {
      s_it = (int)nxt;
      if (!S.one) nxt = atomicAdd(S.ticket, 1u);
    }
    __syncthreads();
    const int it = s_it;
    if (it >= S.nitems) break;
    if (S.one) {  // first stage at or after the item's lower bound: full stages hold Ifull items
      const int full = S.I[0] + S.I[1] + S.I[2];
      t = max(0, it / full - 2 * SKEW);
      tstart = 0;
      for (int u = 0; u < t; u++) tstart += stage_items(S, u);
    }
    while (it >= tstart + stage_items(S, t)) tstart += stage_items(S, t++);
    int l = it - tstart, q = 0, j = t;
    if (t < S.nslab && l < S.I[0]) {
      q = 0, j = t;
    } else {
      if (t < S.nslab) l -= S.I[0];
      if (t >= SKEW && t - SKEW < S.nslab && l < S.I[1]) {
        q = 1, j = t - SKEW;
      } else {
        if (t >= SKEW && t - SKEW < S.nslab) l -= S.I[1];
        q = 2, j = t - 2 * SKEW;
      }
    }
    if (q > 0 && threadIdx.x == 0 && okp[q] < min(S.nslab - 1, j + 1)) {
      const unsigned* d = S.done + (q - 1) * S.nslab;
      const unsigned need = (unsigned)S.I[q - 1];
      const int hi = min(S.nslab - 1, j + 1);
      for (int jj = okp[q] + 1; jj <= hi; jj++)
        while (ld_acquire(d + jj) < need) __nanosleep(32);
      okp[q] = hi;
      // the class arrays written by those items are read through the async (TMA) proxy
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    const int ncls = q == 1 ? 3 : (q == 0 ? 3 : 1);
    const int k = l % ncls;
    const int r = l / ncls;
    const int zb = r % S.nbz, yb = (r / S.nbz) % S.nby, xb = r / (S.nbz * S.nby);
    const int bx = j * (SX / 4) + xb;
    bool used;
    if (q == 0) {
      used = k == 0   ? tp_block<T, DEC, 1, LINEAR, true, 1, 4, true>(S.A[0], SM.M[0], 0, bx, tiles, shist, bar, yb, zb, ph & 1)
             : k == 1 ? tp_block<T, DEC, 1, LINEAR, true, 2, 4, true>(S.A[0], SM.M[0], 1, bx, tiles, shist, bar, yb, zb, ph & 1)
                      : tp_block<T, DEC, 1, LINEAR, true, 4, 4, true>(S.A[0], SM.M[0], 2, bx, tiles, shist, bar, yb, zb, ph & 1);
    } else if (q == 1) {
      used = k == 0   ? tp_block<T, DEC, 2, LINEAR, true, 3, 4, true>(S.A[1], SM.M[1], 0, bx, tiles, shist, bar, yb, zb, ph & 1)
             : k == 1 ? tp_block<T, DEC, 2, LINEAR, true, 5, 4, true>(S.A[1], SM.M[1], 1, bx, tiles, shist, bar, yb, zb, ph & 1)
                      : tp_block<T, DEC, 2, LINEAR, true, 6, 4, true>(S.A[1], SM.M[1], 2, bx, tiles, shist, bar, yb, zb, ph & 1);
    } else {
      used = tp_block<T, DEC, 3, LINEAR, true, 7, 4, true>(S.A[2], SM.M[2], 0, bx, tiles, shist, bar, yb, zb, ph & 1);
    }
    ph += used ? 1u : 0u;
    __syncthreads();  // tiles free for the next item; this item's stores issued
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(S.done + q * S.nslab + j, 1u);
    }
  }
  if (!DEC) {
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += T_THREADS)
      if (shist[i]) atomicAdd(&S.A[0].st->hist[i], (unsigned long long)shist[i]);
  }
}

// level 1 of decompress: the 2-lattice values (E) are output points too
template <typename T>
__global__ void k_even_out(const double* __restrict__ E, LevelGeom g, T* out, DevState* st) {
  const long long n = g.Ed[0] * g.Ed[1] * g.Ed[2];
  bool nf = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long hz = i % g.Ed[2], hy = (i / g.Ed[2]) % g.Ed[1], hx = i / (g.Ed[1] * g.Ed[2]);
    const double v = E[i];
    out[((2 * hx) * g.d[1] + 2 * hy) * g.d[2] + 2 * hz] = (T)v;
    nf |= !isfinite(v);
  }
  if (__any_sync(0xffffffffu, nf) && (threadIdx.x & 31) == 0) raise_flag(st, F_NONFINITE);
}

// class 0 of a level with stride s >= 2 (or odd E rows): dense copy of the
// 2s-lattice out of E, rows padded to even length (TMA global strides)
__global__ void k_gather0(const double* __restrict__ E, LevelGeom g, double* __restrict__ C0, long long n1, long long n2,
                          long long n2p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long w = i % n2p, v = (i / n2p) % n1, u = i / (n2p * n1);
    if (w >= n2) continue;
    C0[i] = E[((u * g.s) * g.Ed[1] + v * g.s) * g.Ed[2] + w * g.s];
  }
}

// ------------------------------------------------------------------ host
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  // thread-safe one-time lookup (a 'tried' flag set before the pointer let a
  // concurrent caller see no entry point and take another kernel path)
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
  }();
  return fn;
}

// 3D f64 array (n0, n1, n2) with rows of n2p doubles; box for an axis-`a` source
// Encoded maps are cached per thread: a context reuses its arena, so from the
// second call on every launch finds its maps here instead of re-encoding
// ~20 per level on the critical path between the tuner read-back and the
// level launches.
struct MapKey {
  const double* base;
  long long n0, n1, n2, n2p;
  int a, tx;
  bool operator==(const MapKey& o) const {
    return base == o.base && n0 == o.n0 && n1 == o.n1 && n2 == o.n2 && n2p == o.n2p && a == o.a && tx == o.tx;
  }
};
struct MapCache {
  static constexpr int CAP = 256;
  MapKey key[CAP];
  alignas(64) CUtensorMap map[CAP];
  int n = 0, next = 0;
};

bool encode_map(CUtensorMap* m, const double* base, long long n0, long long n1, long long n2, long long n2p, int a,
                int tx);

bool make_map(CUtensorMap* m, const double* base, long long n0, long long n1, long long n2, long long n2p, int a,
              int tx) {
  static thread_local MapCache* cache = new MapCache();
  const MapKey k{base, n0, n1, n2, n2p, a, tx};
  for (int i = 0; i < cache->n; i++)
    if (cache->key[i] == k) {
      *m = cache->map[i];
      return true;
    }
  if (!encode_map(m, base, n0, n1, n2, n2p, a, tx)) return false;
  const int slot = cache->n < MapCache::CAP ? cache->n++ : (cache->next++ % MapCache::CAP);
  cache->key[slot] = k;
  cache->map[slot] = *m;
  return true;
}

bool encode_map(CUtensorMap* m, const double* base, long long n0, long long n1, long long n2, long long n2p, int a,
                int tx) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dim[3] = {(cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)n0};
  const cuuint64_t str[2] = {(cuuint64_t)(n2p * 8), (cuuint64_t)(n1 * n2p * 8)};
  const cuuint32_t box[3] = {(cuuint32_t)(a == 2 ? TZH : TZ), (cuuint32_t)(a == 1 ? TY + 3 : TY),
                             (cuuint32_t)(a == 0 ? tx + 3 : tx)};
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dim, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Launch {
  TPassArgs A;
  TMaps M;
  int nmaps;
  bool gathered;  // class 0 read from the dense copy at scr + 6 * cstride
};

// map of class `cn` (0 = E) used as an axis-`a` source; reuses an identical one
int map_for(Launch& L, int cn, int a, int tx, int keys[6]) {
  const int key = cn * 4 + a;
  for (int i = 0; i < L.nmaps; i++)
    if (keys[i] == key) return i;
  if (L.nmaps >= 6) return -1;
  const LevelGeom& g = L.A.g;
  long long n[3];
  for (int b = 0; b < 3; b++) n[b] = ((cn >> b) & 1) ? g.D[b] >> 1 : (g.D[b] + 1) >> 1;
  bool ok;
  if (cn == 0 && !L.gathered)
    ok = make_map(&L.M.m[L.nmaps], L.A.E, g.Ed[0], g.Ed[1], g.Ed[2], g.Ed[2], a, tx);
  else if (cn == 0)
    ok = make_map(&L.M.m[L.nmaps], L.A.scr + 6 * L.A.cstride, n[0], n[1], n[2], (n[2] + 1) & ~1ll, a, tx);
  else
    ok = make_map(&L.M.m[L.nmaps], L.A.scr + (cn - 1) * L.A.cstride, n[0], n[1], n[2], (n[2] + 1) & ~1ll, a, tx);
  if (!ok) return -1;
  keys[L.nmaps] = key;
  return L.nmaps++;
}

// builds the maps of one dependency step (false = not expressible as TMA boxes)
bool plan_step(Launch& L, int K, const int* cls, const int* axm, int n, int tx_override = 0) {
  TPassArgs& A = L.A;
  A.ncls = n;
  L.nmaps = 0;
  int keys[6] = {-1, -1, -1, -1, -1, -1};
  long long mx = 0;
  const int tx = tx_override ? tx_override : txof(K);
  for (int k = 0; k < n; k++) {
    A.cls[k] = cls[k];
    A.axm[k] = axm[k];
    long long nd[3];
    for (int a = 0; a < 3; a++) nd[a] = ((cls[k] >> a) & 1) ? A.g.D[a] >> 1 : (A.g.D[a] + 1) >> 1;
    if (!nd[0] || !nd[1] || !nd[2]) return false;
    mx = std::max(mx, (nd[0] + tx - 1) / tx);
    int m = axm[k];
    for (int j = 0; j < K; j++) {
      const int a = __builtin_ctz(m);
      m &= m - 1;
      const int idx = map_for(L, cls[k] & ~(1 << a), a, tx, keys);
      if (idx < 0) return false;
      A.map[k][j] = idx;
    }
  }
  A.nbx = (int)mx;
  return true;
}

template <typename T, bool DEC, int K, bool LINEAR, bool LV1, int C0 = -1, int C1 = -1, int C2 = -1>
void launch_step(const Launch& L, cudaStream_t s, int* launches) {
  const TPassArgs& A = L.A;
  long long mz = 0, my = 0;
  for (int k = 0; k < A.ncls; k++) {
    const long long n1 = (A.cls[k] & 2) ? A.g.D[1] >> 1 : (A.g.D[1] + 1) >> 1;
    const long long n2 = (A.cls[k] & 4) ? A.g.D[2] >> 1 : (A.g.D[2] + 1) >> 1;
    mz = std::max(mz, (n2 + TZ - 1) / TZ);
    my = std::max(my, (n1 + TY - 1) / TY);
  }
  const size_t smem = (size_t)K * slot_of(txof(K)) * 8;
  static const bool attr = [&] {  // once per process, thread-safe (C++11 static init)
    cudaFuncSetAttribute((const void*)k_tpass<T, DEC, K, LINEAR, LV1, C0, C1, C2>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return true;
  }();
  (void)attr;
  const dim3 grid((unsigned)mz, (unsigned)my, (unsigned)(A.nbx * A.ncls));
  k_tpass<T, DEC, K, LINEAR, LV1, C0, C1, C2><<<grid, T_THREADS, smem, s>>>(A, L.M);
  (*launches)++;
}

long long class_stride(const LevelGeom& g);

// counters of the level-1 sweep live after the seven class arrays
unsigned* sweep_counters(const Launch& L) {
  return reinterpret_cast<unsigned*>(L.A.scr + 7 * L.A.cstride);
}
int sweep_slabs(const LevelGeom& g) { return (int)(((g.D[0] + 1) / 2 + SX - 1) / SX); }

// HB_SWEEP: 0 = seven per-class launches, 1 = sweep with one item per CTA,
// 2 = persistent sweep (one CTA per resident slot looping over tickets)
int sweep_mode() {
  static const int v = [] {
    const char* e = getenv("HB_SWEEP");
    return e ? atoi(e) : 0;
  }();
  return v;
}
bool sweep_on() { return sweep_mode() != 0; }

template <typename T, bool DEC, bool LINEAR>
bool launch_sweep(const Launch& base, cudaStream_t s, int* launches) {
  Launch L[3] = {base, base, base};
  const int c1[3] = {1, 2, 4}, c2[3] = {3, 5, 6}, c3[1] = {7};
  if (!plan_step(L[0], 1, c1, c1, 3, 4) || !plan_step(L[1], 2, c2, c2, 3, 4) || !plan_step(L[2], 3, c3, c3, 1, 4))
    return false;
  static_assert(SX % 4 == 0 && SX / 4 >= 1, "slab = whole 4-plane blocks");
  SweepArgs S;
  SweepMaps SM;
  for (int q = 0; q < 3; q++) {
    S.A[q] = L[q].A;
    SM.M[q] = L[q].M;
  }
  const LevelGeom& g = base.A.g;
  S.nslab = sweep_slabs(g);
  S.nby = (int)((((g.D[1] + 1) / 2) + TY - 1) / TY);
  S.nbz = (int)((((g.D[2] + 1) / 2) + TZ - 1) / TZ);
  S.I[0] = 3 * (SX / 4) * S.nby * S.nbz;
  S.I[1] = 3 * (SX / 4) * S.nby * S.nbz;
  S.I[2] = (SX / 4) * S.nby * S.nbz;
  S.nitems = S.nslab * (S.I[0] + S.I[1] + S.I[2]);
  S.ticket = sweep_counters(base);
  S.done = S.ticket + 1;
  cudaMemsetAsync(S.ticket, 0, sizeof(unsigned) * (1 + 3 * (size_t)S.nslab), s);
  const size_t smem = (size_t)3 * slot_of(4) * 8;
  static const int per_sm = [&] {
    cudaFuncSetAttribute((const void*)k_tsweep<T, DEC, LINEAR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    int v = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_tsweep<T, DEC, LINEAR>, T_THREADS, smem);
    return v < 1 ? 1 : v;
  }();
  S.one = sweep_mode() == 1;
  const int grid = S.one ? S.nitems : std::min(S.nitems, kSMs * per_sm);
  k_tsweep<T, DEC, LINEAR><<<grid, T_THREADS, smem, s>>>(S, SM);
  (*launches) += 2;
  return true;
}

// the three dependency steps of level 1; every map is built before anything
// is launched, so a shape TMA cannot express falls back cleanly
template <typename T, bool DEC, bool LINEAR, bool LV1>
bool run_passes(const Launch& base, int cfg, cudaStream_t s, int* launches) {
  Launch L[7] = {base, base, base, base, base, base, base};
  int K[3];
  if ((cfg & 2) == 0 && !LV1) {  // multidim, small levels: one launch per dependency step, class-specialised bodies
    const int c1[3] = {1, 2, 4}, c2[3] = {3, 5, 6}, c3[1] = {7};
    if (!plan_step(L[0], 1, c1, c1, 3) || !plan_step(L[1], 2, c2, c2, 3) || !plan_step(L[2], 3, c3, c3, 1))
      return false;
    launch_step<T, DEC, 1, LINEAR, LV1, 1, 2, 4>(L[0], s, launches);
    launch_step<T, DEC, 2, LINEAR, LV1, 3, 5, 6>(L[1], s, launches);
    launch_step<T, DEC, 3, LINEAR, LV1, 7>(L[2], s, launches);
    return true;
  }
  if ((cfg & 2) == 0 && LV1 && sweep_on() && launch_sweep<T, DEC, LINEAR>(base, s, launches)) return true;
  if ((cfg & 2) == 0 && !DEC) {  // multidim, level-1 compress: one launch per specialised class
    // (measured faster than the grouped launch below for the quantizing
    // kernels: a single class body keeps the instruction footprint small)
    const int order[7] = {1, 2, 4, 3, 5, 6, 7};
    for (int q = 0; q < 7; q++) {
      const int c = order[q];
      if (!plan_step(L[q], __builtin_popcount(c), &c, &c, 1)) return false;
    }
    launch_step<T, DEC, 1, LINEAR, LV1, 1>(L[0], s, launches);
    launch_step<T, DEC, 1, LINEAR, LV1, 2>(L[1], s, launches);
    launch_step<T, DEC, 1, LINEAR, LV1, 4>(L[2], s, launches);
    launch_step<T, DEC, 2, LINEAR, LV1, 3>(L[3], s, launches);
    launch_step<T, DEC, 2, LINEAR, LV1, 5>(L[4], s, launches);
    launch_step<T, DEC, 2, LINEAR, LV1, 6>(L[5], s, launches);
    launch_step<T, DEC, 3, LINEAR, LV1, 7>(L[6], s, launches);
    return true;
  }
  if ((cfg & 2) == 0) {  // multidim, level-1 decompress: class-specialised bodies, one launch per step
    const int c1[3] = {1, 2, 4}, c2[3] = {3, 5, 6}, c3[1] = {7};
    if (!plan_step(L[0], 1, c1, c1, 3) || !plan_step(L[1], 2, c2, c2, 3) || !plan_step(L[2], 3, c3, c3, 1))
      return false;
    launch_step<T, DEC, 1, LINEAR, LV1, 1, 2, 4>(L[0], s, launches);
    launch_step<T, DEC, 2, LINEAR, LV1, 3, 5, 6>(L[1], s, launches);
    launch_step<T, DEC, 3, LINEAR, LV1, 7>(L[2], s, launches);
    return true;
  }
  // seq1d along seq_order (predictor.py:267-280)
  const int b0 = 1 << base.A.g.seq_order[0], b1 = 1 << base.A.g.seq_order[1], b2 = 1 << base.A.g.seq_order[2];
  const int p1c[1] = {b0}, p1a[1] = {b0};
  const int p2c[2] = {b1, b0 | b1}, p2a[2] = {b1, b1};
  const int p3c[4] = {b2, b0 | b2, b1 | b2, 7}, p3a[4] = {b2, b2, b2, b2};
  (void)K;
  if (!plan_step(L[0], 1, p1c, p1a, 1) || !plan_step(L[1], 1, p2c, p2a, 2) || !plan_step(L[2], 1, p3c, p3a, 4))
    return false;
  for (int i = 0; i < 3; i++) launch_step<T, DEC, 1, LINEAR, LV1>(L[i], s, launches);
  return true;
}

template <typename T, bool DEC>
bool run_level(const Launch& L, int cfg, cudaStream_t s, int* launches) {
  if (L.A.g.level == 1)
    return (cfg & 1) ? run_passes<T, DEC, true, true>(L, cfg, s, launches)
                     : run_passes<T, DEC, false, true>(L, cfg, s, launches);
  return (cfg & 1) ? run_passes<T, DEC, true, false>(L, cfg, s, launches)
                   : run_passes<T, DEC, false, false>(L, cfg, s, launches);
}

long long class_stride(const LevelGeom& g) {
  long long n = ((g.D[0] + 1) / 2) * ((g.D[1] + 1) / 2) * (((g.D[2] + 1) / 2 + 1) & ~1ll);
  return (n + 15) & ~15ll;  // keeps every class array 128-byte aligned
}

// level 1 of a 3D field whose E rows are 16-byte multiples (TMA global strides)
bool tpass_ok(const LevelGeom& g, const double* E, const double* scr, int cfg) {
  return cfg >= 0 && scr && g.d[0] > 1 && g.d[1] > 1 && g.d[2] > 1 && (reinterpret_cast<uintptr_t>(E) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(scr) & 127) == 0 && !getenv("HB_TILED_LEVELS") && encode_fn() != nullptr;
}

// level 1 with even E rows reads class 0 straight from E; otherwise gather it
void prepare_class0(Launch& L, cudaStream_t s, int* launches) {
  const LevelGeom& g = L.A.g;
  L.gathered = !(g.level == 1 && (g.Ed[2] % 2) == 0);
  if (!L.gathered) return;
  const long long n0 = (g.D[0] + 1) / 2, n1 = (g.D[1] + 1) / 2, n2 = (g.D[2] + 1) / 2, n2p = (n2 + 1) & ~1ll;
  const long long n = n0 * n1 * n2p;
  const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 148 * 16);
  k_gather0<<<blocks, 256, 0, s>>>(L.A.E, g, L.A.scr + 6 * L.A.cstride, n1, n2, n2p, n);
  (*launches)++;
}

}  // namespace

size_t level_scratch_bytes(const uint64_t dims[3]) {
  // level 1: six class arrays + (odd E rows) the gathered lattice; a level
  // L >= 2 needs seven arrays of 1/8^(L-1) the size
  LevelGeom g;
  make_level_geom(dims, 1, &g);
  return (size_t)7 * class_stride(g) * 8 + sizeof(unsigned) * (4 + 3 * (size_t)sweep_slabs(g)) + 256;
}

int launch_level_pass_compress(const LevelGeom& g, const void* field, int prec, double* E, uint8_t* seq, uint32_t* obm,
                               double* scr, DevState* st, cudaStream_t s, int cfg) {
  if (!tpass_ok(g, E, scr, cfg)) return 0;
  Launch L{};
  L.A.g = g;
  L.A.field = field;
  L.A.E = E;
  L.A.seq = seq;
  L.A.obm = obm;
  L.A.st = st;
  L.A.scr = scr;
  L.A.cstride = class_stride(g);
  L.gathered = !(g.level == 1 && (g.Ed[2] % 2) == 0);
  {  // every map must be expressible before anything is launched
    Launch t = L;
    const int c1[1] = {1};
    if (!plan_step(t, 1, c1, c1, 1)) return 0;
  }
  int n = 0;
  prepare_class0(L, s, &n);  // harmless if the passes below cannot run (scratch only)
  if (!(prec == 4 ? run_level<float, false>(L, cfg, s, &n) : run_level<double, false>(L, cfg, s, &n))) return 0;
  return n;
}

int launch_level_pass_decompress(const LevelGeom& g, const uint8_t* seq, const uint64_t* oidx, const double* oval,
                                 const unsigned long long* ocount_dev, double* E, void* out, int prec, double* scr,
                                 DevState* st, cudaStream_t s, int cfg) {
  if (!tpass_ok(g, E, scr, cfg)) return 0;
  Launch L{};
  L.A.g = g;
  L.A.E = E;
  L.A.seq = const_cast<uint8_t*>(seq);
  L.A.oidx = oidx;
  L.A.oval = oval;
  L.A.ocount = ocount_dev;
  L.A.out = out;
  L.A.st = st;
  L.A.scr = scr;
  L.A.cstride = class_stride(g);
  L.A.pairs = g.level == 1 && (cfg & 2) == 0 && (g.d[2] % 2) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  L.gathered = !(g.level == 1 && (g.Ed[2] % 2) == 0);
  {  // every map must be expressible before anything is launched
    Launch t = L;
    const int c1[1] = {1};
    if (!plan_step(t, 1, c1, c1, 1)) return 0;
  }
  int n = 0;
  prepare_class0(L, s, &n);  // harmless if the passes below cannot run (scratch only)
  if (!(prec == 4 ? run_level<float, true>(L, cfg, s, &n) : run_level<double, true>(L, cfg, s, &n))) return 0;
  if (g.level == 1 && !L.A.pairs) {  // class 0 (the E lattice) is written by its odd-z partners when pairing
    const long long ne = g.Ed[0] * g.Ed[1] * g.Ed[2];
    const unsigned blocks = (unsigned)std::min<long long>((ne + 255) / 256, 148 * 16);
    if (prec == 4)
      k_even_out<float><<<blocks, 256, 0, s>>>(E, g, reinterpret_cast<float*>(out), st);
    else
      k_even_out<double><<<blocks, 256, 0, s>>>(E, g, reinterpret_cast<double*>(out), st);
    n++;
  }
  return n;
}

}  // namespace hb
