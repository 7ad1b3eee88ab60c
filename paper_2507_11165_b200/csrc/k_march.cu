// k_march.cu -- a whole multidim level in ONE launch: every CTA marches along
// axis 0 through a (y, z) column of the level lattice, keeping a rolling
// window of planes in shared memory.
//
// Level L (stride s, lattice D = ceil(d/s)) predicts every lattice point with
// an odd coordinate from the all-even points (predictor.py:264-304).  Seen
// along axis 0 the dependency steps of the multidim scheme split into
//   even planes P0 = 2j :  c2 (y odd), c4 (z odd)   <- the 2-lattice (E) of plane j
//                          c6 (y, z odd)            <- c4 (along y), c2 (along z)
//   odd planes P0 = 2m+1:  c1                       <- E of planes m-1 .. m+2 (along x)
//                          c3 (x, y odd)            <- c2 of planes m-1..m+2, c1 (along y)
//                          c5 (x, z odd)            <- c4 of planes m-1..m+2, c1 (along z)
//                          c7                       <- c6 of planes m-1..m+2, c5 (y), c3 (z)
// (class bit a = axis a odd; a class interpolates along each of its odd
// axes from the class with that bit cleared, predictor.py:282-296).  Every
// in-plane stencil reaches +-3 lattice points, so a CTA owning a TY x TZ
// core recomputes a 3-point (y, z) halo of the classes its core reads in
// plane, and nothing else: planes stream through rings in shared memory.
// Phase k of the march (one barrier between its two halves):
//   1: c2, c4 of even plane k | c1 of odd plane k-2 | c7 of odd plane k-3
//   2: c6 of even plane k     | c3, c5 of odd plane k-2
// while the inputs of phase k+1 are in flight: the E plane k+1 and the field
// rectangles of even plane k+1 / odd plane k-1 (one TMA box each, on an
// mbarrier; cp.async where TMA cannot describe the layout), and on
// decompress the code bytes of phase k+1 (register prefetch).  Per launch HBM
// sees the field once, E once (+ the halo), and the codes once; the
// per-class f64 round trips of the dependency-pass kernels (k_pass.cu) do
// not exist.
//
// Axis 0 is split into segments of `seg` even planes (grid z); a segment
// recomputes the three even planes around it (js-1, je, je+1) as halo.
//
// Bit-exactness: the same stencil / combine / quantizer device functions as
// every other level kernel (hb_interp.cuh: predictor.py:209-256, :313-329,
// :397-411); the Eq. 3 slot of every code (ordering.py:68-84).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "hb_common.cuh"
#include "hb_interp.cuh"
#include "hb_kernels.h"

namespace hb {

namespace {

constexpr int MT = 256;  // threads per CTA

template <int TY_, int TZ_, int TSZ>
struct MG {
  static constexpr int TY = TY_, TZ = TZ_, HY = TY / 2, HZ = TZ / 2, EY = HY + 3, EZ = HZ + 3;
  // arrays with even z (E, c1, c2, c3) keep rows of EZP doubles, element ez
  // at column ez + 1 (the layout of the E TMA box, which starts one lattice
  // point early so its first coordinate is 16-byte aligned); odd-z arrays
  // (c4, c5, c6) rows of HZ
  static constexpr int EZP = EZ + 1;
  static constexpr int NE = EY * EZP, N2 = HY * EZP, N4 = EY * HZ, N6 = HY * HZ;
  // ring slots padded to 128 bytes (TMA destinations)
  static constexpr int pad16(int n) { return (n + 15) & ~15; }
  static constexpr int SE = pad16(NE), S2 = pad16(N2), S4 = pad16(N4), S6 = pad16(N6);
  // ring depths (powers of two): E planes k-3..k, class planes k-3..k (c6:
  // k-4..k-1 while c6 of k is written after them); the inputs of phase k+1
  // are staged after the phase's middle barrier into the slots of k-3
  static constexpr int RE = 4, RC = 4;
  // field rectangles: rows P1 = Y0-2 .. Y0+TY+2, columns P2 = Z0-4 .. Z0+TZ+3
  static constexpr int FR = TY + 5, FC = TZ + 8, NF = FR * FC;
  static constexpr int SF = TSZ ? ((NF * TSZ + 127) & ~127) / TSZ : 0;
  static constexpr int RFE = 2, RFO = 2;  // even planes k, k+1; odd planes k-2, k-1 (k-3 before the middle barrier)
  static constexpr int oE = 0, oC2 = oE + RE * SE, oC4 = oC2 + RC * S2, oC6 = oC4 + RC * S4,
                       oC1 = oC6 + RC * S6, oC3 = oC1 + SE, oC5 = oC3 + S2, dbl = oC5 + S4;
  static constexpr size_t fbytes = (size_t)(RFE + RFO) * SF * TSZ;
  static constexpr size_t bytes = (size_t)dbl * 8 + fbytes;
};

struct alignas(64) MarchArgs {
  CUtensorMap fmap;  // field (3D, element = T), box FC x FR x 1
  CUtensorMap emap;  // E (3D f64), box EZP x EY x 1
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
  int seg;       // even planes per axis-0 segment
  int nep, nop;  // even / odd planes of the lattice
  int ftma, etma;  // field / E planes arrive by TMA (else cp.async)
};

struct QC {
  double eb, two_eb, inv;
  unsigned long long ocount;
  unsigned long long hp;  // per-thread counts of codes 127 / 128 / 129, 21 bits each
  bool bad, nf;
};

// ---- PTX wrappers: cp.async, mbarrier, TMA
template <int B>
__device__ __forceinline__ void cp_async(void* dst, const void* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d), "l"(ok ? src : nullptr), "n"(B),
               "r"(ok ? B : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count));
}
// expect_tx before the copies it covers, one plain arrive after all of them
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
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

// code 0 on decompress (predictor.py:400-405; orphan -> ArchiveError)
__device__ __noinline__ double m_outlier(const uint64_t* oidx, const double* oval, unsigned long long lin,
                                         unsigned long long cnt, bool* bad) {
  unsigned long long a0 = 0, a1 = cnt;
  while (a0 < a1) {
    const unsigned long long mid = (a0 + a1) >> 1;
    if (oidx[mid] < lin)
      a0 = mid + 1;
    else
      a1 = mid;
  }
  if (a0 < cnt && oidx[a0] == lin) return oval[a0];
  *bad = true;
  return 0.0;
}

// ------------------------------------------------------------ class geometry
// Class C's items in a tile form a [NY][NZ] grid: odd axes carry the core
// (HY / HZ points), even axes the core plus a 3-point halo (EY / EZ, item 0 is
// the point before the core).  Arrays with even z (E, c1, c2, c3) keep rows of
// EZP doubles with item iz at column iz + 1 (the layout of the E TMA box,
// which starts one lattice point early so its first coordinate is 16-byte
// aligned); odd-z arrays (c4, c5, c6) rows of HZ.
template <class G, int C>
struct CG {
  static constexpr bool yo = (C >> 1) & 1, zo = (C >> 2) & 1, xo = C & 1;
  static constexpr int PITCH = zo ? G::HZ : G::EZP, OFFZ = zo ? 0 : 1;
  __device__ static int py(int iy) { return 2 * iy + (yo ? 1 : -2); }
  __device__ static int pz(int iz) { return 2 * iz + (zo ? 1 : -2); }
  __device__ static int e(int iy, int iz) { return iy * PITCH + iz + OFFZ; }
  // this thread's core item (thread t: z = t & 15, row = t >> 4)
  __device__ static int cy(int row) { return row + (yo ? 0 : 1); }
  __device__ static int cz(int z) { return z + (zo ? 0 : 1); }
};

struct PlaneCtx {
  int P0;      // lattice coordinate along axis 0
  bool owned;  // plane belongs to this CTA's segment (codes / outputs are emitted)
  bool live;   // plane is computed at all
  int xcls;    // stencil class along axis 0 (odd planes)
  int sbase;   // Eq. 3 slot of lattice point (P0, 0, 0) without the in-plane terms
  int lbase;   // element index of (P0, 0, 0)
  long long ebase;  // E index of (P0, 0, 0) (levels >= 2)
};

// prediction of item (iy, iz) of class C (predictor.py:209-256): along x from
// the four axis-0 source planes, along y / z from the in-plane sources
template <class G, int C, bool LINEAR, bool FAST>
__device__ __forceinline__ double predict(const LevelGeom& g, int xcls, int P1, int P2, int iy, int iz,
                                          const double* x0, const double* x1, const double* x2, const double* x3,
                                          const double* ys, const double* zs) {
  using cg = CG<G, C>;
  constexpr int K = (int)cg::xo + (int)cg::yo + (int)cg::zo;
  constexpr int ICLS = LINEAR ? ST_MID : ST_CUBIC;
  constexpr int jx = 0, jy = (int)cg::xo, jz = (int)cg::xo + (int)cg::yo;
  const int e = cg::e(iy, iz);
  double pv[3] = {0.0, 0.0, 0.0};
  int ov[3] = {0, 0, 0};
  if (cg::xo) {
    const int c = FAST ? ICLS : xcls;
    pv[jx] = apply_stencil(c, (FAST && LINEAR) ? 0.0 : x0[e], x1[e], x2[e], (FAST && LINEAR) ? 0.0 : x3[e]);
    ov[jx] = stencil_order(c);
  }
  if (cg::yo) {  // rows iy .. iy+3 of the same-z-parity array with y even
    const int c = FAST ? ICLS : classify(P1, g.D[1], 1, LINEAR);
    const double* q0 = ys + e;
    pv[jy] = apply_stencil(c, (FAST && LINEAR) ? 0.0 : q0[0], q0[cg::PITCH], q0[2 * cg::PITCH],
                           (FAST && LINEAR) ? 0.0 : q0[3 * cg::PITCH]);
    ov[jy] = stencil_order(c);
  }
  if (cg::zo) {  // items iz .. iz+3 of the even-z array, row iy
    const int c = FAST ? ICLS : classify(P2, g.D[2], 1, LINEAR);
    const double* q0 = zs + iy * G::EZP + iz + 1;
    pv[jz] = apply_stencil(c, (FAST && LINEAR) ? 0.0 : q0[0], q0[1], q0[2], (FAST && LINEAR) ? 0.0 : q0[3]);
    ov[jz] = stencil_order(c);
  }
  return K == 1 ? pv[0] : combine_axes(K, pv, ov);
}

// in-plane part of the Eq. 3 slot (ordering.py:68-84)
template <int C>
__device__ __forceinline__ int slot_item(const LevelGeom& g, int P1, int P2) {
  int s = P1 * (int)g.D[2] + P2;
  if (!(C & 1)) {  // even plane: the 2-lattice rows / points of the plane are skipped
    s -= ((P1 + 1) >> 1) * (int)g.ez;
    if (!((C >> 1) & 1)) s -= (P2 + 1) >> 1;
  }
  return s;
}

// quantize (predictor.py:313-329) or replay (:397-411) one item; emit = the
// code / output belongs to this CTA.  Returns the reconstruction.
template <typename T, bool DEC, bool LV1, class G, int C>
__device__ __forceinline__ double finish(const MarchArgs& A, const PlaneCtx& pc, int Y0, int Z0, int P1, int P2,
                                         bool emit, double pred, const T* fs, int code_in, QC& q, unsigned* shist) {
  const LevelGeom& g = A.g;
  const int s = (int)g.s;
  double rv;
  if (!DEC) {
    const T o = fs[(P1 - Y0 + 2) * G::FC + (P2 - Z0 + 4)];
    const int code = quantize_fast<sizeof(T) == 4>((double)o, pred, q.eb, q.two_eb, q.inv, &rv);
    if (emit) {
      A.seq[pc.sbase + slot_item<C>(g, P1, P2)] = (uint8_t)code;
      const unsigned d = (unsigned)code - 127u;
      if (d < 3u) {
        q.hp += 1ull << (21 * d);
      } else {
        atomicAdd(&shist[code], 1u);
        if (code == 0) {
          const unsigned lin = (unsigned)(pc.lbase + (P1 * (int)g.d[2] + P2) * s);
          atomicOr(&A.obm[lin >> 5], 1u << (lin & 31));
          q.bad |= !isfinite((double)o);
        }
      }
      if (!LV1) A.E[pc.ebase + ((long long)P1 * (s >> 1)) * g.Ed[2] + (long long)P2 * (s >> 1)] = rv;
    }
  } else {
    const int lin = pc.lbase + (P1 * (int)g.d[2] + P2) * s;
    if (code_in != 0)
      rv = dequantize(pred, q.two_eb, code_in);
    else
      rv = m_outlier(A.oidx, A.oval, (unsigned long long)(unsigned)lin, q.ocount, &q.bad);
    if (emit) {
      if (LV1) {
        reinterpret_cast<T*>(A.out)[lin] = (T)rv;
        q.nf |= !isfinite(rv);
      } else {
        A.E[pc.ebase + ((long long)P1 * (s >> 1)) * g.Ed[2] + (long long)P2 * (s >> 1)] = rv;
      }
    }
  }
  return rv;
}

// the code byte of item (iy, iz) of class C in plane pc (decompress prefetch)
template <class G, int C>
__device__ __forceinline__ int code_of(const MarchArgs& A, const PlaneCtx& pc, int Y0, int Z0, int iy, int iz) {
  using cg = CG<G, C>;
  const int P1 = Y0 + cg::py(iy), P2 = Z0 + cg::pz(iz);
  if (!pc.live || !((unsigned)P1 < (unsigned)A.g.D[1] && (unsigned)P2 < (unsigned)A.g.D[2])) return 0;
  return __ldg(A.seq + pc.sbase + slot_item<C>(A.g, P1, P2));
}

// Halo items (not owned by any thread's core mapping) of the even-axis
// margins: index h of class C's margin list -> (iy, iz)
template <class G, int C>
__device__ __forceinline__ void halo_item(int h, int& iy, int& iz) {
  using cg = CG<G, C>;
  auto m3 = [](int i) { return i == 0 ? 0 : G::HZ + i; };  // margin items 0, H+1, H+2
  if (cg::yo && !cg::zo) {          // c2 / c3: every core row, 3 margin columns
    iy = h / 3, iz = m3(h % 3);
  } else if (!cg::yo && cg::zo) {   // c4 / c5: 3 margin rows, every core column
    iy = m3(h / G::HZ), iz = h % G::HZ;
  } else {                          // c1: 3 margin rows of EZ items, then the core rows' margin columns
    if (h < 3 * G::EZ) {
      iy = m3(h / G::EZ), iz = h % G::EZ;
    } else {
      h -= 3 * G::EZ;
      iy = 1 + h / 3, iz = m3(h % 3);
    }
  }
}

// E plane j (lattice P0 = 2j) into an [EY][EZP] ring slot
template <class G>
__device__ __forceinline__ void stage_E(const MarchArgs& A, int j, int Y0, int Z0, double* dst, uint64_t* bar) {
  const LevelGeom& g = A.g;
  if (j < 0 || j >= A.nep) return;
  if (A.etma) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(bar, G::NE * 8);
      tma_load_3d(dst, &A.emap, Z0 / 2 - 2, Y0 / 2 - 1, (int)(j * g.s), bar);
    }
    return;
  }
  for (int i = threadIdx.x; i < G::NE; i += MT) {
    const int ey = i / G::EZP, c = i - ey * G::EZP;
    const int P1 = Y0 + 2 * ey - 2, P2 = Z0 + 2 * c - 4;
    const bool ok = (unsigned)P1 < (unsigned)g.D[1] && (unsigned)P2 < (unsigned)g.D[2];
    cp_async<8>(dst + i, A.E + (long long)j * g.ke[0] + (long long)(P1 >> 1) * g.ke[1] + (long long)(P2 >> 1) * g.ke[2],
                ok);
  }
}

// field rectangle of lattice plane P0 into an [FR][FC] ring slot
template <typename T, class G>
__device__ __forceinline__ void stage_F(const MarchArgs& A, int P0, int Y0, int Z0, T* dst, uint64_t* bar) {
  const LevelGeom& g = A.g;
  if (A.ftma) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(bar, G::NF * sizeof(T));
      tma_load_3d(dst, &A.fmap, Z0 - 4, Y0 - 2, P0, bar);
    }
    return;
  }
  const int s = (int)g.s;
  for (int i = threadIdx.x; i < G::NF; i += MT) {
    const int r = i / G::FC, c = i - r * G::FC;
    const int P1 = Y0 - 2 + r, P2 = Z0 - 4 + c;
    const bool ok = (unsigned)P1 < (unsigned)g.D[1] && (unsigned)P2 < (unsigned)g.D[2];
    cp_async<sizeof(T)>(dst + i,
                        reinterpret_cast<const T*>(A.field) + (((long long)P0 * s * g.d[1] + (long long)P1 * s) * g.d[2] +
                                                               (long long)P2 * s),
                        ok);
  }
}

// One item of class C: coordinates, prediction, then (after every prediction
// of the half-phase has been issued, so the shared-memory loads of all items
// overlap) quantize / replay and the stores.
template <typename T, bool DEC, bool LINEAR, bool LV1, class G, int C, bool FAST>
struct Job {
  using cg = CG<G, C>;
  int iy, iz, P1, P2;
  bool ok;
  double pred;
  __device__ __forceinline__ void init(const LevelGeom& g, int Y0, int Z0, int iy_, int iz_, bool live) {
    iy = iy_, iz = iz_;
    P1 = Y0 + cg::py(iy), P2 = Z0 + cg::pz(iz);
    ok = live && (FAST || ((unsigned)P1 < (unsigned)g.D[1] && (unsigned)P2 < (unsigned)g.D[2]));
  }
  __device__ __forceinline__ void predict_(const LevelGeom& g, int xcls, const double* x0, const double* x1,
                                           const double* x2, const double* x3, const double* ys, const double* zs) {
    if (ok) pred = predict<G, C, LINEAR, FAST>(g, xcls, P1, P2, iy, iz, x0, x1, x2, x3, ys, zs);
  }
  __device__ __forceinline__ void finish_(const MarchArgs& A, const PlaneCtx& pc, int Y0, int Z0, bool core,
                                          double* dst, const T* fs, int code, QC& q, unsigned* shist) {
    if (!ok) return;
    const double rv = finish<T, DEC, LV1, G, C>(A, pc, Y0, Z0, P1, P2, core && pc.owned, pred, fs, code, q, shist);
    if (C != 7) dst[cg::e(iy, iz)] = rv;
  }
};

template <bool B>
struct BT {
  static constexpr bool v = B;
};

template <typename T, bool DEC, bool LINEAR, bool LV1, int TY, int TZ>
__global__ void __launch_bounds__(MT, DEC ? 3 : 3) k_march(const __grid_constant__ MarchArgs A) {
  using G = MG<TY, TZ, DEC ? 0 : sizeof(T)>;
  static_assert(G::HY * G::HZ == MT, "one core item per class per thread");
  extern __shared__ __align__(128) double sm[];
  __shared__ unsigned shist[256];
  __shared__ __align__(8) uint64_t bar;
  const LevelGeom& g = A.g;
  const int Y0 = (int)blockIdx.y * TY, Z0 = (int)blockIdx.x * TZ;
  const int js = (int)blockIdx.z * A.seg, je = min(js + A.seg, A.nep);
  const int tz = (int)threadIdx.x % G::HZ, row = (int)threadIdx.x / G::HZ;
  QC q;
  q.eb = A.st->eb;
  q.two_eb = A.st->two_eb;
  q.inv = __ddiv_rn(1.0, q.two_eb);
  q.ocount = DEC ? *A.ocount : 0;
  q.hp = 0;
  q.bad = q.nf = false;
  if (!DEC)
    for (int i = threadIdx.x; i < 256; i += MT) shist[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const bool yzint = Y0 >= 2 && Y0 + TY + 2 < g.D[1] && Z0 >= 2 && Z0 + TZ + 2 < g.D[2];
  // this thread's halo items: half 1 deals [c2 | c4 | c1] margins from
  // thread 0, half 2 [c3 | c5] from the thread after the last half-1 item
  constexpr int NH2 = 3 * G::HY, NH4 = 3 * G::HZ, NH1 = 3 * G::EZ + 3 * G::HY;
  constexpr int NHA = NH2 + NH4 + NH1, NHB = NH2 + NH4;
  static_assert(NHA <= MT && NHB <= MT, "one halo item per thread and half");
  int ha = (int)threadIdx.x, hb = (int)threadIdx.x - NHA;
  if (hb < 0) hb += MT;
  int hcA = 0, hyA = 0, hzA = 0, hcB = 0, hyB = 0, hzB = 0;
  if (ha < NH2) {
    hcA = 2, halo_item<G, 2>(ha, hyA, hzA);
  } else if (ha < NH2 + NH4) {
    hcA = 4, halo_item<G, 4>(ha - NH2, hyA, hzA);
  } else if (ha < NHA) {
    hcA = 1, halo_item<G, 1>(ha - NH2 - NH4, hyA, hzA);
  }
  if (hb < NH2) {
    hcB = 3, halo_item<G, 3>(hb, hyB, hzB);
  } else if (hb < NHB) {
    hcB = 5, halo_item<G, 5>(hb - NH2, hyB, hzB);
  }
  double* const sE = sm + G::oE;
  double* const sC2 = sm + G::oC2;
  double* const sC4 = sm + G::oC4;
  double* const sC6 = sm + G::oC6;
  double* const sC1 = sm + G::oC1;
  double* const sC3 = sm + G::oC3;
  double* const sC5 = sm + G::oC5;
  T* const sFe = reinterpret_cast<T*>(sm + G::dbl);  // even planes: slot j % RFE
  T* const sFo = sFe + G::RFE * G::SF;               // odd planes: slot m % RFO
  const int D1 = (int)g.D[1], D2 = (int)g.D[2], eyez = (int)g.eyez, pre = (int)g.prefix;
  const int plane = (int)(g.d[1] * g.d[2]) * (int)g.s;
  auto ctx = [&](int P0, bool owned, bool live) {
    PlaneCtx c;
    c.P0 = P0;
    c.owned = owned;
    c.live = live;
    c.xcls = (P0 & 1) ? classify(P0, g.D[0], 1, LINEAR) : 0;
    c.sbase = pre + P0 * D1 * D2 - ((P0 + 1) >> 1) * eyez;
    c.lbase = P0 * plane;
    c.ebase = LV1 ? 0 : ((long long)P0 * (g.s >> 1)) * g.Ed[1] * g.Ed[2];
    return c;
  };
  auto even_ctx = [&](int j) { return ctx(2 * j, j >= js && j < je, j >= 0 && j < A.nep && j >= js - 1 && j <= je + 1); };
  auto odd_ctx = [&](int m) { return ctx(2 * m + 1, true, m >= js && m < je && m < A.nop); };
  // decompress: the code bytes of the next phase, prefetched a phase ahead
  int c2 = 0, c4 = 0, c1 = 0, c7 = 0, c6 = 0, c3 = 0, c5 = 0, cA = 0, cB = 0;
  auto prefetch_codes = [&](int k) {
    if (!DEC) return;
    const PlaneCtx pe = even_ctx(k), p1 = odd_ctx(k - 2), p7 = odd_ctx(k - 3);
    c2 = code_of<G, 2>(A, pe, Y0, Z0, row, tz + 1);
    c4 = code_of<G, 4>(A, pe, Y0, Z0, row + 1, tz);
    c6 = code_of<G, 6>(A, pe, Y0, Z0, row, tz);
    c1 = code_of<G, 1>(A, p1, Y0, Z0, row + 1, tz + 1);
    c3 = code_of<G, 3>(A, p1, Y0, Z0, row, tz + 1);
    c5 = code_of<G, 5>(A, p1, Y0, Z0, row + 1, tz);
    c7 = code_of<G, 7>(A, p7, Y0, Z0, row, tz);
    cA = hcA == 2 ? code_of<G, 2>(A, pe, Y0, Z0, hyA, hzA)
                  : (hcA == 4 ? code_of<G, 4>(A, pe, Y0, Z0, hyA, hzA)
                              : (hcA == 1 ? code_of<G, 1>(A, p1, Y0, Z0, hyA, hzA) : 0));
    cB = hcB == 3 ? code_of<G, 3>(A, p1, Y0, Z0, hyB, hzB) : (hcB == 5 ? code_of<G, 5>(A, p1, Y0, Z0, hyB, hzB) : 0);
  };
  unsigned phase = 0;
  constexpr int ME = G::RE - 1, MC = G::RC - 1;
  auto stage = [&](int k) {  // the TMA / cp.async inputs of phase k
    if (k <= je + 1) stage_E<G>(A, k, Y0, Z0, sE + (k & ME) * G::SE, &bar);
    if (!DEC && even_ctx(k).live) stage_F<T, G>(A, 2 * k, Y0, Z0, sFe + (k & (G::RFE - 1)) * G::SF, &bar);
    if (!DEC && odd_ctx(k - 2).live)
      stage_F<T, G>(A, 2 * (k - 2) + 1, Y0, Z0, sFo + ((k - 2) & (G::RFO - 1)) * G::SF, &bar);
    if (threadIdx.x == 0) mbar_arrive(&bar);
    cp_commit();
  };
  stage(js - 1);
  prefetch_codes(js - 1);
  cp_async_wait_all();
  mbar_wait(&bar, phase);
  phase ^= 1;
  __syncthreads();
  for (int k = js - 1; k <= je + 2; k++) {
    const int m1 = k - 2, m7 = k - 3;  // odd planes of c1/c3/c5 and of c7
    const PlaneCtx pe = even_ctx(k), p1 = odd_ctx(m1), p7 = odd_ctx(m7);
    // half-phase variant: every item of the tile has complete cubic / linear
    // stencils along every axis (no per-item validity or classification)
    const bool fast = yzint && 2 * m7 + 1 >= 3 && 2 * m1 + 4 < g.D[0];
    const double* Ek = sE + (k & ME) * G::SE;
    const T* fe = sFe + (k & (G::RFE - 1)) * G::SF;
    const T* f1 = sFo + (m1 & (G::RFO - 1)) * G::SF;
    const T* f7 = sFo + (m7 & (G::RFO - 1)) * G::SF;
    double* c2k = sC2 + (k & MC) * G::S2;
    double* c4k = sC4 + (k & MC) * G::S4;
    double* c6k = sC6 + (k & MC) * G::S6;
    const int k2 = c2, k4 = c4, k1 = c1, k7 = c7, k6 = c6, k3 = c3, k5 = c5, kA = cA, kB = cB;
    if (DEC) prefetch_codes(k + 1);
    // ---- half 1: c2, c4 of plane k | c1 of odd m1 | c7 of odd m7 (| E points of plane k on decompress)
    auto half1 = [&](auto F) {
      constexpr bool FA = decltype(F)::v;
      Job<T, DEC, LINEAR, LV1, G, 2, FA> j2, h2;
      Job<T, DEC, LINEAR, LV1, G, 4, FA> j4, h4;
      Job<T, DEC, LINEAR, LV1, G, 1, FA> j1, h1;
      Job<T, DEC, LINEAR, LV1, G, 7, FA> j7;
      j2.init(g, Y0, Z0, row, tz + 1, pe.live);
      j4.init(g, Y0, Z0, row + 1, tz, pe.live);
      j1.init(g, Y0, Z0, row + 1, tz + 1, p1.live);
      j7.init(g, Y0, Z0, row, tz, p7.live);
      h2.init(g, Y0, Z0, hyA, hzA, pe.live && hcA == 2);
      h4.init(g, Y0, Z0, hyA, hzA, pe.live && hcA == 4);
      h1.init(g, Y0, Z0, hyA, hzA, p1.live && hcA == 1);
      const double* e0 = sE + ((m1 - 1) & ME) * G::SE;
      const double* e1 = sE + (m1 & ME) * G::SE;
      const double* e2 = sE + ((m1 + 1) & ME) * G::SE;
      const double* e3 = sE + ((m1 + 2) & ME) * G::SE;
      const double* s0 = sC6 + ((m7 - 1) & MC) * G::S6;
      const double* s1 = sC6 + (m7 & MC) * G::S6;
      const double* s2 = sC6 + ((m7 + 1) & MC) * G::S6;
      const double* s3 = sC6 + ((m7 + 2) & MC) * G::S6;
      j2.predict_(g, 0, 0, 0, 0, 0, Ek, 0);
      j4.predict_(g, 0, 0, 0, 0, 0, 0, Ek);
      j1.predict_(g, p1.xcls, e0, e1, e2, e3, 0, 0);
      j7.predict_(g, p7.xcls, s0, s1, s2, s3, sC5, sC3);
      h2.predict_(g, 0, 0, 0, 0, 0, Ek, 0);
      h4.predict_(g, 0, 0, 0, 0, 0, 0, Ek);
      h1.predict_(g, p1.xcls, e0, e1, e2, e3, 0, 0);
      j2.finish_(A, pe, Y0, Z0, true, c2k, fe, k2, q, shist);
      j4.finish_(A, pe, Y0, Z0, true, c4k, fe, k4, q, shist);
      j1.finish_(A, p1, Y0, Z0, true, sC1, f1, k1, q, shist);
      j7.finish_(A, p7, Y0, Z0, true, nullptr, f7, k7, q, shist);
      h2.finish_(A, pe, Y0, Z0, false, c2k, fe, kA, q, shist);
      h4.finish_(A, pe, Y0, Z0, false, c4k, fe, kA, q, shist);
      h1.finish_(A, p1, Y0, Z0, false, sC1, f1, kA, q, shist);
    };
    if (fast)
      half1(BT<true>{});
    else
      half1(BT<false>{});
    if (DEC && LV1 && pe.live && pe.owned) {  // the 2-lattice points of plane k are outputs too
      const int P1 = Y0 + 2 * row, P2 = Z0 + 2 * tz;
      if (P1 < D1 && P2 < D2) {
        const double v = Ek[(row + 1) * G::EZP + tz + 2];
        reinterpret_cast<T*>(A.out)[pe.lbase + P1 * (int)g.d[2] + P2] = (T)v;
        q.nf |= !isfinite(v);
      }
    }
    __syncthreads();
    // the inputs of phase k+1 land in the slots of planes k-3 (E, odd field)
    // and k-1 (even field), free from here on
    stage(k + 1);
    // ---- half 2: c6 of plane k | c3, c5 of odd m1
    auto half2 = [&](auto F) {
      constexpr bool FA = decltype(F)::v;
      Job<T, DEC, LINEAR, LV1, G, 6, FA> j6;
      Job<T, DEC, LINEAR, LV1, G, 3, FA> j3, h3;
      Job<T, DEC, LINEAR, LV1, G, 5, FA> j5, h5;
      j6.init(g, Y0, Z0, row, tz, pe.live);
      j3.init(g, Y0, Z0, row, tz + 1, p1.live);
      j5.init(g, Y0, Z0, row + 1, tz, p1.live);
      h3.init(g, Y0, Z0, hyB, hzB, p1.live && hcB == 3);
      h5.init(g, Y0, Z0, hyB, hzB, p1.live && hcB == 5);
      const double* b0 = sC2 + ((m1 - 1) & MC) * G::S2;
      const double* b1 = sC2 + (m1 & MC) * G::S2;
      const double* b2 = sC2 + ((m1 + 1) & MC) * G::S2;
      const double* b3 = sC2 + ((m1 + 2) & MC) * G::S2;
      const double* d0 = sC4 + ((m1 - 1) & MC) * G::S4;
      const double* d1 = sC4 + (m1 & MC) * G::S4;
      const double* d2 = sC4 + ((m1 + 1) & MC) * G::S4;
      const double* d3 = sC4 + ((m1 + 2) & MC) * G::S4;
      j6.predict_(g, 0, 0, 0, 0, 0, c4k, c2k);
      j3.predict_(g, p1.xcls, b0, b1, b2, b3, sC1, 0);
      j5.predict_(g, p1.xcls, d0, d1, d2, d3, 0, sC1);
      h3.predict_(g, p1.xcls, b0, b1, b2, b3, sC1, 0);
      h5.predict_(g, p1.xcls, d0, d1, d2, d3, 0, sC1);
      j6.finish_(A, pe, Y0, Z0, true, c6k, fe, k6, q, shist);
      j3.finish_(A, p1, Y0, Z0, true, sC3, f1, k3, q, shist);
      j5.finish_(A, p1, Y0, Z0, true, sC5, f1, k5, q, shist);
      h3.finish_(A, p1, Y0, Z0, false, sC3, f1, kB, q, shist);
      h5.finish_(A, p1, Y0, Z0, false, sC5, f1, kB, q, shist);
    };
    if (fast)
      half2(BT<true>{});
    else
      half2(BT<false>{});
    cp_async_wait_all();
    mbar_wait(&bar, phase);
    phase ^= 1;
    __syncthreads();
  }
  if (DEC && __any_sync(0xffffffffu, q.nf) && (threadIdx.x & 31) == 0) raise_flag(A.st, F_NONFINITE);
  if (__any_sync(0xffffffffu, q.bad) && (threadIdx.x & 31) == 0) raise_flag(A.st, DEC ? F_ORPHAN : F_NONFINITE);
  if (!DEC) {
    const unsigned m = (1u << 21) - 1;
    const unsigned h7 = __reduce_add_sync(0xffffffffu, (unsigned)q.hp & m),
                   h8 = __reduce_add_sync(0xffffffffu, (unsigned)(q.hp >> 21) & m),
                   h9 = __reduce_add_sync(0xffffffffu, (unsigned)(q.hp >> 42) & m);
    if ((threadIdx.x & 31) == 0) {
      if (h7) atomicAdd(&shist[127], h7);
      if (h8) atomicAdd(&shist[128], h8);
      if (h9) atomicAdd(&shist[129], h9);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += MT)
      if (shist[i]) atomicAdd(&A.st->hist[i], (unsigned long long)shist[i]);
  }
}

constexpr int MTY = 32, MTZ = 32;

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3D tiled map over a C-order (n0, n1, n2) array with one-plane boxes
bool encode3(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int esz, long long n0, long long n1,
             long long n2, int b2, int b1) {
  auto fn = encode_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(base) & 15) || (n2 * esz) % 16 || n0 > INT_MAX) return false;
  const cuuint64_t dim[3] = {(cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)n0};
  const cuuint64_t str[2] = {(cuuint64_t)(n2 * esz), (cuuint64_t)(n1 * n2 * esz)};
  const cuuint32_t box[3] = {(cuuint32_t)b2, (cuuint32_t)b1, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(m, dt, 3, const_cast<void*>(base), dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <typename T, bool DEC, bool LINEAR, bool LV1>
void launch_march(const MarchArgs& A, cudaStream_t s) {
  using G = MG<MTY, MTZ, DEC ? 0 : sizeof(T)>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute((const void*)k_march<T, DEC, LINEAR, LV1, MTY, MTZ>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::bytes);
    attr = true;
  }
  const LevelGeom& g = A.g;
  const dim3 grid((unsigned)((g.D[2] + MTZ - 1) / MTZ), (unsigned)((g.D[1] + MTY - 1) / MTY),
                  (unsigned)((A.nep + A.seg - 1) / A.seg));
  k_march<T, DEC, LINEAR, LV1, MTY, MTZ><<<grid, MT, G::bytes, s>>>(A);
}

// multidim 3D levels whose lattice fits 32-bit indexing
bool march_ok(const LevelGeom& g, int cfg) {
  if (cfg < 0 || (cfg & 2) || !getenv("HB_MARCH")) return false;  // opt-in while it trails k_pass.cu
  for (int a = 0; a < 3; a++)
    if (g.D[a] < 4) return false;
  return g.d[0] * g.d[1] * g.d[2] < INT_MAX - 64;
}

int seg_len(const LevelGeom& g) {
  // enough CTAs for ~3 waves of 148 SMs x 2 resident CTAs, segments of >= 8 even planes
  const long long tiles = ((g.D[2] + MTZ - 1) / MTZ) * ((g.D[1] + MTY - 1) / MTY);
  const long long nep = (g.D[0] + 1) / 2;
  long long seg = nep;
  while (seg > 8 && tiles * ((nep + seg - 1) / seg) < 3 * 2 * kSMs) seg = (seg + 1) / 2;
  if (const char* e = getenv("HB_MARCH_SEG")) seg = std::max(1, atoi(e));
  return (int)std::max(1ll, seg);
}

void prepare(MarchArgs& A, int prec) {
  const LevelGeom& g = A.g;
  A.nep = (int)((g.D[0] + 1) / 2);
  A.nop = (int)(g.D[0] / 2);
  A.seg = seg_len(g);
  using G = MG<MTY, MTZ, 4>;
  const bool notma = getenv("HB_MARCH_NO_TMA") != nullptr;
  // TMA boxes need unit element strides: level 1 only (levels >= 2 sample the
  // field and E at stride s and take the cp.async path)
  A.etma = !notma && g.s == 1 &&
           encode3(&A.emap, A.E, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, g.Ed[0], g.Ed[1], g.Ed[2], G::EZP, G::EY);
  A.ftma = !notma && g.s == 1 && A.field &&
           encode3(&A.fmap, A.field, prec == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                   prec, g.d[0], g.d[1], g.d[2], G::FC, G::FR);
}

template <typename T, bool DEC>
void dispatch(const MarchArgs& A, bool linear, cudaStream_t s) {
  if (A.g.level == 1)
    linear ? launch_march<T, DEC, true, true>(A, s) : launch_march<T, DEC, false, true>(A, s);
  else
    linear ? launch_march<T, DEC, true, false>(A, s) : launch_march<T, DEC, false, false>(A, s);
}

}  // namespace

int launch_level_march_compress(const LevelGeom& g, const void* field, int prec, double* E, uint8_t* seq,
                                uint32_t* obm, DevState* st, cudaStream_t s, int cfg) {
  if (!march_ok(g, cfg)) return 0;
  MarchArgs A{};
  A.g = g;
  A.field = field;
  A.E = E;
  A.seq = seq;
  A.obm = obm;
  A.st = st;
  prepare(A, prec);
  if (prec == 4)
    dispatch<float, false>(A, cfg & 1, s);
  else
    dispatch<double, false>(A, cfg & 1, s);
  return 1;
}

int launch_level_march_decompress(const LevelGeom& g, const uint8_t* seq, const uint64_t* oidx, const double* oval,
                                  const unsigned long long* ocount_dev, double* E, void* out, int prec, DevState* st,
                                  cudaStream_t s, int cfg) {
  if (!march_ok(g, cfg)) return 0;
  MarchArgs A{};
  A.g = g;
  A.E = E;
  A.seq = const_cast<uint8_t*>(seq);
  A.oidx = oidx;
  A.oval = oval;
  A.ocount = ocount_dev;
  A.out = out;
  A.st = st;
  prepare(A, prec);
  if (prec == 4)
    dispatch<float, true>(A, cfg & 1, s);
  else
    dispatch<double, true>(A, cfg & 1, s);
  return 1;
}

}  // namespace hb
