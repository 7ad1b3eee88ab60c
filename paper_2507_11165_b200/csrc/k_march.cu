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

// --------------------------------------------------------------- item bodies
template <bool B>
struct BT {
  static constexpr bool v = B;
};

// A thread's item of some class: where it lives in the class array (e), where
// its y / z stencil sources start (ey: same layout, rows iy..iy+3; ez: the
// even-z array, items iz..iz+3), its field value in the staged rectangle (f),
// the in-plane parts of its Eq. 3 slot / element index / E index, and its
// lattice coordinates (edge tiles classify and bound-check from them).
struct ItemAt {
  int e, ez, f, slot, lin, P1, P2;
  long long eidx;
};

template <class G, int C>
__device__ __forceinline__ ItemAt item_at(const LevelGeom& g, int Y0, int Z0, int iy, int iz) {
  using cg = CG<G, C>;
  ItemAt it;
  it.P1 = Y0 + cg::py(iy), it.P2 = Z0 + cg::pz(iz);
  it.e = cg::e(iy, iz);
  it.ez = iy * G::EZP + iz + 1;
  it.f = (it.P1 - Y0 + 2) * G::FC + (it.P2 - Z0 + 4);
  it.slot = slot_item<C>(g, it.P1, it.P2);
  const int s = (int)g.s;
  it.lin = (it.P1 * (int)g.d[2] + it.P2) * s;
  it.eidx = ((long long)it.P1 * (s >> 1)) * g.Ed[2] + (long long)it.P2 * (s >> 1);
  return it;
}

// stencil along an in-plane axis (taps p[0], p[st], p[2st], p[3st]) or along
// axis 0 (tap i from plane i at e)
template <bool LINEAR, bool INT>
__device__ __forceinline__ double st_in(const double* p, int st, int cls) {
  const int c = INT ? (LINEAR ? ST_MID : ST_CUBIC) : cls;
  return apply_stencil(c, (INT && LINEAR) ? 0.0 : p[0], p[st], p[2 * st], (INT && LINEAR) ? 0.0 : p[3 * st]);
}
template <bool LINEAR, bool INT>
__device__ __forceinline__ double st_x(const double* a, const double* b, const double* c, const double* d, int e,
                                       int cls) {
  const int k = INT ? (LINEAR ? ST_MID : ST_CUBIC) : cls;
  return apply_stencil(k, (INT && LINEAR) ? 0.0 : a[e], b[e], c[e], (INT && LINEAR) ? 0.0 : d[e]);
}
// multi-axis average (predictor.py:247-256); interior: every order is equal
template <bool INT>
__device__ __forceinline__ double comb2(double a, int oa, double b, int ob) {
  if (INT) return __dmul_rn(__dadd_rn(__dadd_rn(0.0, a), b), 0.5);
  const double p[2] = {a, b};
  const int o[2] = {oa, ob};
  return combine_axes(2, p, o);
}
template <bool INT>
__device__ __forceinline__ double comb3(double a, int oa, double b, int ob, double c, int oc) {
  if (INT) return __ddiv_rn(__dadd_rn(__dadd_rn(__dadd_rn(0.0, a), b), c), 3.0);
  const double p[3] = {a, b, c};
  const int o[3] = {oa, ob, oc};
  return combine_axes(3, p, o);
}

// quantize (predictor.py:313-329) / replay (:397-411) of one item and its
// emission when the CTA owns it
template <typename T, bool DEC, bool LV1>
__device__ __forceinline__ double fin(const MarchArgs& A, double pred, const T* fs, int f, int code_in, int slot,
                                      int lin, long long eidx, bool emit, QC& q, unsigned* shist) {
  double rv;
  if (!DEC) {
    const T o = fs[f];
    const int code = quantize_fast<sizeof(T) == 4>((double)o, pred, q.eb, q.two_eb, q.inv, &rv);
    if (emit) {
      A.seq[slot] = (uint8_t)code;
      const unsigned d = (unsigned)code - 127u;
      if (d < 3u) {
        q.hp += 1ull << (21 * d);
      } else {
        atomicAdd(&shist[code], 1u);
        if (code == 0) {
          atomicOr(&A.obm[(unsigned)lin >> 5], 1u << (lin & 31));
          q.bad |= !isfinite((double)o);
        }
      }
      if (!LV1) A.E[eidx] = rv;
    }
  } else {
    if (code_in != 0)
      rv = dequantize(pred, q.two_eb, code_in);
    else
      rv = m_outlier(A.oidx, A.oval, (unsigned long long)(unsigned)lin, q.ocount, &q.bad);
    if (emit) {
      if (LV1) {
        reinterpret_cast<T*>(A.out)[lin] = (T)rv;
        q.nf |= !isfinite(rv);
      } else {
        A.E[eidx] = rv;
      }
    }
  }
  return rv;
}

template <typename T, bool DEC, bool LINEAR, bool LV1, int TY, int TZ>
__global__ void __launch_bounds__(MT, 2) k_march(const __grid_constant__ MarchArgs A) {
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
  // this thread's core items (one per class) and halo items (at most one per
  // half-phase: half 1 deals the [c2 | c4 | c1] margins from thread 0, half 2
  // the [c3 | c5] margins from the thread after the last half-1 item)
  const ItemAt i1 = item_at<G, 1>(g, Y0, Z0, row + 1, tz + 1), i2 = item_at<G, 2>(g, Y0, Z0, row, tz + 1),
               i3 = item_at<G, 3>(g, Y0, Z0, row, tz + 1), i4 = item_at<G, 4>(g, Y0, Z0, row + 1, tz),
               i5 = item_at<G, 5>(g, Y0, Z0, row + 1, tz), i6 = item_at<G, 6>(g, Y0, Z0, row, tz),
               i7 = item_at<G, 7>(g, Y0, Z0, row, tz);
  constexpr int NH2 = 3 * G::HY, NH4 = 3 * G::HZ, NH1 = 3 * G::EZ + 3 * G::HY;
  constexpr int NHA = NH2 + NH4 + NH1, NHB = NH2 + NH4;
  static_assert(NHA <= MT && NHB <= MT, "one halo item per thread and half");
  int hcA = 0, hcB = 0;
  ItemAt hA{}, hB{};
  {
    int ha = (int)threadIdx.x, hb = (int)threadIdx.x - NHA, iy = 0, iz = 0;
    if (hb < 0) hb += MT;
    if (ha < NH2) {
      halo_item<G, 2>(ha, iy, iz), hcA = 2, hA = item_at<G, 2>(g, Y0, Z0, iy, iz);
    } else if (ha < NH2 + NH4) {
      halo_item<G, 4>(ha - NH2, iy, iz), hcA = 4, hA = item_at<G, 4>(g, Y0, Z0, iy, iz);
    } else if (ha < NHA) {
      halo_item<G, 1>(ha - NH2 - NH4, iy, iz), hcA = 1, hA = item_at<G, 1>(g, Y0, Z0, iy, iz);
    }
    if (hb < NH2) {
      halo_item<G, 3>(hb, iy, iz), hcB = 3, hB = item_at<G, 3>(g, Y0, Z0, iy, iz);
    } else if (hb < NHB) {
      halo_item<G, 5>(hb - NH2, iy, iz), hcB = 5, hB = item_at<G, 5>(g, Y0, Z0, iy, iz);
    }
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
  const long long eplane = LV1 ? 0 : (g.s >> 1) * g.Ed[1] * g.Ed[2];
  auto sbase = [&](int P0) { return pre + P0 * D1 * D2 - ((P0 + 1) >> 1) * eyez; };
  auto elive = [&](int j) { return j >= 0 && j < A.nep && j >= js - 1 && j <= je + 1; };
  auto olive = [&](int m) { return m >= js && m < je && m < A.nop; };
  auto code_at = [&](bool live, int P0, const ItemAt& it, bool edge) -> int {
    if (!live || (edge && !((unsigned)it.P1 < (unsigned)D1 && (unsigned)it.P2 < (unsigned)D2))) return 0;
    return __ldg(A.seq + sbase(P0) + it.slot);
  };
  // decompress: the code bytes of the next phase, prefetched a phase ahead
  int c2 = 0, c4 = 0, c1 = 0, c7 = 0, c6 = 0, c3 = 0, c5 = 0, cA = 0, cB = 0;
  auto prefetch_codes = [&](int k) {
    if (!DEC) return;
    const bool le = elive(k), l1 = olive(k - 2), l7 = olive(k - 3), ed = !yzint;
    const int Pe = 2 * k, P1 = 2 * (k - 2) + 1, P7 = 2 * (k - 3) + 1;
    c2 = code_at(le, Pe, i2, ed), c4 = code_at(le, Pe, i4, ed), c6 = code_at(le, Pe, i6, ed);
    c1 = code_at(l1, P1, i1, ed), c3 = code_at(l1, P1, i3, ed), c5 = code_at(l1, P1, i5, ed);
    c7 = code_at(l7, P7, i7, ed);
    cA = code_at(hcA == 1 ? l1 : (hcA != 0 && le), hcA == 1 ? P1 : Pe, hA, true);
    cB = code_at(hcB != 0 && l1, P1, hB, true);
  };
  unsigned phase = 0;
  constexpr int ME = G::RE - 1, MC = G::RC - 1;
  auto stage = [&](int k) {  // the TMA / cp.async inputs of phase k
    if (k <= je + 1) stage_E<G>(A, k, Y0, Z0, sE + (k & ME) * G::SE, &bar);
    if (!DEC && elive(k)) stage_F<T, G>(A, 2 * k, Y0, Z0, sFe + (k & (G::RFE - 1)) * G::SF, &bar);
    if (!DEC && olive(k - 2))
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
    const bool le = elive(k), l1 = olive(m1), l7 = olive(m7);
    const bool oe = k >= js && k < je;  // even plane k is owned
    const int Pe = 2 * k, P1 = 2 * m1 + 1, P7 = 2 * m7 + 1;
    const int sbE = sbase(Pe), sb1 = sbase(P1), sb7 = sbase(P7);
    const int lbE = Pe * plane, lb1 = P1 * plane, lb7 = P7 * plane;
    const long long ebE = Pe * eplane, eb1 = P1 * eplane, eb7 = P7 * eplane;
    const int x1c = classify(P1, g.D[0], 1, LINEAR), x7c = classify(P7, g.D[0], 1, LINEAR);
    // interior phase: every item of the tile has complete cubic / linear
    // stencils along every axis (no per-item bounds or classification)
    const bool fast = LV1 && yzint && P7 >= 3 && P1 + 3 < g.D[0];
    const double* Ek = sE + (k & ME) * G::SE;
    const T* fe = sFe + (k & (G::RFE - 1)) * G::SF;
    const T* f1 = sFo + (m1 & (G::RFO - 1)) * G::SF;
    const T* f7 = sFo + (m7 & (G::RFO - 1)) * G::SF;
    double* c2k = sC2 + (k & MC) * G::S2;
    double* c4k = sC4 + (k & MC) * G::S4;
    double* c6k = sC6 + (k & MC) * G::S6;
    const int k2 = c2, k4 = c4, k1 = c1, k7 = c7, k6 = c6, k3 = c3, k5 = c5, kA = cA, kB = cB;
    if (DEC) prefetch_codes(k + 1);
    auto phase_body = [&](auto F) {
      constexpr bool I = decltype(F)::v;  // interior
      auto ok = [&](const ItemAt& it) {
        return I || ((unsigned)it.P1 < (unsigned)D1 && (unsigned)it.P2 < (unsigned)D2);
      };
      auto cy = [&](const ItemAt& it) { return I ? 0 : classify(it.P1, g.D[1], 1, LINEAR); };
      auto cz = [&](const ItemAt& it) { return I ? 0 : classify(it.P2, g.D[2], 1, LINEAR); };
      auto od = [&](int c) { return I ? (LINEAR ? 2 : 4) : stencil_order(c); };
      // ---- half 1: c2, c4 of plane k | c1 of odd m1 | c7 of odd m7
      {
        const double* e0 = sE + ((m1 - 1) & ME) * G::SE;
        const double* e1 = sE + (m1 & ME) * G::SE;
        const double* e2 = sE + ((m1 + 1) & ME) * G::SE;
        const double* e3 = sE + ((m1 + 2) & ME) * G::SE;
        const double* s0 = sC6 + ((m7 - 1) & MC) * G::S6;
        const double* s1 = sC6 + (m7 & MC) * G::S6;
        const double* s2 = sC6 + ((m7 + 1) & MC) * G::S6;
        const double* s3 = sC6 + ((m7 + 2) & MC) * G::S6;
        const bool v2 = le && ok(i2), v4 = le && ok(i4), v1 = l1 && ok(i1), v7 = l7 && ok(i7);
        double p2 = 0, p4 = 0, p1 = 0, p7 = 0;
        if (v2) p2 = st_in<LINEAR, I>(Ek + i2.e, G::EZP, cy(i2));
        if (v4) p4 = st_in<LINEAR, I>(Ek + i4.ez, 1, cz(i4));
        if (v1) p1 = st_x<LINEAR, I>(e0, e1, e2, e3, i1.e, x1c);
        if (v7) {
          const int a = x7c, b = cy(i7), c = cz(i7);
          p7 = comb3<I>(st_x<LINEAR, I>(s0, s1, s2, s3, i7.e, a), od(a), st_in<LINEAR, I>(sC5 + i7.e, G::HZ, b), od(b),
                        st_in<LINEAR, I>(sC3 + i7.ez, 1, c), od(c));
        }
        if (v2) c2k[i2.e] = fin<T, DEC, LV1>(A, p2, fe, i2.f, k2, sbE + i2.slot, lbE + i2.lin, ebE + i2.eidx, oe, q, shist);
        if (v4) c4k[i4.e] = fin<T, DEC, LV1>(A, p4, fe, i4.f, k4, sbE + i4.slot, lbE + i4.lin, ebE + i4.eidx, oe, q, shist);
        if (v1) sC1[i1.e] = fin<T, DEC, LV1>(A, p1, f1, i1.f, k1, sb1 + i1.slot, lb1 + i1.lin, eb1 + i1.eidx, true, q, shist);
        if (v7) fin<T, DEC, LV1>(A, p7, f7, i7.f, k7, sb7 + i7.slot, lb7 + i7.lin, eb7 + i7.eidx, true, q, shist);
        // halo item of half 1
        if (hcA == 2 && le && ok(hA)) {
          c2k[hA.e] = fin<T, DEC, LV1>(A, st_in<LINEAR, I>(Ek + hA.e, G::EZP, cy(hA)), fe, hA.f, kA, 0, lbE + hA.lin, 0, false, q, shist);
        } else if (hcA == 4 && le && ok(hA)) {
          c4k[hA.e] = fin<T, DEC, LV1>(A, st_in<LINEAR, I>(Ek + hA.ez, 1, cz(hA)), fe, hA.f, kA, 0, lbE + hA.lin, 0, false, q, shist);
        } else if (hcA == 1 && l1 && ok(hA)) {
          sC1[hA.e] = fin<T, DEC, LV1>(A, st_x<LINEAR, I>(e0, e1, e2, e3, hA.e, x1c), f1, hA.f, kA, 0, lb1 + hA.lin, 0,
                                       false, q, shist);
        }
        if (DEC && LV1 && le && oe) {  // the 2-lattice points of plane k are outputs too
          if (ok(i1)) {
            const double v = Ek[i1.e];
            reinterpret_cast<T*>(A.out)[lbE + i1.lin] = (T)v;
            q.nf |= !isfinite(v);
          }
        }
      }
      __syncthreads();
      // the inputs of phase k+1 land in the slots of planes k-3 (E, odd
      // field) and k-1 (even field), free from here on
      stage(k + 1);
      // ---- half 2: c6 of plane k | c3, c5 of odd m1
      {
        const double* b0 = sC2 + ((m1 - 1) & MC) * G::S2;
        const double* b1 = sC2 + (m1 & MC) * G::S2;
        const double* b2 = sC2 + ((m1 + 1) & MC) * G::S2;
        const double* b3 = sC2 + ((m1 + 2) & MC) * G::S2;
        const double* d0 = sC4 + ((m1 - 1) & MC) * G::S4;
        const double* d1 = sC4 + (m1 & MC) * G::S4;
        const double* d2 = sC4 + ((m1 + 1) & MC) * G::S4;
        const double* d3 = sC4 + ((m1 + 2) & MC) * G::S4;
        const bool v6 = le && ok(i6), v3 = l1 && ok(i3), v5 = l1 && ok(i5);
        double p6 = 0, p3 = 0, p5 = 0;
        if (v6) {
          const int b = cy(i6), c = cz(i6);
          p6 = comb2<I>(st_in<LINEAR, I>(c4k + i6.e, G::HZ, b), od(b), st_in<LINEAR, I>(c2k + i6.ez, 1, c), od(c));
        }
        if (v3) {
          const int b = cy(i3);
          p3 = comb2<I>(st_x<LINEAR, I>(b0, b1, b2, b3, i3.e, x1c), od(x1c), st_in<LINEAR, I>(sC1 + i3.e, G::EZP, b),
                        od(b));
        }
        if (v5) {
          const int c = cz(i5);
          p5 = comb2<I>(st_x<LINEAR, I>(d0, d1, d2, d3, i5.e, x1c), od(x1c), st_in<LINEAR, I>(sC1 + i5.ez, 1, c), od(c));
        }
        if (v6) c6k[i6.e] = fin<T, DEC, LV1>(A, p6, fe, i6.f, k6, sbE + i6.slot, lbE + i6.lin, ebE + i6.eidx, oe, q, shist);
        if (v3) sC3[i3.e] = fin<T, DEC, LV1>(A, p3, f1, i3.f, k3, sb1 + i3.slot, lb1 + i3.lin, eb1 + i3.eidx, true, q, shist);
        if (v5) sC5[i5.e] = fin<T, DEC, LV1>(A, p5, f1, i5.f, k5, sb1 + i5.slot, lb1 + i5.lin, eb1 + i5.eidx, true, q, shist);
        if (hcB == 3 && l1 && ok(hB)) {
          const int b = cy(hB);
          sC3[hB.e] = fin<T, DEC, LV1>(A,
                                       comb2<I>(st_x<LINEAR, I>(b0, b1, b2, b3, hB.e, x1c), od(x1c),
                                                st_in<LINEAR, I>(sC1 + hB.e, G::EZP, b), od(b)),
                                       f1, hB.f, kB, 0, lb1 + hB.lin, 0, false, q, shist);
        } else if (hcB == 5 && l1 && ok(hB)) {
          const int c = cz(hB);
          sC5[hB.e] = fin<T, DEC, LV1>(A,
                                       comb2<I>(st_x<LINEAR, I>(d0, d1, d2, d3, hB.e, x1c), od(x1c),
                                                st_in<LINEAR, I>(sC1 + hB.ez, 1, c), od(c)),
                                       f1, hB.f, kB, 0, lb1 + hB.lin, 0, false, q, shist);
        }
      }
    };
    // Interior phase (every stencil of the tile complete): the items of each
    // half go through prediction, quantization / replay and stores as one
    // batch, written breadth-first (each step for every item before the next
    // step) so the FP64 dependency chains of different items interleave; the
    // rare paths (exact-division quantizer fallback, histogram bins other
    // than 127..129, outliers) are deferred behind one branch.  Planes that
    // are not live are computed on stale shared memory and their stores
    // predicated off.
    auto fast_body = [&]() {
      constexpr double W0 = LINEAR ? 0.0 : -0.0625, W1 = LINEAR ? 0.5 : 0.5625;
      // NG stencil groups of 4 taps -> NG one-axis predictions, breadth-first
      auto stencils = [&](auto& tp, auto& res, int ng) {
#pragma unroll
        for (int g_ = 0; g_ < 7; g_++) {
          if (g_ >= ng) break;
          if (LINEAR) {
            res[g_] = __dadd_rn(__dmul_rn(tp[g_][1], 0.5), __dmul_rn(tp[g_][2], 0.5));
          }
        }
        if (!LINEAR) {
          double m0[7], m1[7], m2[7], m3[7];
#pragma unroll
          for (int g_ = 0; g_ < 7; g_++)
            if (g_ < ng) m0[g_] = __dmul_rn(tp[g_][0], W0), m1[g_] = __dmul_rn(tp[g_][1], W1);
#pragma unroll
          for (int g_ = 0; g_ < 7; g_++)
            if (g_ < ng) m2[g_] = __dmul_rn(tp[g_][2], W1), m3[g_] = __dmul_rn(tp[g_][3], W0);
#pragma unroll
          for (int g_ = 0; g_ < 7; g_++)
            if (g_ < ng) res[g_] = __dadd_rn(m0[g_], m1[g_]);
#pragma unroll
          for (int g_ = 0; g_ < 7; g_++)
            if (g_ < ng) res[g_] = __dadd_rn(res[g_], m2[g_]);
#pragma unroll
          for (int g_ = 0; g_ < 7; g_++)
            if (g_ < ng) res[g_] = __dadd_rn(res[g_], m3[g_]);
        }
      };
      constexpr int NB = 5;
      double p[NB], o[NB], rv[NB];
      int cd[NB];
      bool lv[NB], em[NB];
      auto batch = [&](int n, const int* f_lin, const int* slot) {
        if (!DEC) {
          double err[NB], u[NB], f[NB], fr[NB];
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) err[j] = __dsub_rn(o[j], p[j]);
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) u[j] = __dmul_rn(fabs(err[j]), q.inv);
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) u[j] = __dadd_rn(u[j], 0.5);
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) f[j] = floor(u[j]);
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) fr[j] = __dsub_rn(u[j], f[j]);
          unsigned ex = 0;
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) ex |= (!(fr[j] > 0x1p-40 && fr[j] < 1.0 - 0x1p-40) && !(u[j] >= 200.5)) ? (1u << j) : 0u;
          if (ex) {
#pragma unroll
            for (int j = 0; j < NB; j++)
              if (j < n && ((ex >> j) & 1)) f[j] = floor(__dadd_rn(__ddiv_rn(fabs(err[j]), q.two_eb), 0.5));
          }
          double qv[NB], r[NB], st[NB];
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) qv[j] = copysign(f[j], err[j]);
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) r[j] = __dmul_rn(q.two_eb, qv[j]);
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) r[j] = __dadd_rn(p[j], r[j]);
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) st[j] = sizeof(T) == 4 ? (double)__double2float_rn(r[j]) : r[j];
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) st[j] = __dsub_rn(o[j], st[j]);
#pragma unroll
          for (int j = 0; j < NB; j++) {
            if (j < n) {
              const bool ok = fabs(qv[j]) <= 127.0 && fabs(st[j]) <= q.eb;
              rv[j] = ok ? r[j] : o[j];
              cd[j] = ok ? (int)__dadd_rn(qv[j], 128.0) : 0;
            }
          }
          unsigned rare = 0;
#pragma unroll
          for (int j = 0; j < NB; j++) {
            if (j >= n) break;
            if (em[j]) A.seq[slot[j]] = (uint8_t)cd[j];
            const unsigned d = (unsigned)cd[j] - 127u;
            q.hp += (em[j] && d < 3u) ? (1ull << (21 * d)) : 0ull;
            rare |= (em[j] && d >= 3u) ? (1u << j) : 0u;
          }
          if (rare) {
#pragma unroll
            for (int j = 0; j < NB; j++)
              if (j < n && ((rare >> j) & 1)) {
                atomicAdd(&shist[cd[j]], 1u);
                if (cd[j] == 0) {
                  atomicOr(&A.obm[(unsigned)f_lin[j] >> 5], 1u << (f_lin[j] & 31));
                  q.bad |= !isfinite(o[j]);
                }
              }
          }
        } else {
          double r[NB];
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) r[j] = __dsub_rn((double)cd[j], 128.0);
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) r[j] = __dmul_rn(q.two_eb, r[j]);
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) rv[j] = __dadd_rn(p[j], r[j]);
          unsigned z = 0;
#pragma unroll
          for (int j = 0; j < NB; j++)
            if (j < n) z |= (lv[j] && cd[j] == 0) ? (1u << j) : 0u;
          if (z) {
#pragma unroll
            for (int j = 0; j < NB; j++)
              if (j < n && ((z >> j) & 1))
                rv[j] = m_outlier(A.oidx, A.oval, (unsigned long long)(unsigned)f_lin[j], q.ocount, &q.bad);
          }
#pragma unroll
          for (int j = 0; j < NB; j++) {
            if (j >= n) break;
            if (em[j]) {
              reinterpret_cast<T*>(A.out)[f_lin[j]] = (T)rv[j];
              q.nf |= !isfinite(rv[j]);
            }
          }
        }
      };
      // ---- half 1: c2, c4 of plane k | c1 of odd m1 | c7 of odd m7 | halo of c2 / c4 / c1
      {
        const double* e0 = sE + ((m1 - 1) & ME) * G::SE;
        const double* e1 = sE + (m1 & ME) * G::SE;
        const double* e2 = sE + ((m1 + 1) & ME) * G::SE;
        const double* e3 = sE + ((m1 + 2) & ME) * G::SE;
        const double* s0 = sC6 + ((m7 - 1) & MC) * G::S6;
        const double* s1 = sC6 + (m7 & MC) * G::S6;
        const double* s2 = sC6 + ((m7 + 1) & MC) * G::S6;
        const double* s3 = sC6 + ((m7 + 2) & MC) * G::S6;
        // halo taps: along x (c1) from the E planes at ea, else in plane k at ea + t * sa
        const bool hx = hcA == 1;
        const int sa = hcA == 4 ? 1 : G::EZP, ea = hcA == 4 ? hA.ez : hA.e;
        double tp[7][4], res[7];
#pragma unroll
        for (int t = 0; t < 4; t++) {
          tp[0][t] = Ek[i2.e + t * G::EZP];
          tp[1][t] = Ek[i4.ez + t];
          tp[3][t] = sC5[i7.e + t * G::HZ];
          tp[4][t] = sC3[i7.ez + t];
        }
        tp[2][0] = e0[i1.e], tp[2][1] = e1[i1.e], tp[2][2] = e2[i1.e], tp[2][3] = e3[i1.e];
        tp[5][0] = s0[i7.e], tp[5][1] = s1[i7.e], tp[5][2] = s2[i7.e], tp[5][3] = s3[i7.e];
        tp[6][0] = hx ? e0[ea] : Ek[ea];
        tp[6][1] = hx ? e1[ea] : Ek[ea + sa];
        tp[6][2] = hx ? e2[ea] : Ek[ea + 2 * sa];
        tp[6][3] = hx ? e3[ea] : Ek[ea + 3 * sa];
        const T* fa = hx ? f1 : fe;
        if (!DEC) {
          o[0] = (double)fe[i2.f], o[1] = (double)fe[i4.f], o[2] = (double)f1[i1.f], o[3] = (double)f7[i7.f];
          o[4] = (double)fa[hA.f];
        } else {
          cd[0] = k2, cd[1] = k4, cd[2] = k1, cd[3] = k7, cd[4] = kA;
        }
        stencils(tp, res, 7);
        p[0] = res[0], p[1] = res[1], p[2] = res[2], p[4] = res[6];
        p[3] = __ddiv_rn(__dadd_rn(__dadd_rn(__dadd_rn(0.0, res[5]), res[3]), res[4]), 3.0);  // axes x, y, z
        lv[0] = le, lv[1] = le, lv[2] = l1, lv[3] = l7, lv[4] = hcA != 0 && (hx ? l1 : le);
        em[0] = le && oe, em[1] = le && oe, em[2] = l1, em[3] = l7, em[4] = false;
        const int slot[NB] = {sbE + i2.slot, sbE + i4.slot, sb1 + i1.slot, sb7 + i7.slot, 0};
        const int lin[NB] = {lbE + i2.lin, lbE + i4.lin, lb1 + i1.lin, lb7 + i7.lin, (hx ? lb1 : lbE) + hA.lin};
        batch(NB, lin, slot);
        if (le) c2k[i2.e] = rv[0], c4k[i4.e] = rv[1];
        if (l1) sC1[i1.e] = rv[2];
        if (lv[4]) (hx ? sC1 : (hcA == 2 ? c2k : c4k))[hA.e] = rv[4];
        if (DEC && LV1 && le && oe) {  // the 2-lattice points of plane k are outputs too
          const double v = Ek[i1.e];
          reinterpret_cast<T*>(A.out)[lbE + i1.lin] = (T)v;
          q.nf |= !isfinite(v);
        }
      }
      __syncthreads();
      // the inputs of phase k+1 land in the slots of planes k-3 (E, odd
      // field) and k-1 (even field), free from here on
      stage(k + 1);
      // ---- half 2: c6 of plane k | c3, c5 of odd m1 | halo of c3 / c5
      {
        const double* b0 = sC2 + ((m1 - 1) & MC) * G::S2;
        const double* b1 = sC2 + (m1 & MC) * G::S2;
        const double* b2 = sC2 + ((m1 + 1) & MC) * G::S2;
        const double* b3 = sC2 + ((m1 + 2) & MC) * G::S2;
        const double* d0 = sC4 + ((m1 - 1) & MC) * G::S4;
        const double* d1 = sC4 + (m1 & MC) * G::S4;
        const double* d2 = sC4 + ((m1 + 1) & MC) * G::S4;
        const double* d3 = sC4 + ((m1 + 2) & MC) * G::S4;
        const bool h3 = hcB == 3;
        const double *x0 = h3 ? b0 : d0, *x1 = h3 ? b1 : d1, *x2 = h3 ? b2 : d2, *x3 = h3 ? b3 : d3;
        const int sb = h3 ? G::EZP : 1, eb = h3 ? hB.e : hB.ez;
        double tp[7][4], res[7];
#pragma unroll
        for (int t = 0; t < 4; t++) {
          tp[0][t] = c4k[i6.e + t * G::HZ];  // c6 along y
          tp[1][t] = c2k[i6.ez + t];         // c6 along z
          tp[3][t] = sC1[i3.e + t * G::EZP];  // c3 along y
          tp[5][t] = sC1[i5.ez + t];          // c5 along z
          tp[6][t] = sC1[eb + t * sb];        // halo in plane
        }
        tp[2][0] = b0[i3.e], tp[2][1] = b1[i3.e], tp[2][2] = b2[i3.e], tp[2][3] = b3[i3.e];  // c3 along x
        tp[4][0] = d0[i5.e], tp[4][1] = d1[i5.e], tp[4][2] = d2[i5.e], tp[4][3] = d3[i5.e];  // c5 along x
        double hxv[4] = {x0[hB.e], x1[hB.e], x2[hB.e], x3[hB.e]};
        if (!DEC) {
          o[0] = (double)fe[i6.f], o[1] = (double)f1[i3.f], o[2] = (double)f1[i5.f], o[3] = (double)f1[hB.f];
        } else {
          cd[0] = k6, cd[1] = k3, cd[2] = k5, cd[3] = kB;
        }
        stencils(tp, res, 7);
        double hres[1];
        {
          double htp[1][4] = {{hxv[0], hxv[1], hxv[2], hxv[3]}};
          stencils(htp, hres, 1);
        }
        auto avg2 = [](double a, double b) { return __dmul_rn(__dadd_rn(__dadd_rn(0.0, a), b), 0.5); };
        p[0] = avg2(res[0], res[1]);  // axes y, z
        p[1] = avg2(res[2], res[3]);  // x, y
        p[2] = avg2(res[4], res[5]);  // x, z
        p[3] = avg2(hres[0], res[6]);  // x, then y (c3) or z (c5)
        lv[0] = le, lv[1] = l1, lv[2] = l1, lv[3] = hcB != 0 && l1;
        em[0] = le && oe, em[1] = l1, em[2] = l1, em[3] = false;
        const int slot[NB] = {sbE + i6.slot, sb1 + i3.slot, sb1 + i5.slot, 0, 0};
        const int lin[NB] = {lbE + i6.lin, lb1 + i3.lin, lb1 + i5.lin, lb1 + hB.lin, 0};
        batch(4, lin, slot);
        if (le) c6k[i6.e] = rv[0];
        if (l1) sC3[i3.e] = rv[1], sC5[i5.e] = rv[2];
        if (lv[3]) (h3 ? sC3 : sC5)[hB.e] = rv[3];
      }
    };
    if (fast)
      fast_body();
    else
      phase_body(BT<false>{});
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
  // thread-safe one-time lookup (a 'tried' flag set before the pointer let a
  // concurrent caller see no entry point and take another kernel path)
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
  }();
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
  static const bool attr = [&] {  // once per process, thread-safe (C++11 static init)
    cudaFuncSetAttribute((const void*)k_march<T, DEC, LINEAR, LV1, MTY, MTZ>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::bytes);
    return true;
  }();
  (void)attr;
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
  // enough CTAs for ~6 waves of 148 SMs x 2 resident CTAs (a short tail),
  // segments of >= 8 even planes
  const long long tiles = ((g.D[2] + MTZ - 1) / MTZ) * ((g.D[1] + MTY - 1) / MTY);
  const long long nep = (g.D[0] + 1) / 2;
  long long seg = nep;
  while (seg > 8 && tiles * ((nep + seg - 1) / seg) < 6 * 2 * kSMs) seg = (seg + 1) / 2;
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
