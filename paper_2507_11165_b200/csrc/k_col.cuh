// k_col.cuh -- column-mapped level kernels for 3D fields (16^3 lattice tiles).
//
// Same tile, shared-memory class arrays and arithmetic as k_level.cuh (one
// f64 array per parity class with a +-3 halo on even axes, halo recompute,
// phases separated by __syncthreads), but a different thread mapping: a lane
// owns one (y, z) column of a class and walks it along x with a fully
// unrolled loop.  Consequences:
//  * all per-point addresses (shared memory, field, Eq. 3 slot, E lattice)
//    are a per-column base plus a compile-time / strength-reduced offset,
//    so the integer work per point is a few adds instead of div/mod chains;
//  * stencils along x read a register window (n + 3 loads for n targets);
//  * lanes of a warp are consecutive in z, so shared-memory and global
//    accesses stay contiguous across the warp;
//  * the classes of one phase are independent, so warps take (class, column
//    chunk) tasks from one flattened list and no lane idles on a small class;
//  * the Huffman histogram counts the dominant code 128 in a register.
// Reference: predictor.py:181-304 (prediction), :313-329 (quantize), :397-411
// (replay), ordering.py:68-84 (slot of every code).
#pragma once
#include "k_level.cuh"

namespace hb {

constexpr int CW = 5;               // warps per CTA
constexpr int C_THREADS = CW * 32;

// Shared-memory layout of the class arrays.  seq1d keeps every class live to
// the last phase (TileShape order, + a class-7 staging area).  multidim reads
// class 0 only in phase 1 and classes 1/2/4 only in phase 2, so classes
// 3/5/6 overlay class 0 and the class-7 staging overlays 1/2/4:
//   [ 1 | 2 | 4 ][ 0 -> 3 | 5 | 6 ]      5016 doubles (40 KB) for 16^3 tiles
template <class TL, bool MD>
struct Lay {
  static constexpr __host__ __device__ int off(int c) {
    if (!MD) return c == 7 ? TL::total() : TL::off(c);
    const int s124 = TL::size(1) + TL::size(2) + TL::size(4);
    switch (c) {
      case 1: return 0;
      case 2: return TL::size(1);
      case 4: return TL::size(1) + TL::size(2);
      case 0:
      case 3: return s124;
      case 5: return s124 + TL::size(3);
      case 6: return s124 + TL::size(3) + TL::size(5);
      default: return 0;  // class-7 staging
    }
  }
  static constexpr __host__ __device__ int total() {
    if (!MD) return TL::total() + TL::size(7);
    const int a = off(0) + TL::size(0), b = off(6) + TL::size(6);
    return a > b ? a : b;
  }
};

// CLS: parity mask (bit a = odd on axis a); AXM: interpolation axes; HALO:
// even axes computed over the halo; SEG: the x range of a column is split in
// SEG tasks (balances phases with few columns)
template <int CLS_, int AXM_, int HALO_, int SEG_ = 1>
struct Cls {
  static constexpr int CLS = CLS_, AXM = AXM_, HALO = HALO_, SEG = SEG_;
};

struct ColAcc {
  unsigned h127, h128, h129;  // owned points with the three dominant codes (compress)
  bool bad, nf;
};

// code 0 on decompress: the outlier value at linear index `lin`
// (predictor.py:400-405; orphan -> ArchiveError).  Rare, kept out of line.
static __device__ __noinline__ double outlier_value(const LvArgs& A, const CtaCtx& c, unsigned long long lin, bool& bad) {
  unsigned long long a0 = 0, a1 = c.ocount;
  while (a0 < a1) {
    const unsigned long long mid = (a0 + a1) >> 1;
    if (A.oidx[mid] < lin)
      a0 = mid + 1;
    else
      a1 = mid;
  }
  if (a0 < c.ocount && A.oidx[a0] == lin) return A.oval[a0];
  bad = true;
  return 0.0;
}

// runtime class geometry (CLS = parity mask, bit a = odd on axis a)
template <class TL>
__device__ __forceinline__ int rext(int cls, int a) {
  return ((cls >> a) & 1) ? TL::no(a) : TL::E(a);
}
template <class TL, bool MD>
__device__ __forceinline__ int roff(int cls) {
  int o = Lay<TL, MD>::off(0);
#pragma unroll
  for (int k = 1; k < 8; k++) o = cls == k ? Lay<TL, MD>::off(k) : o;
  return o;
}

// One task of one class: a lane owns one (y, z) column of the class and
// walks x over [ibeg, iend).  K = number of interpolation axes (compile
// time, equal for all classes of a phase); the class itself is a runtime
// parameter so a phase executes ONE loop body (small instruction footprint).
// MODE 0: only issue the task's staging copies; MODE 1: only compute (the
// caller has waited for the copies).
template <class TL, bool MD, int K, bool LINEAR, bool DEC, typename T, bool INT, int MODE>
__device__ __forceinline__ void col_body(const LvArgs& A, const CtaCtx& c, double* sm, unsigned* shist, int CLS,
                                         int AXM, int HALO, int SEG, int task, ColAcc& acc) {
  const bool odd0 = CLS & 1, odd1 = (CLS >> 1) & 1, odd2 = (CLS >> 2) & 1;
  const bool h0 = HALO & 1, h1 = (HALO >> 1) & 1, h2 = (HALO >> 2) & 1;
  const int n0 = odd0 ? TL::no(0) : (h0 ? TL::E(0) : TL::ne(0));
  const int n2 = odd2 ? TL::no(2) : (h2 ? TL::E(2) : TL::ne(2));
  const int lo0 = (odd0 || h0) ? 0 : TL::eoff(0), lo1 = (odd1 || h1) ? 0 : TL::eoff(1);
  const int lo2 = (odd2 || h2) ? 0 : TL::eoff(2);
  const int n1 = odd1 ? TL::no(1) : (h1 ? TL::E(1) : TL::ne(1));
  const int chunk = task / SEG, seg = task - chunk * SEG;
  const int ibeg = seg * n0 / SEG, iend = (seg + 1) * n0 / SEG;
  const int col = chunk * 32 + (threadIdx.x & 31);
  if (col >= n1 * n2) return;
  static_assert(TL::no(2) == 8, "column split assumes 8 / 11 points along z");
  const int i1 = n2 == 8 ? col >> 3 : (int)((unsigned)col / 11u), i2 = col - i1 * n2;
  const int l1 = lo1 + i1, l2 = lo2 + i2;
  const LevelGeom& g = A.g;
  const int xb0 = c.hb0[0] - (odd0 ? 0 : TL::eoff(0)) + lo0;
  const int xb1 = c.hb0[1] - (odd1 ? 0 : TL::eoff(1)) + lo1;
  const int xb2 = c.hb0[2] - (odd2 ? 0 : TL::eoff(2)) + lo2;
  const int ilo0 = -xb0, ihi0 = ((c.D[0] - odd0 + 1) >> 1) - xb0;
  if (!INT) {
    const int ilo1 = -xb1, ihi1 = ((c.D[1] - odd1 + 1) >> 1) - xb1;
    const int ilo2 = -xb2, ihi2 = ((c.D[2] - odd2 + 1) >> 1) - xb2;
    if (i1 < ilo1 || i1 >= ihi1 || i2 < ilo2 || i2 >= ihi2) return;  // column outside the field
  }
  bool own12 = true;
  if (!odd1 && h1) own12 &= l1 >= TL::eoff(1) && l1 < TL::eoff(1) + TL::ne(1);
  if (!odd2 && h2) own12 &= l2 >= TL::eoff(2) && l2 < TL::eoff(2) + TL::ne(2);
  // owned x range [olo, ohi) in local index l0
  const int olo = (odd0 || !h0) ? 0 : TL::eoff(0), ohi = (odd0 || !h0) ? 64 : TL::eoff(0) + TL::ne(0);
  const int P00 = 2 * xb0 + odd0, P1 = 2 * (xb1 + i1) + odd1, P2 = 2 * (xb2 + i2) + odd2;
  // per-column affine bases (element index, Eq. 3 slot, E index)
  const int s = (int)g.s;
  const int kl0 = (int)g.kl[0];
  const int lin_c = (int)((((long long)P00 * s) * g.d[1] + (long long)P1 * s) * g.d[2] + (long long)P2 * s);
  long long slc = g.prefix + ((long long)P00 * g.D[1] + P1) * g.D[2] + P2 - (((long long)P00 + 1) >> 1) * g.eyez;
  if (!odd0) {
    slc -= (((long long)P1 + 1) >> 1) * g.ez;
    if (!odd1) slc -= ((long long)P2 + 1) >> 1;
  }
  const int ks0 = (int)g.ks0;
  const int ke0 = (int)g.ke[0];
  const int E_c = (int)((((long long)P00 * s) >> 1) * g.Ed[1] * g.Ed[2] + (((long long)P1 * s) >> 1) * g.Ed[2] +
                        ((long long)P2 * s >> 1));
  uint8_t* seqp = A.seq + (int)slc;
  // ---- stage the column's originals (compress) or code words (decompress)
  // in the class's own shared-memory slots (class 7: a staging area); a slot
  // is overwritten with the reconstruction once its point is done, and no
  // class reads its own array, so this is race-free.
  const int e1 = rext<TL>(CLS, 1), e2 = rext<TL>(CLS, 2);
  const int ps = e1 * e2;  // x step in this class's array
  double* bs = sm + roff<TL, MD>(CLS) + l1 * e2 + l2;
  if (MODE == 0) {
    const uint8_t* gs = DEC ? seqp : reinterpret_cast<const uint8_t*>(A.field) + (long long)lin_c * sizeof(T);
    const int gstep = DEC ? ks0 : kl0 * (int)sizeof(T);
#pragma unroll 4
    for (int i0 = ibeg; i0 < iend; i0++) {
      const bool live0 = INT || (i0 >= ilo0 && i0 < ihi0);
      const uint8_t* src = gs + i0 * gstep;
      if (!DEC) {
        cp_async<sizeof(T)>(bs + (lo0 + i0) * ps, live0 ? src : reinterpret_cast<const uint8_t*>(A.field), live0);
      } else {
        const uintptr_t ad = reinterpret_cast<uintptr_t>(live0 ? src : A.seq) & ~uintptr_t(3);
        cp_async<4>(bs + (lo0 + i0) * ps, reinterpret_cast<const void*>(ad), live0);
      }
    }
    return;
  }
  // ---- the K interpolation axes in ascending order (predictor.py:247-256)
  const double* sb[K];
  int sp[K], st[K], sax[K], scls[K];
  {
    int m = AXM;
#pragma unroll
    for (int j = 0; j < K; j++) {
      const int a = __ffs(m) - 1;
      m &= m - 1;
      const int cn = CLS & ~(1 << a);
      const int f1 = rext<TL>(cn, 1), f2 = rext<TL>(cn, 2);
      sax[j] = a;
      sb[j] = sm + roff<TL, MD>(cn) + l1 * f2 + l2;
      sp[j] = f1 * f2;
      st[j] = a == 0 ? f1 * f2 : (a == 1 ? f2 : 1);
      // stencil class of the y / z axes is uniform over the column
      scls[j] = INT ? (LINEAR ? ST_MID : ST_CUBIC)
                    : classify(a == 1 ? P1 : P2, a == 1 ? c.D[1] : c.D[2], 1, LINEAR);
    }
  }
#pragma unroll 2
  for (int i0 = ibeg; i0 < iend; i0++) {
    const int l0 = lo0 + i0;
    if (!INT && !(i0 >= ilo0 && i0 < ihi0)) continue;
    const bool owned = own12 && l0 >= olo && l0 < ohi;
    double pv[K];
    int ov[K];
#pragma unroll
    for (int j = 0; j < K; j++) {
      int cls = scls[j];
      if (!INT && sax[j] == 0) cls = classify(P00 + 2 * i0, c.D[0], 1, LINEAR);
      const double* b = sb[j] + l0 * sp[j];
      const int t = st[j];
      pv[j] = INT ? apply_stencil(LINEAR ? ST_MID : ST_CUBIC, b[0], b[t], b[2 * t], b[3 * t])
                  : apply_stencil(cls, b[0], b[t], b[2 * t], b[3 * t]);
      ov[j] = INT ? (LINEAR ? 2 : 4) : stencil_order(cls);
    }
    const double pred = K == 1 ? pv[0] : combine_axes(K, pv, ov);
    double* slotp = bs + l0 * ps;
    double r;
    if (!DEC) {
      const double o = sizeof(T) == 4 ? (double)*reinterpret_cast<const float*>(slotp) : *slotp;
      const int code = quantize_fast<sizeof(T) == 4>(o, pred, c.eb, c.two_eb, c.inv_two_eb, &r);
      if (owned) {
        seqp[i0 * ks0] = (uint8_t)code;
        if (c.wE) A.E[E_c + i0 * ke0] = r;
        if (code == 128) {
          acc.h128++;
        } else if (code == 127) {
          acc.h127++;
        } else if (code == 129) {
          acc.h129++;
        } else {
          atomicAdd(&shist[code], 1u);
          if (code == 0) {  // outlier (non-finite originals always land here)
            const int lin = lin_c + i0 * kl0;
            atomicOr(&A.obm[lin >> 5], 1u << (lin & 31));
            acc.bad |= !isfinite(o);
          }
        }
      }
    } else {
      const unsigned word = *reinterpret_cast<const unsigned*>(slotp);
      const int code = (word >> (8 * (reinterpret_cast<uintptr_t>(seqp + i0 * ks0) & 3))) & 0xFF;
      if (code != 0) {
        r = dequantize(pred, c.two_eb, code);
      } else {
        r = outlier_value(A, c, (unsigned long long)(unsigned)(lin_c + i0 * kl0), acc.bad);
      }
      if (owned) {
        if (c.wE) {
          A.E[E_c + i0 * ke0] = r;
        } else {
          reinterpret_cast<T*>(A.out)[lin_c + i0 * kl0] = (T)r;
          acc.nf |= !isfinite(r);
        }
      }
    }
    if (CLS != 7) *slotp = r;
  }
}

// warp tasks of one phase: the classes Cs (all with K axes) flattened into
// (class, column chunk, x segment) tasks, handed out round-robin to warps
template <class TL, class C>
struct ColTasks {
  static constexpr bool od(int a) { return (C::CLS >> a) & 1; }
  static constexpr bool hl(int a) { return (C::HALO >> a) & 1; }
  static constexpr int n(int a) { return od(a) ? TL::no(a) : (hl(a) ? TL::E(a) : TL::ne(a)); }
  static constexpr int value = n(0) * n(1) * n(2) == 0 ? 0 : (n(1) * n(2) + 31) / 32 * C::SEG;
};

// MODE 0: issue the staging copies of all of this warp's tasks; MODE 1:
// compute them (after cp.async.wait_all -- each thread reads back only its
// own copies, and a phase never reads the slots of its own classes).
template <class TL, bool MD, int K, bool LINEAR, bool DEC, typename T, bool INT, int MODE, class... Cs>
__device__ __forceinline__ void col_tasks(const LvArgs& A, const CtaCtx& c, double* sm, unsigned* sh, ColAcc& acc) {
  constexpr int tot = (ColTasks<TL, Cs>::value + ...);
  constexpr int nt[] = {ColTasks<TL, Cs>::value...};
  constexpr int cl[] = {Cs::CLS...}, ax[] = {Cs::AXM...}, ha[] = {Cs::HALO...}, sg[] = {Cs::SEG...};
  const int warp = threadIdx.x >> 5;
#pragma unroll 1
  for (int t = warp; t < tot; t += CW) {
    int CLS = cl[0], AXM = ax[0], HALO = ha[0], SEG = sg[0], lt = t, acc_n = 0;
#pragma unroll
    for (int k = 1; k < (int)sizeof...(Cs); k++) {
      acc_n += nt[k - 1];
      if (t >= acc_n) CLS = cl[k], AXM = ax[k], HALO = ha[k], SEG = sg[k], lt = t - acc_n;
    }
    col_body<TL, MD, K, LINEAR, DEC, T, INT, MODE>(A, c, sm, sh, CLS, AXM, HALO, SEG, lt, acc);
  }
}

// one phase; STAGED = its copies were issued earlier (phase 1, overlapped
// with the lattice load)
template <class TL, bool MD, int K, bool LINEAR, bool DEC, typename T, bool INT, bool STAGED, class... Cs>
__device__ __forceinline__ void col_phase(const LvArgs& A, const CtaCtx& c, double* sm, unsigned* sh, ColAcc& acc) {
  if (!STAGED) {
    col_tasks<TL, MD, K, LINEAR, DEC, T, INT, 0, Cs...>(A, c, sm, sh, acc);
    cp_async_wait_all();
  }
  col_tasks<TL, MD, K, LINEAR, DEC, T, INT, 1, Cs...>(A, c, sm, sh, acc);
}

// multidim (predictor.py:282-296); SEG balances the 5 warps: 10 / 10 / 4 tasks
// MODE 0: issue phase 1's copies; MODE 1: run the level (phase 1 already staged)
template <class TL, bool LINEAR, bool DEC, typename T, bool INT, int MODE>
__device__ __forceinline__ void col_multidim(const LvArgs& A, const CtaCtx& c, double* sm, unsigned* sh, ColAcc& acc) {
  using P1 = Cls<1, 1, 6>;
  using P2 = Cls<2, 2, 5>;
  using P4 = Cls<4, 4, 3>;
  if (MODE == 0) {
    col_tasks<TL, true, 1, LINEAR, DEC, T, INT, 0, P1, P2, P4>(A, c, sm, sh, acc);
    return;
  }
  col_phase<TL, true, 1, LINEAR, DEC, T, INT, true, P1, P2, P4>(A, c, sm, sh, acc);
  __syncthreads();
  col_phase<TL, true, 2, LINEAR, DEC, T, INT, false, Cls<3, 3, 4>, Cls<5, 5, 2>, Cls<6, 6, 1, 2>>(A, c, sm, sh, acc);
  __syncthreads();
  col_phase<TL, true, 3, LINEAR, DEC, T, INT, false, Cls<7, 7, 0, 2>>(A, c, sm, sh, acc);
}

// seq1d (predictor.py:267-280) with axis order (O0, O1, O2)
template <class TL, int O0, int O1, int O2, bool LINEAR, bool DEC, typename T, bool INT, int MODE>
__device__ __forceinline__ void col_seq1d(const LvArgs& A, const CtaCtx& c, double* sm, unsigned* sh, ColAcc& acc) {
  constexpr int b0 = 1 << O0, b1 = 1 << O1, b2 = 1 << O2;
  if (MODE == 0) {
    col_tasks<TL, false, 1, LINEAR, DEC, T, INT, 0, Cls<b0, b0, b1 | b2>>(A, c, sm, sh, acc);
    return;
  }
  col_phase<TL, false, 1, LINEAR, DEC, T, INT, true, Cls<b0, b0, b1 | b2>>(A, c, sm, sh, acc);
  __syncthreads();
  col_phase<TL, false, 1, LINEAR, DEC, T, INT, false, Cls<b1, b1, b2>, Cls<b0 | b1, b1, b2>>(A, c, sm, sh, acc);
  __syncthreads();
  col_phase<TL, false, 1, LINEAR, DEC, T, INT, false, Cls<b2, b2, 0>, Cls<b0 | b2, b2, 0>, Cls<b1 | b2, b2, 0>,
            Cls<7, b2, 0>>(A, c, sm, sh, acc);
}

template <int OID>
struct SeqOrder {
  static constexpr int o0 = OID < 2 ? 0 : (OID < 4 ? 1 : 2);
  static constexpr int o1 = (OID == 0 || OID == 5) ? 1 : ((OID == 1 || OID == 3) ? 2 : 0);
  static constexpr int o2 = 3 - o0 - o1;
};

template <class TL, int CFG, int OID, bool DEC, typename T, bool INT, int MODE>
__device__ __forceinline__ void col_levels(const LvArgs& A, const CtaCtx& c, double* sm, unsigned* sh, ColAcc& acc) {
  constexpr bool LINEAR = CFG & 1;
  if constexpr ((CFG & 2) == 0) {
    col_multidim<TL, LINEAR, DEC, T, INT, MODE>(A, c, sm, sh, acc);
  } else {
    using O = SeqOrder<OID>;
    col_seq1d<TL, O::o0, O::o1, O::o2, LINEAR, DEC, T, INT, MODE>(A, c, sm, sh, acc);
  }
}

// One CTA per 16^3 lattice tile of one level; CFG = the level's interpolation
// config byte (bit0 linear, bit1 seq1d, predictor.py:80-95), OID = seq1d axis order.
// Tiles are split into two launches: the interior box (every stencil
// complete, INT code path) and the boundary shell, so an SM runs one code
// path at a time.  Per axis the interior tiles are [ia, ia + ni).
struct ColPart {
  int ia[3], ni[3], nt[3];
};

__device__ __forceinline__ void col_tile(const ColPart& P, bool interior, unsigned b, int tix[3]) {
  if (interior) {
    const unsigned n12 = (unsigned)(P.ni[1] * P.ni[2]), r = b % n12;
    tix[0] = P.ia[0] + (int)(b / n12);
    tix[1] = P.ia[1] + (int)(r / (unsigned)P.ni[2]);
    tix[2] = P.ia[2] + (int)(r % (unsigned)P.ni[2]);
    return;
  }
  // shell: (x in shell, any y, z) | (x inner, y in shell, any z) | (x, y inner, z in shell)
  auto shell = [&](int a, unsigned k) { return (int)k < P.ia[a] ? (int)k : (int)k + P.ni[a]; };
  const unsigned s0 = (unsigned)(P.nt[0] - P.ni[0]), s1 = (unsigned)(P.nt[1] - P.ni[1]),
                 s2 = (unsigned)(P.nt[2] - P.ni[2]);
  const unsigned c1 = s0 * P.nt[1] * P.nt[2], c2 = (unsigned)P.ni[0] * s1 * P.nt[2];
  if (b < c1) {
    const unsigned n12 = (unsigned)(P.nt[1] * P.nt[2]), r = b % n12;
    tix[0] = shell(0, b / n12), tix[1] = (int)(r / (unsigned)P.nt[2]), tix[2] = (int)(r % (unsigned)P.nt[2]);
  } else if (b < c1 + c2) {
    b -= c1;
    const unsigned n12 = s1 * P.nt[2], r = b % n12;
    tix[0] = P.ia[0] + (int)(b / n12), tix[1] = shell(1, r / (unsigned)P.nt[2]), tix[2] = (int)(r % (unsigned)P.nt[2]);
  } else {
    b -= c1 + c2;
    const unsigned n12 = (unsigned)P.ni[1] * s2, r = b % n12;
    tix[0] = P.ia[0] + (int)(b / n12), tix[1] = P.ia[1] + (int)(r / s2), tix[2] = shell(2, r % s2);
  }
}

template <class TL, typename T, bool DEC, int CFG, int OID, bool INT>
__global__ void __launch_bounds__(C_THREADS, (CFG & 2) == 0 ? 5 : 4) k_level_col(LvArgs A, ColPart P) {
  extern __shared__ double sm[];
  __shared__ unsigned shist[256];
  constexpr bool MD = (CFG & 2) == 0;
  const LevelGeom& g = A.g;
  int tix[3];
  col_tile(P, INT, blockIdx.x, tix);
  CtaCtx c;
  for (int a = 0; a < 3; a++) {
    c.hb0[a] = (tix[a] * TL::t(a)) >> 1;
    c.D[a] = (int)g.D[a];
  }
  c.d1 = g.d[1], c.d2 = g.d[2], c.e1 = g.Ed[1], c.e2 = g.Ed[2], c.s = g.s;
  c.eb = A.st->eb;
  c.two_eb = A.st->two_eb;
  c.inv_two_eb = __ddiv_rn(1.0, c.two_eb);
  c.ocount = DEC ? *A.ocount : 0;
  c.wE = g.level >= 2;
  c.out0 = g.level == 1;
  if (!DEC)
    for (int i = threadIdx.x; i < 256; i += C_THREADS) shist[i] = 0;
  ColAcc acc{0u, 0u, 0u, false, false};
  // the known 2s-lattice (class 0) with halo, from E (cp.async, zero-filled
  // outside): half a warp per row along z, two rows per warp and step
  double* s0 = sm + Lay<TL, MD>::off(0);
  {
    constexpr int e0 = TL::E(0), e1 = TL::E(1), e2 = TL::E(2);
    static_assert(e2 <= 16, "one half-warp per row");
    constexpr int rows = e0 * e1;
    const int lane = threadIdx.x & 31, l2 = lane & 15;
    const int s = (int)c.s, ce1 = (int)c.e1, ce2 = (int)c.e2;
    const int h2 = c.hb0[2] - TL::eoff(2) + l2;
    const bool ok2 = l2 < e2 && (INT || (h2 >= 0 && 2 * h2 < c.D[2]));
    // row = l0 * e1 + l1, walked incrementally (step 2 * CW < e1 rows)
    static_assert(2 * CW < e1, "one wrap per step");
    const int row0 = 2 * (threadIdx.x >> 5) + (lane >> 4);
    int l0 = row0 / e1, l1 = row0 - (row0 / e1) * e1;
    const int hz = h2 * s;
    for (int row = row0; row < rows; row += 2 * CW) {
      const int h0 = c.hb0[0] - TL::eoff(0) + l0, h1 = c.hb0[1] - TL::eoff(1) + l1;
      const bool ok = ok2 && (INT || (h0 >= 0 && 2 * h0 < c.D[0] && h1 >= 0 && 2 * h1 < c.D[1]));
      const int eidx = ((h0 * s) * ce1 + h1 * s) * ce2 + hz;
      if (l2 < e2) cp_async<8>(s0 + row * e2 + l2, A.E + (ok ? eidx : 0), ok);
      l1 += 2 * CW;
      if (l1 >= e1) l1 -= e1, l0++;
    }
    // phase 1's originals / codes go into slots disjoint from class 0
    col_levels<TL, CFG, OID, DEC, T, INT, 0>(A, c, sm, shist, acc);
    cp_async_wait_all();
    if (DEC && c.out0) {  // level 1 writes the even lattice to the output (same rows as copied)
      l0 = row0 / e1, l1 = row0 - (row0 / e1) * e1;
      for (int row = row0; row < rows; row += 2 * CW) {
        const int h0 = c.hb0[0] - TL::eoff(0) + l0, h1 = c.hb0[1] - TL::eoff(1) + l1;
        const bool owned = ok2 && l0 >= TL::eoff(0) && l0 < TL::eoff(0) + TL::ne(0) && l1 >= TL::eoff(1) &&
                           l1 < TL::eoff(1) + TL::ne(1) && l2 >= TL::eoff(2) && l2 < TL::eoff(2) + TL::ne(2) &&
                           2 * h0 < c.D[0] && 2 * h1 < c.D[1];
        if (owned) {
          const double v = s0[row * e2 + l2];
          reinterpret_cast<T*>(A.out)[((2ll * h0) * c.d1 + 2ll * h1) * c.d2 + 2ll * h2] = (T)v;
          acc.nf |= !isfinite(v);
        }
        l1 += 2 * CW;
        if (l1 >= e1) l1 -= e1, l0++;
      }
    }
  }
  __syncthreads();
  col_levels<TL, CFG, OID, DEC, T, INT, 1>(A, c, sm, shist, acc);
  if (DEC && __any_sync(0xffffffffu, acc.nf) && (threadIdx.x & 31) == 0) raise_flag(A.st, F_NONFINITE);
  if (__any_sync(0xffffffffu, acc.bad) && (threadIdx.x & 31) == 0) raise_flag(A.st, DEC ? F_ORPHAN : F_NONFINITE);
  if (!DEC) {
    const unsigned h7 = __reduce_add_sync(0xffffffffu, acc.h127), h8 = __reduce_add_sync(0xffffffffu, acc.h128),
                   h9 = __reduce_add_sync(0xffffffffu, acc.h129);
    if ((threadIdx.x & 31) == 0) {
      if (h7) atomicAdd(&shist[127], h7);
      if (h8) atomicAdd(&shist[128], h8);
      if (h9) atomicAdd(&shist[129], h9);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += C_THREADS)
      if (shist[i]) atomicAdd(&A.st->hist[i], (unsigned long long)shist[i]);
  }
}

template <bool DEC, typename T>
int col_launch(const LvArgs& A, unsigned blocks, int cfg, cudaStream_t s);  // k_col_{c,d}{f,d}.cu

template <typename T, bool DEC, int CFG, int OID>
static int col_launch_one(const LvArgs& A, unsigned /*blocks*/, cudaStream_t s) {
  using TL = Tile3;
  constexpr size_t smem = (size_t)Lay<TL, (CFG & 2) == 0>::total() * 8;
  static const bool attr = [&] {  // once per process, thread-safe (C++11 static init)
    for (const void* f : {(const void*)k_level_col<TL, T, DEC, CFG, OID, true>,
                          (const void*)k_level_col<TL, T, DEC, CFG, OID, false>}) {
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    return true;
  }();
  (void)attr;
  // interior box per axis: tiles t with 16t >= 2 and 16t + 16 + 3 <= D
  ColPart P;
  bool empty = false;
  for (int a = 0; a < 3; a++) {
    P.nt[a] = A.g.ntile[a];
    const long long D = A.g.D[a];
    const int ib = D >= TL::t(a) + 3 ? (int)((D - TL::t(a) - 3) / TL::t(a)) + 1 : 0;
    P.ia[a] = 1;
    P.ni[a] = ib > 1 ? ib - 1 : 0;
    empty |= P.ni[a] == 0;
  }
  if (empty)
    for (int a = 0; a < 3; a++) P.ia[a] = 0, P.ni[a] = 0;
  const unsigned all = (unsigned)(P.nt[0] * P.nt[1] * P.nt[2]);
  const unsigned inner = (unsigned)(P.ni[0] * P.ni[1] * P.ni[2]);
  if (inner) k_level_col<TL, T, DEC, CFG, OID, true><<<inner, C_THREADS, smem, s>>>(A, P);
  if (all > inner) k_level_col<TL, T, DEC, CFG, OID, false><<<all - inner, C_THREADS, smem, s>>>(A, P);
  return (inner ? 1 : 0) + (all > inner ? 1 : 0);
}

// definition, included by the four instantiation units
template <bool DEC, typename T>
int col_launch_impl(const LvArgs& A, unsigned blocks, int cfg, cudaStream_t s) {
  const int oid = order_id(A.g);
  switch (cfg & 3) {
    case 0: return col_launch_one<T, DEC, 0, 0>(A, blocks, s);
    case 1: return col_launch_one<T, DEC, 1, 0>(A, blocks, s);
    case 2:
      switch (oid) {
        case 0: return col_launch_one<T, DEC, 2, 0>(A, blocks, s);
        case 1: return col_launch_one<T, DEC, 2, 1>(A, blocks, s);
        case 2: return col_launch_one<T, DEC, 2, 2>(A, blocks, s);
        case 3: return col_launch_one<T, DEC, 2, 3>(A, blocks, s);
        case 4: return col_launch_one<T, DEC, 2, 4>(A, blocks, s);
        default: return col_launch_one<T, DEC, 2, 5>(A, blocks, s);
      }
    default:
      switch (oid) {
        case 0: return col_launch_one<T, DEC, 3, 0>(A, blocks, s);
        case 1: return col_launch_one<T, DEC, 3, 1>(A, blocks, s);
        case 2: return col_launch_one<T, DEC, 3, 2>(A, blocks, s);
        case 3: return col_launch_one<T, DEC, 3, 3>(A, blocks, s);
        case 4: return col_launch_one<T, DEC, 3, 4>(A, blocks, s);
        default: return col_launch_one<T, DEC, 3, 5>(A, blocks, s);
      }
  }
}

// 3D fields with 32-bit element indices; false = caller uses another kernel
template <bool DEC>
static inline int launch_col(LevelGeom g, const LvArgs& base, int prec, int cfg, cudaStream_t s) {
  if (cfg < 0) return 0;  // the config byte must be known on the host
  if (!(g.d[0] > 1 && g.d[1] > 1 && g.d[2] > 1)) return 0;
  if (g.d[0] * g.d[1] * g.d[2] >= (1ll << 31) - (1ll << 24)) return 0;
  using TL = Tile3;
  LvArgs A = base;
  for (int a = 0; a < 3; a++) {
    g.T[a] = TL::t(a);
    g.ntile[a] = (int)((g.D[a] + TL::t(a) - 1) / TL::t(a));
  }
  A.g = g;
  const unsigned blocks = (unsigned)((long long)g.ntile[0] * g.ntile[1] * g.ntile[2]);
  return prec == 4 ? col_launch<DEC, float>(A, blocks, cfg, s) : col_launch<DEC, double>(A, blocks, cfg, s);
}

}  // namespace hb
