// k_march.cuh -- 2.5D "marching" level kernels for 3D fields.
//
// Same arithmetic as the tiled kernels (k_level.cuh), different blocking: a
// CTA owns a 32x32 column of the level lattice in (y, z) and marches along x
// over a segment of planes.  Even-x planes (the lattice eee and the classes
// odd in y and/or z) depend only on their own plane; odd-x planes interpolate
// along x from the four even planes at x-3, x-1, x+1, x+3, which stay
// resident in a 4-slot ring.  So the +-3 halo is needed only in y and z, the
// halo-recompute factor drops from ~1.54x (16^3 tiles) to ~1.17x, and each
// class is a 2D box per plane (cheap index math).  Reference:
// predictor.py:181-304 / 313-329 / 397-411, ordering.py:68-84.
#pragma once
#include "k_level.cuh"
#include "k_march_plan.h"

namespace hb {


struct MarchCtx {
  int hb1, hb2;  // half-index of the column origin in y, z
  int D0, D1, D2;
  int X0, X1;    // owned plane range [X0, X1)
  double eb, two_eb, inv_two_eb;
  unsigned long long ocount;
};

__host__ __device__ constexpr int m_ext(int cls, int a) { return ((cls >> a) & 1) ? MH : ME; }

// offset of class `cls` of plane P0 in shared memory (-1 = not stored)
__device__ __forceinline__ int m_base(int cls, int P0) {
  if (!(cls & 1)) {
    const int slot = (P0 >> 1) & 3;
    const int o = cls == 0 ? SL_EEE : (cls == 2 ? SL_EY : (cls == 4 ? SL_EZ : SL_EYZ));
    return slot * SL_SIZE + o;
  }
  return cls == 1 ? OD_X : (cls == 3 ? OD_XY : (cls == 5 ? OD_XZ : -1));
}

// One class of one plane.  CLS: parity mask (bit0 x, bit1 y, bit2 z); AXM:
// interpolation axes; HALO: even y/z axes computed over the halo; SID: staging
// area index within the phase.
template <int CLS, int AXM, int HALO, int SID, bool LINEAR, bool DEC, typename T, bool INT>
__device__ __forceinline__ void m_issue(const LvArgs& A, const MarchCtx& c, double* sm, int P0) {
  constexpr bool oy = (CLS >> 1) & 1, oz = (CLS >> 2) & 1;
  constexpr int ny = oy ? MH : (((HALO >> 1) & 1) ? ME : MH), nz = oz ? MH : (((HALO >> 2) & 1) ? ME : MH);
  constexpr int loy = (oy || ((HALO >> 1) & 1)) ? 0 : 1, loz = (oz || ((HALO >> 2) & 1)) ? 0 : 1;
  constexpr int total = ny * nz;
  const LevelGeom& g = A.g;
  const int xby = c.hb1 - (oy ? 0 : 1) + loy, xbz = c.hb2 - (oz ? 0 : 1) + loz;
  const int iylo = -xby, iyhi = ((c.D1 - (int)oy + 1) >> 1) - xby;
  const int izlo = -xbz, izhi = ((c.D2 - (int)oz + 1) >> 1) - xbz;
  const long long P1b = 2ll * xby + oy, P2b = 2ll * xbz + oz;
  const int s = (int)g.s;
  T* stf = reinterpret_cast<T*>(sm + M_STAGE + SID * ME * ME);
  uint32_t* stc = reinterpret_cast<uint32_t*>(sm + M_STAGE + SID * ME * ME);
  if (!DEC) {
    const int lin0 = (int)((((long long)P0 * s) * g.d[1] + P1b * s) * g.d[2] + P2b * s);
    const int kly = (int)g.kl[1], klz = (int)g.kl[2];
    for (int idx = threadIdx.x; idx < total; idx += M_THREADS) {
      const int iy = idx / nz, iz = idx % nz;
      const bool live = INT || (iy >= iylo && iy < iyhi && iz >= izlo && iz < izhi);
      const T* src = reinterpret_cast<const T*>(A.field) + (live ? lin0 + iy * kly + iz * klz : 0);
      cp_async<sizeof(T)>(stf + idx, src, live);
    }
  } else {
    long long sl0 = g.prefix + ((long long)P0 * g.D[1] + P1b) * g.D[2] + P2b - (((long long)P0 + 1) >> 1) * g.eyez;
    if (!(CLS & 1)) {
      sl0 -= ((P1b + 1) >> 1) * g.ez;
      if (!oy) sl0 -= (P2b + 1) >> 1;
    }
    const int ksy = (int)((CLS & 1) ? g.ks1_odd0 : g.ks1_even0);
    constexpr int ksz = ((CLS & 1) || oy) ? 2 : 1;
    for (int idx = threadIdx.x; idx < total; idx += M_THREADS) {
      const int iy = idx / nz, iz = idx % nz;
      const bool live = INT || (iy >= iylo && iy < iyhi && iz >= izlo && iz < izhi);
      const int sl = live ? (int)sl0 + iy * ksy + iz * ksz : 0;
      const uintptr_t ad = reinterpret_cast<uintptr_t>(A.seq + sl) & ~uintptr_t(3);
      cp_async<4>(stc + idx, reinterpret_cast<const void*>(ad), live);
    }
  }
}

template <int CLS, int AXM, int HALO, int SID, bool LINEAR, bool DEC, typename T, bool INT>
__device__ __forceinline__ void m_compute(const LvArgs& A, const MarchCtx& c, double* sm, unsigned* shist, int P0,
                                          bool& bad, bool& nf) {
  constexpr bool oy = (CLS >> 1) & 1, oz = (CLS >> 2) & 1;
  constexpr int ny = oy ? MH : (((HALO >> 1) & 1) ? ME : MH), nz = oz ? MH : (((HALO >> 2) & 1) ? ME : MH);
  constexpr int loy = (oy || ((HALO >> 1) & 1)) ? 0 : 1, loz = (oz || ((HALO >> 2) & 1)) ? 0 : 1;
  constexpr int total = ny * nz;
  constexpr int ex_z = m_ext(CLS, 2);
  const LevelGeom& g = A.g;
  const int s = (int)g.s;
  const int xby = c.hb1 - (oy ? 0 : 1) + loy, xbz = c.hb2 - (oz ? 0 : 1) + loz;
  const int iylo = -xby, iyhi = ((c.D1 - (int)oy + 1) >> 1) - xby;
  const int izlo = -xbz, izhi = ((c.D2 - (int)oz + 1) >> 1) - xbz;
  const long long P1b = 2ll * xby + oy, P2b = 2ll * xbz + oz;
  const bool own_x = P0 >= c.X0 && P0 < c.X1;
  // affine address maps of this plane / class
  const int lin0 = (int)((((long long)P0 * s) * g.d[1] + P1b * s) * g.d[2] + P2b * s);
  const int kly = (int)g.kl[1], klz = (int)g.kl[2];
  long long sl0l = g.prefix + ((long long)P0 * g.D[1] + P1b) * g.D[2] + P2b - (((long long)P0 + 1) >> 1) * g.eyez;
  if (!(CLS & 1)) {
    sl0l -= ((P1b + 1) >> 1) * g.ez;
    if (!oy) sl0l -= (P2b + 1) >> 1;
  }
  const int sl0 = (int)sl0l;
  const int ksy = (int)((CLS & 1) ? g.ks1_odd0 : g.ks1_even0);
  constexpr int ksz = ((CLS & 1) || oy) ? 2 : 1;
  const int E0 = (int)(((((long long)P0 * s) >> 1) * g.Ed[1] + ((P1b * s) >> 1)) * g.Ed[2] + ((P2b * s) >> 1));
  const int key = (int)g.ke[1], kez = (int)g.ke[2];
  // x-stencil (uniform over the plane) and its source planes
  int clsx = 0;
  const double* xs[4] = {nullptr, nullptr, nullptr, nullptr};
  if (AXM & 1) {
    clsx = classify(P0, c.D0, 1, LINEAR);
    for (int k = 0; k < 4; k++) {
      const int Pn = P0 - 3 + 2 * k;
      xs[k] = sm + m_base(CLS ^ 1, Pn & ~0) + 0;
      if (Pn < 0) xs[k] = sm;  // unused by clsx (m3 false)
    }
  }
  const T* stf = reinterpret_cast<const T*>(sm + M_STAGE + SID * ME * ME);
  const uint32_t* stc = reinterpret_cast<const uint32_t*>(sm + M_STAGE + SID * ME * ME);
  const int base_c = m_base(CLS, P0);
  const int lane = threadIdx.x & 31;
  constexpr int ITERS = (total + M_THREADS - 1) / M_THREADS;
#pragma unroll 1
  for (int it = 0; it < ITERS; it++) {
    const int idx = it * M_THREADS + threadIdx.x;
    const int iy = idx / nz, iz = idx % nz;
    const bool live = idx < total && (INT || (iy >= iylo && iy < iyhi && iz >= izlo && iz < izhi));
    const int ly = loy + iy, lz = loz + iz;
    bool owned = own_x;
    if (!oy && ((HALO >> 1) & 1)) owned &= ly >= 1 && ly <= MH;
    if (!oz && ((HALO >> 2) & 1)) owned &= lz >= 1 && lz <= MH;
    int code = 128;
    if (live) {
      double pv[3];
      int ov[3];
      int k = 0;
      if (AXM & 1) {  // along x from the even-plane ring
        const int off = ly * m_ext(CLS ^ 1, 2) + lz;
        pv[k] = apply_stencil(clsx, xs[0][off], xs[1][off], xs[2][off], xs[3][off]);
        ov[k] = stencil_order(clsx);
        k++;
      }
      if (AXM & 2) {  // along y within the plane
        constexpr int cn = CLS ^ 2;
        const double* b = sm + m_base(cn, P0) + ly * m_ext(cn, 2) + lz;
        constexpr int st = m_ext(cn, 2);
        const int cls = INT ? (LINEAR ? ST_MID : ST_CUBIC) : classify((int)P1b + 2 * iy, c.D1, 1, LINEAR);
        pv[k] = apply_stencil(cls, b[0], b[st], b[2 * st], b[3 * st]);
        ov[k] = stencil_order(cls);
        k++;
      }
      if (AXM & 4) {  // along z within the plane
        constexpr int cn = CLS ^ 4;
        const double* b = sm + m_base(cn, P0) + ly * m_ext(cn, 2) + lz;
        const int cls = INT ? (LINEAR ? ST_MID : ST_CUBIC) : classify((int)P2b + 2 * iz, c.D2, 1, LINEAR);
        pv[k] = apply_stencil(cls, b[0], b[1], b[2], b[3]);
        ov[k] = stencil_order(cls);
        k++;
      }
      const double pred = k == 1 ? pv[0] : combine_axes(k, pv, ov);
      double r;
      if (!DEC) {
        const double o = (double)stf[idx];
        code = quantize_fast<sizeof(T) == 4>(o, pred, c.eb, c.two_eb, c.inv_two_eb, &r);
        if (owned) {
          A.seq[sl0 + iy * ksy + iz * ksz] = (uint8_t)code;
          const int lin = lin0 + iy * kly + iz * klz;
          if (code == 0) atomicOr(&A.obm[lin >> 5], 1u << (lin & 31));
          bad |= !isfinite(o);
          if (g.level >= 2) A.E[E0 + iy * key + iz * kez] = r;
        }
      } else {
        const int sl = sl0 + iy * ksy + iz * ksz;
        code = (stc[idx] >> (8 * (reinterpret_cast<uintptr_t>(A.seq + sl) & 3))) & 0xFF;
        if (code != 0) {
          r = dequantize(pred, c.two_eb, code);
        } else {
          const unsigned long long lin = (unsigned long long)(unsigned)(lin0 + iy * kly + iz * klz);
          unsigned long long a0 = 0, a1 = c.ocount;
          while (a0 < a1) {
            const unsigned long long mid = (a0 + a1) >> 1;
            if (A.oidx[mid] < lin)
              a0 = mid + 1;
            else
              a1 = mid;
          }
          if (a0 < c.ocount && A.oidx[a0] == lin) {
            r = A.oval[a0];
          } else {
            r = 0.0;
            bad = true;
          }
        }
        if (owned) {
          if (g.level >= 2) {
            A.E[E0 + iy * key + iz * kez] = r;
          } else {
            reinterpret_cast<T*>(A.out)[lin0 + iy * kly + iz * klz] = (T)r;
            nf |= !isfinite(r);
          }
        }
      }
      if (base_c >= 0) sm[base_c + ly * ex_z + lz] = r;
    }
    if (!DEC) {
      const bool cnt = live && owned;
      const unsigned m128 = __ballot_sync(0xffffffffu, cnt && code == 128);
      if (lane == 0 && m128) atomicAdd(&shist[128], (unsigned)__popc(m128));
      if (cnt && code != 128) atomicAdd(&shist[code], 1u);
    }
  }
}

// load the lattice (eee) of even plane P0 into its ring slot; level-1 replay
// also writes the owned lattice points to the output
template <bool DEC, typename T>
__device__ __forceinline__ void m_load_eee(const LvArgs& A, const MarchCtx& c, double* sm, int P0, bool& nf) {
  const LevelGeom& g = A.g;
  double* dst = sm + m_base(0, P0);
  const int s = (int)g.s, e1 = (int)g.Ed[1], e2 = (int)g.Ed[2];
  const int hx = P0 >> 1;
  for (int idx = threadIdx.x; idx < ME * ME; idx += M_THREADS) {
    const int ly = idx / ME, lz = idx % ME;
    const int h1 = c.hb1 - 1 + ly, h2 = c.hb2 - 1 + lz;
    const bool ok = h1 >= 0 && 2 * h1 < c.D1 && h2 >= 0 && 2 * h2 < c.D2;
    const double* src = A.E + (ok ? ((hx * s) * e1 + h1 * s) * e2 + h2 * s : 0);
    cp_async<8>(dst + idx, src, ok);
  }
  cp_async_wait_all();
  if (DEC && g.level == 1 && P0 >= c.X0 && P0 < c.X1) {
    for (int idx = threadIdx.x; idx < ME * ME; idx += M_THREADS) {
      const int ly = idx / ME, lz = idx % ME;
      const int h1 = c.hb1 - 1 + ly, h2 = c.hb2 - 1 + lz;
      if (ly >= 1 && ly <= MH && lz >= 1 && lz <= MH && 2 * h1 < c.D1 && 2 * h2 < c.D2) {
        const double v = dst[idx];
        reinterpret_cast<T*>(A.out)[((long long)P0 * g.d[1] + 2ll * h1) * g.d[2] + 2ll * h2] = (T)v;
        nf |= !isfinite(v);
      }
    }
  }
}

// phase helper: issue the loads of up to four classes, wait, compute them
#define M_CLASS(CLS, AXM, HALO, SID) CLS, AXM, HALO, SID
template <int C0, int A0, int H0, int C1, int A1, int H1, int NC, bool LINEAR, bool DEC, typename T, bool INT>
__device__ __forceinline__ void m_phase2(const LvArgs& A, const MarchCtx& c, double* sm, unsigned* sh, int P0,
                                         bool& bad, bool& nf) {
  m_issue<C0, A0, H0, 0, LINEAR, DEC, T, INT>(A, c, sm, P0);
  if (NC > 1) m_issue<C1, A1, H1, 1, LINEAR, DEC, T, INT>(A, c, sm, P0);
  cp_async_wait_all();
  m_compute<C0, A0, H0, 0, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
  if (NC > 1) m_compute<C1, A1, H1, 1, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
  __syncthreads();
}

// multidim (predictor.py:282-296): every even axis carries the halo
template <bool LINEAR, bool DEC, typename T, bool INT>
__device__ __forceinline__ void m_even_multidim(const LvArgs& A, const MarchCtx& c, double* sm, unsigned* sh, int P0,
                                                bool& bad, bool& nf) {
  m_phase2<2, 2, 4, 4, 4, 2, 2, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);  // {y}, {z}
  m_phase2<6, 6, 0, 6, 6, 0, 1, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);  // {yz}
}
template <bool LINEAR, bool DEC, typename T, bool INT>
__device__ __forceinline__ void m_odd_multidim(const LvArgs& A, const MarchCtx& c, double* sm, unsigned* sh, int P0,
                                               bool& bad, bool& nf) {
  m_phase2<1, 1, 6, 1, 1, 6, 1, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);  // {x}
  m_phase2<3, 3, 4, 5, 5, 2, 2, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);  // {xy}, {xz}
  m_phase2<7, 7, 0, 7, 7, 0, 1, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);  // {xyz}
}

// seq1d with axis order (O0, O1, O2) (predictor.py:267-280): a class
// interpolates along its last odd axis in the order; halo on the even y/z
// axes that come later in the order
template <int O0, int O1, int O2>
struct SeqOrder {
  static constexpr __host__ __device__ int pos(int a) { return a == O0 ? 0 : (a == O1 ? 1 : 2); }
  static constexpr __host__ __device__ int pass(int cls) {
    int p = -1;
    for (int a = 0; a < 3; a++)
      if (((cls >> a) & 1) && pos(a) > p) p = pos(a);
    return p;
  }
  static constexpr __host__ __device__ int axis(int cls) {
    int best = 0, p = -1;
    for (int a = 0; a < 3; a++)
      if (((cls >> a) & 1) && pos(a) > p) p = pos(a), best = a;
    return best;
  }
  static constexpr __host__ __device__ int halo(int cls) {
    int h = 0;
    for (int a = 1; a < 3; a++)
      if (!((cls >> a) & 1) && pos(a) > pass(cls)) h |= 1 << a;
    return h;
  }
};

template <int CLS, class SO, bool LINEAR, bool DEC, typename T, bool INT>
__device__ __forceinline__ void m_seq_class(const LvArgs& A, const MarchCtx& c, double* sm, unsigned* sh, int P0,
                                            bool& bad, bool& nf) {
  constexpr int ax = SO::axis(CLS);
  m_phase2<CLS, (1 << ax), SO::halo(CLS), CLS, (1 << ax), SO::halo(CLS), 1, LINEAR, DEC, T, INT>(A, c, sm, sh, P0,
                                                                                                   bad, nf);
}

// classes of a plane in pass order (one phase per class keeps it simple)
template <int O0, int O1, int O2, bool LINEAR, bool DEC, typename T, bool INT>
__device__ __forceinline__ void m_even_seq(const LvArgs& A, const MarchCtx& c, double* sm, unsigned* sh, int P0,
                                           bool& bad, bool& nf) {
  using SO = SeqOrder<O0, O1, O2>;
  // even-plane classes {y}=2, {z}=4, {yz}=6 ordered by pass
  constexpr int py = SO::pass(2), pz = SO::pass(4);
  if (py <= pz) {
    m_seq_class<2, SO, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
    m_seq_class<4, SO, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
  } else {
    m_seq_class<4, SO, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
    m_seq_class<2, SO, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
  }
  m_seq_class<6, SO, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
}
template <int O0, int O1, int O2, bool LINEAR, bool DEC, typename T, bool INT>
__device__ __forceinline__ void m_odd_seq(const LvArgs& A, const MarchCtx& c, double* sm, unsigned* sh, int P0,
                                          bool& bad, bool& nf) {
  using SO = SeqOrder<O0, O1, O2>;
  // odd-plane classes {x}=1, {xy}=3, {xz}=5, {xyz}=7 in non-decreasing pass order
  constexpr int p1 = SO::pass(1), p3 = SO::pass(3), p5 = SO::pass(5);
  m_seq_class<1, SO, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
  if (p3 <= p5) {
    m_seq_class<3, SO, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
    m_seq_class<5, SO, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
  } else {
    m_seq_class<5, SO, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
    m_seq_class<3, SO, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
  }
  m_seq_class<7, SO, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
  (void)p1;
}

template <int SCH, bool LINEAR, bool DEC, typename T, bool INT>
__device__ __forceinline__ void m_plane(bool odd, const LvArgs& A, const MarchCtx& c, double* sm, unsigned* sh,
                                        int P0, bool& bad, bool& nf) {
  // SCH 0: multidim; 1..6: seq1d with axis order id SCH-1 (see order_id)
  constexpr int O0 = SCH <= 2 ? 0 : (SCH <= 4 ? 1 : 2);
  constexpr int O1 = SCH == 1 ? 1 : (SCH == 2 ? 2 : (SCH == 3 ? 0 : (SCH == 4 ? 2 : (SCH == 5 ? 0 : 1))));
  constexpr int O2 = 3 - O0 - O1;
  if (SCH == 0) {
    if (odd)
      m_odd_multidim<LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
    else
      m_even_multidim<LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
  } else {
    if (odd)
      m_odd_seq<O0, O1, O2, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
    else
      m_even_seq<O0, O1, O2, LINEAR, DEC, T, INT>(A, c, sm, sh, P0, bad, nf);
  }
}

template <int SCH, bool LINEAR, bool DEC, typename T>
__device__ __forceinline__ void m_do_plane(bool interior, const LvArgs& A, const MarchCtx& c, double* sm,
                                           unsigned* sh, int P0, bool& bad, bool& nf) {
  const bool odd = P0 & 1;
  if (!odd) m_load_eee<DEC, T>(A, c, sm, P0, nf);
  __syncthreads();
  if (interior)
    m_plane<SCH, LINEAR, DEC, T, true>(odd, A, c, sm, sh, P0, bad, nf);
  else
    m_plane<SCH, LINEAR, DEC, T, false>(odd, A, c, sm, sh, P0, bad, nf);
}

// One instantiation per (dtype, direction, spline, scheme): the host knows
// the level's interpolation config (read back after the tuner / from the
// archive header), so each kernel stays small.
template <typename T, bool DEC, bool LINEAR, int SCH>
__global__ void __launch_bounds__(M_THREADS, 3) k_level_march(LvArgs A, int segp, int ncz, int ncy) {
  extern __shared__ double sm[];
  __shared__ unsigned shist[256];
  const LevelGeom& g = A.g;
  const int col = blockIdx.x % (ncy * ncz), seg = blockIdx.x / (ncy * ncz);
  const int ty = col / ncz, tz = col % ncz;
  MarchCtx c;
  c.hb1 = ty * MH;
  c.hb2 = tz * MH;
  c.D0 = (int)g.D[0], c.D1 = (int)g.D[1], c.D2 = (int)g.D[2];
  c.X0 = seg * segp;
  c.X1 = min(c.X0 + segp, c.D0);
  c.eb = A.st->eb;
  c.two_eb = A.st->two_eb;
  c.inv_two_eb = __ddiv_rn(1.0, c.two_eb);
  c.ocount = DEC ? *A.ocount : 0;
  if (!DEC)
    for (int i = threadIdx.x; i < 256; i += M_THREADS) shist[i] = 0;
  const bool interior = c.hb1 * 2 >= 2 && c.hb1 * 2 + MT + 3 <= c.D1 && c.hb2 * 2 >= 2 && c.hb2 * 2 + MT + 3 <= c.D2;
  bool bad = false, nf = false;
  // prologue: even planes X0-2, X0, X0+2; then even plane 2m+4 followed by odd plane 2m+1
  const int mlo = c.X0 >> 1;
  for (int m = mlo - 1; m <= mlo + 1; m++)
    if (m >= 0 && 2 * m < c.D0) m_do_plane<SCH, LINEAR, DEC, T>(interior, A, c, sm, shist, 2 * m, bad, nf);
  for (int m = mlo; 2 * m + 1 < c.X1; m++) {
    if (2 * (m + 2) < c.D0) m_do_plane<SCH, LINEAR, DEC, T>(interior, A, c, sm, shist, 2 * (m + 2), bad, nf);
    m_do_plane<SCH, LINEAR, DEC, T>(interior, A, c, sm, shist, 2 * m + 1, bad, nf);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) raise_flag(A.st, DEC ? F_ORPHAN : F_NONFINITE);
  if (DEC && __any_sync(0xffffffffu, nf) && (threadIdx.x & 31) == 0) raise_flag(A.st, F_NONFINITE);
  if (!DEC) {
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += M_THREADS)
      if (shist[i]) atomicAdd(&A.st->hist[i], (unsigned long long)shist[i]);
  }
}

template <typename T, bool DEC, bool LINEAR, int SCH>
inline void march_launch_one(const LvArgs& A, const MarchLaunch& L, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_level_march<T, DEC, LINEAR, SCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
    cudaFuncSetAttribute(k_level_march<T, DEC, LINEAR, SCH>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = true;
  }
  k_level_march<T, DEC, LINEAR, SCH><<<L.blocks, M_THREADS, L.smem, s>>>(A, L.segp, L.ncz, L.ncy);
}

template <typename T, bool DEC>
inline void march_launch_T(const LvArgs& A, const MarchLaunch& L, int cfg, int oid, cudaStream_t s) {
  const int sch = (cfg & 2) ? 1 + oid : 0;
  const bool lin = cfg & 1;
#define HB_MC(SCHV)                                       \
  case SCHV:                                              \
    if (lin)                                              \
      march_launch_one<T, DEC, true, SCHV>(A, L, s);      \
    else                                                  \
      march_launch_one<T, DEC, false, SCHV>(A, L, s);     \
    break;
  switch (sch) {
    HB_MC(0) HB_MC(1) HB_MC(2) HB_MC(3) HB_MC(4) HB_MC(5) HB_MC(6)
  }
#undef HB_MC
}

}  // namespace hb
