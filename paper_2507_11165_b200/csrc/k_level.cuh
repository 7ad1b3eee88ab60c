// k_level.cuh -- specialised level kernels (compress + decompress) for 2D
// fields (64x64x1 tiles, d2 == 1); 3D fields use the column kernel k_col.cuh,
// which shares TileShape, LvArgs, CtaCtx and cp_async from this header.
//
// Same algorithm as the generic kernel in k_predict.cu (one CTA per lattice
// tile, one shared-memory f64 array per parity class, halo recompute, phases
// separated by __syncthreads), but every class, its interpolation axes, halo
// axes, storage extents/offsets and the Eq. 3 sequence-slot formula are
// compile-time constants, so the inner loop is pure address arithmetic, f64
// stencil math and the quantizer.  Reference: predictor.py:181-304 (+ :313-329
// quantize, :397-411 replay), ordering.py:68-84 (slot of each code).
#pragma once
#include <cuda_runtime.h>

#include "hb_common.cuh"
#include "hb_interp.cuh"
#include "hb_kernels.h"

namespace hb {

constexpr int LV_THREADS = 256;

// cp.async (LDGSTS) global -> shared copies: the loads of a phase are all in
// flight at once without holding registers; src-size 0 zero-fills.
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? BYTES : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(sa), "l"(gmem), "n"(BYTES), "r"(sz));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <int T0, int T1, int T2>
struct TileShape {
  static constexpr __host__ __device__ int t(int a) { return a == 0 ? T0 : (a == 1 ? T1 : T2); }
  static constexpr __host__ __device__ bool big(int a) { return t(a) > 1; }
  static constexpr __host__ __device__ int ne(int a) { return big(a) ? t(a) / 2 : 1; }  // owned even positions
  static constexpr __host__ __device__ int no(int a) { return big(a) ? t(a) / 2 : 0; }  // odd positions
  static constexpr __host__ __device__ int E(int a) { return big(a) ? t(a) / 2 + 3 : 1; }  // even incl. halo
  static constexpr __host__ __device__ int eoff(int a) { return big(a) ? 1 : 0; }
  static constexpr __host__ __device__ int ext(int c, int a) { return ((c >> a) & 1) ? no(a) : E(a); }
  static constexpr __host__ __device__ int size(int c) { return ext(c, 0) * ext(c, 1) * ext(c, 2); }
  static constexpr __host__ __device__ int off(int c) {
    int o = 0;
    for (int k = 0; k < c; k++) o += size(k);
    return o;
  }
  static constexpr __host__ __device__ int total() { return off(7); }  // classes 0..6 (7 is never re-read)
  static constexpr __host__ __device__ int stage_doubles() {
    int m = 0;
    for (int k = 1; k < 8; k++) m = size(k) > m ? size(k) : m;
    return m;
  }
  static constexpr __host__ __device__ size_t smem_bytes() { return (size_t)(total() + stage_doubles()) * 8; }
};

struct LvArgs {
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
};

struct CtaCtx {
  int hb0[3];  // half-index of the tile origin
  int D[3];
  long long d1, d2, e1, e2, s;
  double eb, two_eb, inv_two_eb;
  unsigned long long ocount;
  bool wE, out0;  // level >= 2 (writes the E lattice) / level 1 (writes the output)
};

// Eq. 3 slot of a point of class C (bit a = coordinate odd on axis a)
template <int C>
__device__ __forceinline__ long long slot(const LevelGeom& g, long long P0, long long P1, long long P2) {
  const long long D1 = g.D[1], D2 = g.D[2];
  const long long ey = (D1 + 1) >> 1, ez = (D2 + 1) >> 1;
  long long r = g.prefix + (P0 * D1 + P1) * D2 + P2 - ((P0 + 1) >> 1) * ey * ez;
  if (!(C & 1)) {
    r -= ((P1 + 1) >> 1) * ez;
    if (!(C & 2)) r -= (P2 + 1) >> 1;
  }
  return r;
}

// One class: CLS = parity mask, AXM = interpolation axes, HALO = even axes
// computed over the halo (others over the owned tile positions only).
// All per-point addresses (field, Eq. 3 slot, E, shared memory) are affine
// in the local index, so they are evaluated as base + i*stride; the global
// loads of a thread's points are issued up front (one batch per class) so
// their latency overlaps.
template <class TL, int CLS, int AXM, int HALO, bool LINEAR, bool DEC, typename T, bool INT>
__device__ __forceinline__ void process_class(const LvArgs& A, const CtaCtx& c, double* sm, unsigned* shist,
                                              bool& bad, bool& nf) {
  double* stage = sm + TL::total();  // per-class load staging (after the class arrays)
  constexpr bool odd0 = (CLS >> 0) & 1, odd1 = (CLS >> 1) & 1, odd2 = (CLS >> 2) & 1;
  constexpr int n0 = odd0 ? TL::no(0) : (((HALO >> 0) & 1) ? TL::E(0) : TL::ne(0));
  constexpr int n1 = odd1 ? TL::no(1) : (((HALO >> 1) & 1) ? TL::E(1) : TL::ne(1));
  constexpr int n2 = odd2 ? TL::no(2) : (((HALO >> 2) & 1) ? TL::E(2) : TL::ne(2));
  constexpr int lo0 = odd0 || ((HALO >> 0) & 1) ? 0 : TL::eoff(0);
  constexpr int lo1 = odd1 || ((HALO >> 1) & 1) ? 0 : TL::eoff(1);
  constexpr int lo2 = odd2 || ((HALO >> 2) & 1) ? 0 : TL::eoff(2);
  constexpr int total = n0 * n1 * n2;
  if constexpr (total == 0) {
    return;
  } else {
    constexpr int ITERS = (total + LV_THREADS - 1) / LV_THREADS;
    constexpr int cx1 = TL::ext(CLS, 1), cx2 = TL::ext(CLS, 2);
    constexpr bool stored = CLS != 7 && TL::size(CLS) > 0;
    const int lane = threadIdx.x & 31;
    // half-index of local index 0 per axis, P = 2*x + odd with x = xb + i
    const int xb0 = c.hb0[0] - (odd0 ? 0 : TL::eoff(0)) + lo0;
    const int xb1 = c.hb0[1] - (odd1 ? 0 : TL::eoff(1)) + lo1;
    const int xb2 = c.hb0[2] - (odd2 ? 0 : TL::eoff(2)) + lo2;
    // valid i range per axis: 0 <= P < D  <=>  0 <= x < (D - odd + 1) >> 1
    const int ilo0 = -xb0, ihi0 = ((c.D[0] - odd0 + 1) >> 1) - xb0;
    const int ilo1 = -xb1, ihi1 = ((c.D[1] - odd1 + 1) >> 1) - xb1;
    const int ilo2 = -xb2, ihi2 = ((c.D[2] - odd2 + 1) >> 1) - xb2;
    // affine maps at i = 0 (P may be negative there; the maps stay linear)
    const LevelGeom& g = A.g;  // kernel-parameter constants
    // (the tiled kernels only run when every element index fits in int32,
    // so all per-point address arithmetic below is 32-bit)
    const long long P00 = 2ll * xb0 + odd0, P10 = 2ll * xb1 + odd1, P20 = 2ll * xb2 + odd2;
    const int lin0 = (int)(((P00 * g.s) * g.d[1] + P10 * g.s) * g.d[2] + P20 * g.s);
    const int kl0 = (int)g.kl[0], kl1 = (int)g.kl[1], kl2 = (int)g.kl[2];
    long long sl0l = g.prefix + (P00 * g.D[1] + P10) * g.D[2] + P20 - ((P00 + 1) >> 1) * g.eyez;
    if (!odd0) {
      sl0l -= ((P10 + 1) >> 1) * g.ez;
      if (!odd1) sl0l -= (P20 + 1) >> 1;
    }
    const int sl0 = (int)sl0l;
    const int ks0 = (int)g.ks0;
    const int ks1 = (int)(odd0 ? g.ks1_odd0 : g.ks1_even0);
    constexpr int ks2 = (odd0 || odd1) ? 2 : 1;
    const int ke0 = (int)g.ke[0], ke1 = (int)g.ke[1], ke2 = (int)g.ke[2];
    const int E0 = (int)((((P00 * g.s) >> 1) * g.Ed[1] + ((P10 * g.s) >> 1)) * g.Ed[2] + ((P20 * g.s) >> 1));
    // ---- phase A: issue all of this thread's global loads (independent, so
    // their latency overlaps) into a per-thread slot of the staging area
    T* stf = reinterpret_cast<T*>(stage);
    uint32_t* stc = reinterpret_cast<uint32_t*>(stage);  // aligned word holding the code byte
#pragma unroll
    for (int it = 0; it < ITERS; it++) {
      const int idx = it * LV_THREADS + threadIdx.x;
      const int i2 = idx % n2, i1 = (idx / n2) % n1, i0 = idx / (n2 * n1);
      const bool live = INT ? idx < total
                            : idx < total && i0 >= ilo0 && i0 < ihi0 && i1 >= ilo1 && i1 < ihi1 && i2 >= ilo2 && i2 < ihi2;
      if (idx < total) {
        if (!DEC) {
          const T* src = reinterpret_cast<const T*>(A.field) + (live ? lin0 + i0 * kl0 + i1 * kl1 + i2 * kl2 : 0);
          cp_async<sizeof(T)>(stf + idx, src, live);
        } else {
          const int sl = live ? sl0 + i0 * ks0 + i1 * ks1 + i2 * ks2 : 0;
          const uintptr_t ad = reinterpret_cast<uintptr_t>(A.seq + sl) & ~uintptr_t(3);
          cp_async<4>(stc + idx, reinterpret_cast<const void*>(ad), live);
        }
      }
    }
    cp_async_wait_all();
    // ---- phase B: predict, quantize / replay, write
#pragma unroll 1
    for (int it = 0; it < ITERS; it++) {
      const int idx = it * LV_THREADS + threadIdx.x;
      const int i2 = idx % n2, i1 = (idx / n2) % n1, i0 = idx / (n2 * n1);
      const bool live = INT ? idx < total
                            : idx < total && i0 >= ilo0 && i0 < ihi0 && i1 >= ilo1 && i1 < ihi1 && i2 >= ilo2 && i2 < ihi2;
      const int l[3] = {lo0 + i0, lo1 + i1, lo2 + i2};
      bool owned = true;
#pragma unroll
      for (int a = 0; a < 3; a++)
        if (!((CLS >> a) & 1) && ((HALO >> a) & 1)) owned &= l[a] >= TL::eoff(a) && l[a] < TL::eoff(a) + TL::ne(a);
      int code = 128;
      if (live) {
        // prediction (predictor.py:209-256)
        double pv[3];
        int ov[3];
        int k = 0;
#pragma unroll
        for (int a = 0; a < 3; a++) {
          if (!((AXM >> a) & 1)) continue;
          const int cn = CLS & ~(1 << a);
          const int s1 = TL::ext(cn, 2), s0 = TL::ext(cn, 1) * TL::ext(cn, 2);
          const int step = a == 0 ? s0 : (a == 1 ? s1 : 1);
          const double* b = sm + TL::off(cn) + l[0] * s0 + l[1] * s1 + l[2];
          const int Pa = a == 0 ? (int)P00 + 2 * i0 : (a == 1 ? (int)P10 + 2 * i1 : (int)P20 + 2 * i2);
          // interior tiles: every stencil is the full one (cubic / linear mid-point)
          const int cls = INT ? (LINEAR ? ST_MID : ST_CUBIC) : classify(Pa, c.D[a], 1, LINEAR);
          pv[k] = cls == ST_CUBIC ? apply_stencil(ST_CUBIC, b[0], b[step], b[2 * step], b[3 * step])
                                  : apply_stencil(cls, b[0], b[step], b[2 * step], b[3 * step]);
          ov[k] = stencil_order(cls);
          k++;
        }
        const double pred = k == 1 ? pv[0] : combine_axes(k, pv, ov);
        double r;
        if (!DEC) {
          const double o = (double)stf[idx];
          code = quantize_fast<sizeof(T) == 4>(o, pred, c.eb, c.two_eb, c.inv_two_eb, &r);
          if (owned) {
            A.seq[sl0 + i0 * ks0 + i1 * ks1 + i2 * ks2] = (uint8_t)code;
            const int lin = lin0 + i0 * kl0 + i1 * kl1 + i2 * kl2;
            if (code == 0) atomicOr(&A.obm[lin >> 5], 1u << (lin & 31));
            bad |= !isfinite(o);
            if (A.g.level >= 2) A.E[E0 + i0 * ke0 + i1 * ke1 + i2 * ke2] = r;
          }
        } else {
          code = (stc[idx] >> (8 * (reinterpret_cast<uintptr_t>(A.seq + (sl0 + i0 * ks0 + i1 * ks1 + i2 * ks2)) & 3))) &
                 0xFF;
          if (code != 0) {
            r = dequantize(pred, c.two_eb, code);
          } else {
            const unsigned long long lin = (unsigned long long)(unsigned)(lin0 + i0 * kl0 + i1 * kl1 + i2 * kl2);
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
            if (A.g.level >= 2) {
              A.E[E0 + i0 * ke0 + i1 * ke1 + i2 * ke2] = r;
            } else {
              reinterpret_cast<T*>(A.out)[lin0 + i0 * kl0 + i1 * kl1 + i2 * kl2] = (T)r;
              nf |= !isfinite(r);
            }
          }
        }
        if (stored) sm[TL::off(CLS) + (l[0] * cx1 + l[1]) * cx2 + l[2]] = r;
      }
      if (!DEC) {  // code histogram (Huffman input), warp-aggregated for the dominant code
        const bool cnt = live && owned;
        const unsigned m128 = __ballot_sync(0xffffffffu, cnt && code == 128);
        if (lane == 0 && m128) atomicAdd(&shist[128], (unsigned)__popc(m128));
        if (cnt && code != 128) atomicAdd(&shist[code], 1u);
      }
    }
  }
}

// multidim (predictor.py:282-296): phases by number of odd axes, every even
// axis carries the halo, a class interpolates along all its odd axes
template <class TL, bool LINEAR, bool DEC, typename T, bool INT>
__device__ __forceinline__ void run_multidim(const LvArgs& A, const CtaCtx& c, double* sm, unsigned* sh, bool& bad, bool& nf) {
  process_class<TL, 1, 1, 6, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
  process_class<TL, 2, 2, 5, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
  process_class<TL, 4, 4, 3, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
  __syncthreads();
  process_class<TL, 3, 3, 4, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
  process_class<TL, 5, 5, 2, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
  process_class<TL, 6, 6, 1, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
  __syncthreads();
  process_class<TL, 7, 7, 0, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
}

// seq1d (predictor.py:267-280) with axis order (O0, O1, O2): pass k predicts
// points odd on Ok along Ok only; halo on the axes of later passes
template <class TL, int O0, int O1, int O2, bool LINEAR, bool DEC, typename T, bool INT>
__device__ __forceinline__ void run_seq1d(const LvArgs& A, const CtaCtx& c, double* sm, unsigned* sh, bool& bad, bool& nf) {
  constexpr int b0 = 1 << O0, b1 = 1 << O1, b2 = 1 << O2;
  process_class<TL, b0, b0, b1 | b2, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
  __syncthreads();
  process_class<TL, b1, b1, b2, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
  process_class<TL, b0 | b1, b1, b2, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
  __syncthreads();
  process_class<TL, b2, b2, 0, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
  process_class<TL, b0 | b2, b2, 0, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
  process_class<TL, b1 | b2, b2, 0, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
  process_class<TL, 7, b2, 0, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
}

template <class TL, bool LINEAR, bool DEC, typename T, bool INT>
__device__ __forceinline__ void run_seq1d_any(int order_id, const LvArgs& A, const CtaCtx& c, double* sm, unsigned* sh, bool& bad, bool& nf) {
  if (TL::big(2)) {
    switch (order_id) {
      case 0: run_seq1d<TL, 0, 1, 2, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf); break;
      case 1: run_seq1d<TL, 0, 2, 1, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf); break;
      case 2: run_seq1d<TL, 1, 0, 2, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf); break;
      case 3: run_seq1d<TL, 1, 2, 0, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf); break;
      case 4: run_seq1d<TL, 2, 0, 1, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf); break;
      default: run_seq1d<TL, 2, 1, 0, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf); break;
    }
  } else {  // d2 == 1 sorts last
    if (order_id == 2)
      run_seq1d<TL, 1, 0, 2, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
    else
      run_seq1d<TL, 0, 1, 2, LINEAR, DEC, T, INT>(A, c, sm, sh, bad, nf);
  }
}

template <class TL, typename T, bool DEC>
__global__ void __launch_bounds__(LV_THREADS, 3) k_level_tiled(LvArgs A, int order_id) {
  extern __shared__ double sm[];
  __shared__ unsigned shist[256];
  const LevelGeom& g = A.g;
  const int nt2 = g.ntile[2], nt1 = g.ntile[1];
  const int tix[3] = {(int)(blockIdx.x / (nt2 * nt1)), (int)((blockIdx.x / nt2) % nt1), (int)(blockIdx.x % nt2)};
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
  if (!DEC)
    for (int i = threadIdx.x; i < 256; i += LV_THREADS) shist[i] = 0;
  bool nf0 = false;
  // the known 2s-lattice (class 0) with halo, from E (cp.async, zero-filled outside)
  {
    constexpr int e0 = TL::E(0), e1 = TL::E(1), e2 = TL::E(2);
    constexpr int cnt = e0 * e1 * e2;
    for (int idx = threadIdx.x; idx < cnt; idx += LV_THREADS) {
      const int l2 = idx % e2, l1 = (idx / e2) % e1, l0 = idx / (e2 * e1);
      const int h0 = c.hb0[0] - TL::eoff(0) + l0, h1 = c.hb0[1] - TL::eoff(1) + l1, h2 = c.hb0[2] - TL::eoff(2) + l2;
      const bool ok = h0 >= 0 && 2 * h0 < c.D[0] && h1 >= 0 && 2 * h1 < c.D[1] && h2 >= 0 && 2 * h2 < c.D[2];
      const double* src = A.E + (ok ? ((h0 * (int)c.s) * (int)c.e1 + h1 * (int)c.s) * (int)c.e2 + h2 * (int)c.s : 0);
      cp_async<8>(sm + idx, src, ok);
    }
    cp_async_wait_all();
    if (DEC && g.level == 1) {
      for (int idx = threadIdx.x; idx < cnt; idx += LV_THREADS) {
        const int l2 = idx % e2, l1 = (idx / e2) % e1, l0 = idx / (e2 * e1);
        const int h0 = c.hb0[0] - TL::eoff(0) + l0, h1 = c.hb0[1] - TL::eoff(1) + l1,
                  h2 = c.hb0[2] - TL::eoff(2) + l2;
        const bool owned = l0 >= TL::eoff(0) && l0 < TL::eoff(0) + TL::ne(0) && l1 >= TL::eoff(1) &&
                           l1 < TL::eoff(1) + TL::ne(1) && l2 >= TL::eoff(2) && l2 < TL::eoff(2) + TL::ne(2) &&
                           2 * h0 < c.D[0] && 2 * h1 < c.D[1] && 2 * h2 < c.D[2];
        if (owned) {
          const double v = sm[idx];
          reinterpret_cast<T*>(A.out)[((2ll * h0) * c.d1 + 2ll * h1) * c.d2 + 2ll * h2] = (T)v;
          nf0 |= !isfinite(v);
        }
      }
    }
  }
  __syncthreads();
  const int cfg = A.st->cfg[g.level - 1] & 3;
  // interior tile: all computed points (tile + halo) exist and every stencil is complete
  bool interior = true;
  for (int a = 0; a < 3; a++)
    if (TL::big(a)) {
      const int P0 = tix[a] * TL::t(a);
      interior &= P0 >= 2 && P0 + TL::t(a) + 3 <= c.D[a];
    }
  bool bad = false, nf = nf0;
  switch (cfg) {
    case 0:
      if (interior) run_multidim<TL, false, DEC, T, true>(A, c, sm, shist, bad, nf);
      else run_multidim<TL, false, DEC, T, false>(A, c, sm, shist, bad, nf);
      break;
    case 1:
      if (interior) run_multidim<TL, true, DEC, T, true>(A, c, sm, shist, bad, nf);
      else run_multidim<TL, true, DEC, T, false>(A, c, sm, shist, bad, nf);
      break;
    case 2:
      if (interior) run_seq1d_any<TL, false, DEC, T, true>(order_id, A, c, sm, shist, bad, nf);
      else run_seq1d_any<TL, false, DEC, T, false>(order_id, A, c, sm, shist, bad, nf);
      break;
    default:
      if (interior) run_seq1d_any<TL, true, DEC, T, true>(order_id, A, c, sm, shist, bad, nf);
      else run_seq1d_any<TL, true, DEC, T, false>(order_id, A, c, sm, shist, bad, nf);
      break;
  }
  if (DEC && __any_sync(0xffffffffu, nf) && (threadIdx.x & 31) == 0) raise_flag(A.st, F_NONFINITE);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) raise_flag(A.st, DEC ? F_ORPHAN : F_NONFINITE);
  if (!DEC) {
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += LV_THREADS)
      if (shist[i]) atomicAdd(&A.st->hist[i], (unsigned long long)shist[i]);
  }
}

using Tile3 = TileShape<16, 16, 16>;
using Tile2 = TileShape<64, 64, 1>;

static inline int order_id(const LevelGeom& g) {
  const int* o = g.seq_order;
  if (o[0] == 0) return o[1] == 1 ? 0 : 1;
  if (o[0] == 1) return o[1] == 0 ? 2 : 3;
  return o[1] == 0 ? 4 : 5;
}

// returns false if the shape needs the generic kernel
template <bool DEC>
static inline bool launch_tiled(LevelGeom g, const LvArgs& base, int prec, cudaStream_t s) {
  const bool b0 = g.d[0] > 1, b1 = g.d[1] > 1, b2 = g.d[2] > 1;
  LvArgs A = base;
  if (g.d[0] * g.d[1] * g.d[2] >= (1ll << 31) - (1ll << 24)) return false;  // 32-bit indexing only
  (void)b0, (void)b1;
  if (!(b0 && b1 && !b2)) return false;  // 3D shapes use the column kernel (k_col.cuh)
  const int T[3] = {64, 64, 1};
  for (int a = 0; a < 3; a++) {
    g.T[a] = T[a];
    g.ntile[a] = (int)((g.D[a] + T[a] - 1) / T[a]);
  }
  A.g = g;
  const unsigned blocks = (unsigned)((long long)g.ntile[0] * g.ntile[1] * g.ntile[2]);
  const int oid = order_id(g);
  static const bool attr = [&] {  // once per process, thread-safe (C++11 static init)
    auto set = [](const void* f, int bytes) {
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    };
    set((const void*)k_level_tiled<Tile2, float, DEC>, Tile2::smem_bytes());
    set((const void*)k_level_tiled<Tile2, double, DEC>, Tile2::smem_bytes());
    return true;
  }();
  (void)attr;
  {
    const size_t smem = Tile2::smem_bytes();
    if (prec == 4)
      k_level_tiled<Tile2, float, DEC><<<blocks, LV_THREADS, smem, s>>>(A, oid);
    else
      k_level_tiled<Tile2, double, DEC><<<blocks, LV_THREADS, smem, s>>>(A, oid);
  }
  return true;
}

}  // namespace hb
