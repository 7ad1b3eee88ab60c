// k_predict.cu -- value range, anchors, the per-level tile kernels of the
// interpolation predictor/quantizer (compress) and its replay (decompress),
// outlier compaction and the level-grouped reorder.
//
// Reference: predictor.py:114-416, ordering.py:24-179, field.py:129-142.
//
// Design: level L (stride s) is executed as "level 1 on the
// D = ceil(d/s) lattice".  A CTA owns a T^3 tile of that lattice and keeps, in
// shared memory, one f64 array per parity class (bit a of the class mask =
// coordinate odd along axis a) covering the tile plus the +-3 halo each
// class needs.  All sub-steps of the level run inside the CTA with
// __syncthreads between dependent phases; halo points are recomputed (exact,
// because every target depends only on the 2s-lattice inside a +-3 box,
// SURVEY A.7).  Codes are written straight to their Eq. 3 sequence slot
// (reorder fused), the code histogram for the Huffman stage is accumulated
// in shared memory, outliers set a bit in a linear-order bitmap, and levels
// >= 2 store their f64 reconstruction into the even lattice E that the next
// level reads.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "hb_common.cuh"
#include "hb_interp.cuh"
#include "hb_kernels.h"

namespace hb {

// ------------------------------------------------------------ geometry

static int ilog2i(int a) {
  int t = 0;
  while ((1 << (t + 1)) <= a) t++;
  return t;
}

void make_level_geom(const uint64_t dims[3], int level, LevelGeom* g) {
  memset(g, 0, sizeof *g);
  const long long s = 1ll << (level - 1);
  int nbig = 0;
  for (int a = 0; a < 3; a++) {
    g->d[a] = (long long)dims[a];
    g->D[a] = (g->d[a] + s - 1) / s;
    g->Ed[a] = (g->d[a] + 1) / 2;
    nbig += g->D[a] > 1;
  }
  g->s = s;
  g->level = level;
  const int tdef = nbig >= 3 ? 16 : (nbig == 2 ? 64 : 1024);
  for (int a = 0; a < 3; a++) {
    if (g->D[a] == 1) {
      g->T[a] = 1;
    } else {
      long long ev = (g->D[a] + 1) & ~1ll;
      g->T[a] = (int)(ev < tdef ? ev : tdef);
    }
    g->ntile[a] = (int)((g->D[a] + g->T[a] - 1) / g->T[a]);
  }
  // seq1d order: axes sorted by (-d, a) on the global dims (predictor.py:177)
  int o[3] = {0, 1, 2};
  for (int i = 0; i < 3; i++)
    for (int j = i + 1; j < 3; j++)
      if (g->d[o[j]] > g->d[o[i]] || (g->d[o[j]] == g->d[o[i]] && o[j] < o[i])) {
        int t = o[i];
        o[i] = o[j];
        o[j] = t;
      }
  for (int i = 0; i < 3; i++) g->seq_order[i] = o[i];
  // class storage: even axes carry the halo [P0-2, P0+T+2], odd axes the tile
  int total = 0;
  for (int c = 0; c < 8; c++) {
    int sz = 1;
    for (int a = 0; a < 3; a++) {
      const bool big = g->D[a] > 1;
      const int h = big ? g->T[a] / 2 : 1;
      int e = ((c >> a) & 1) ? (big ? g->T[a] / 2 : 0) : (big ? h + 3 : 1);
      g->ext[c][a] = e;
      sz *= e;
    }
    if (c == 7 || sz == 0) {
      g->off[c] = -1;  // the all-odd class is never re-read
    } else {
      g->off[c] = total;
      total += sz;
    }
  }
  g->smem_doubles = total;
  long long pre = 1;
  for (int a = 0; a < 3; a++) pre *= (g->d[a] + (1ll << level) - 1) >> level;
  g->prefix = pre;
  g->kl[0] = 2 * s * g->d[1] * g->d[2];
  g->kl[1] = 2 * s * g->d[2];
  g->kl[2] = 2 * s;
  g->ke[0] = s * g->Ed[1] * g->Ed[2];
  g->ke[1] = s * g->Ed[2];
  g->ke[2] = s;
  const long long ey = (g->D[1] + 1) >> 1, ez = (g->D[2] + 1) >> 1;
  g->eyez = ey * ez;
  g->ez = ez;
  g->ks0 = 2 * g->D[1] * g->D[2] - ey * ez;
  g->ks1_odd0 = 2 * g->D[2];
  g->ks1_even0 = 2 * g->D[2] - ez;
}

// ---------------------------------------------------------- value range

template <typename T>
__global__ void __launch_bounds__(256) k_minmax(const T* __restrict__ v, unsigned long long n, DevState* st) {
  // min / max in the field's own type (exact), widened once at the end; a
  // value is non-finite iff its exponent field is all ones
  T lo = (T)INFINITY, hi = (T)-INFINITY;
  bool bad = false;
  constexpr int V = 32 / sizeof(T);  // elements per thread per step (two 16-byte loads)
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x * V;
  for (unsigned long long i = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) * V; i < n; i += stride) {
    T x[V];
    if (i + V <= n) {
      const uint4* p = reinterpret_cast<const uint4*>(v + i);
      const uint4 a = __ldcs(p), b = __ldcs(p + 1);
      const uint4 ab[2] = {a, b};
#pragma unroll
      for (int h = 0; h < 2; h++)
        memcpy(x + h * (V / 2), &ab[h], 16);
    } else {
      for (int k = 0; k < V; k++) x[k] = i + k < n ? v[i + k] : v[i];
    }
#pragma unroll
    for (int k = 0; k < V; k++) {
      if (sizeof(T) == 4) {
        bad |= (__float_as_uint((float)x[k]) & 0x7f800000u) == 0x7f800000u;
      } else {
        bad |= (((unsigned long long)__double_as_longlong((double)x[k])) & 0x7ff0000000000000ull) ==
               0x7ff0000000000000ull;
      }
      lo = x[k] < lo ? x[k] : lo;
      hi = x[k] > hi ? x[k] : hi;
    }
  }
  double dlo = (double)lo, dhi = (double)hi;
  for (int o = 16; o > 0; o >>= 1) {
    dlo = fmin(dlo, __shfl_xor_sync(0xffffffffu, dlo, o));
    dhi = fmax(dhi, __shfl_xor_sync(0xffffffffu, dhi, o));
  }
  bad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&st->vmin_bits, ord_bits(dlo));
    atomicMax(&st->vmax_bits, ord_bits(dhi));
    if (bad) raise_flag(st, F_NONFINITE);
  }
}

// field.py:135-142: rel eb = mag * float(max - min), the subtraction rounded
// in the field dtype.
template <typename T>
__global__ void k_finish_eb(DevState* st, int eb_mode, double mag) {
  double eb = mag;
  if (eb_mode == 1) {
    const double lo = from_ord_bits(st->vmin_bits), hi = from_ord_bits(st->vmax_bits);
    double rng;
    if (sizeof(T) == 4)
      rng = (double)__fsub_rn((float)hi, (float)lo);
    else
      rng = __dsub_rn(hi, lo);
    if (rng == 0.0) raise_flag(st, F_DEGENERATE, 1);
    eb = __dmul_rn(mag, rng);
  }
  if (!(isfinite(eb) && eb > 0)) raise_flag(st, F_DEGENERATE, 2);
  st->eb = eb;
  st->two_eb = __dmul_rn(2.0, eb);
  st->inv_two_eb = __ddiv_rn(1.0, st->two_eb);
}

__global__ void k_minmax_init(DevState* st) {
  st->vmin_bits = ~0ull;
  st->vmax_bits = 0ull;
}

void launch_minmax(const void* field, int prec, unsigned long long n, DevState* st, int eb_mode, double mag,
                   cudaStream_t s, int* launches) {
  if (eb_mode == 1) {
    k_minmax_init<<<1, 1, 0, s>>>(st);
    (*launches)++;
    unsigned long long blocks = cdiv(n, 256ull * (32 / prec));
    if (blocks > 148ull * 8) blocks = 148ull * 8;
    if (prec == 4)
      k_minmax<float><<<(unsigned)blocks, 256, 0, s>>>((const float*)field, n, st);
    else
      k_minmax<double><<<(unsigned)blocks, 256, 0, s>>>((const double*)field, n, st);
    (*launches)++;
  }
  if (prec == 4)
    k_finish_eb<float><<<1, 1, 0, s>>>(st, eb_mode, mag);
  else
    k_finish_eb<double><<<1, 1, 0, s>>>(st, eb_mode, mag);
  (*launches)++;
}

__global__ void k_set_eb(DevState* st, double eb) {
  if (!(isfinite(eb) && eb > 0)) raise_flag(st, F_DEGENERATE, 2);
  st->eb = eb;
  st->two_eb = __dmul_rn(2.0, eb);
  st->inv_two_eb = __ddiv_rn(1.0, st->two_eb);
}

void launch_set_eb(DevState* st, double eb, cudaStream_t s, int* launches) {
  k_set_eb<<<1, 1, 0, s>>>(st, eb);
  (*launches)++;
}

// ------------------------------------------------------------- anchors

template <typename T>
__global__ void k_anchor_init(const T* __restrict__ f, long long d0, long long d1, long long d2, int A, long long a1,
                              long long a2, unsigned long long na, double* E, long long e1, long long e2,
                              uint8_t* seq, uint8_t* anc_out, DevState* st, int count_hist) {
  unsigned long long j = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  if (j < na) {
    const long long az = j % a2, ay = (j / a2) % a1, ax = j / (a1 * a2);
    const long long x = ax * A, y = ay * A, z = az * A;
    const T v = f[(x * d1 + y) * d2 + z];
    bad = !isfinite((double)v);
    if (E) E[((x >> 1) * e1 + (y >> 1)) * e2 + (z >> 1)] = (double)v;
    seq[j] = 128;
    if (anc_out) {
      const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
#pragma unroll
      for (int k = 0; k < (int)sizeof(T); k++) anc_out[j * sizeof(T) + k] = b[k];
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) raise_flag(st, F_NONFINITE);
  if (count_hist && j == 0) atomicAdd(&st->hist[128], na);
}

void launch_anchor_init(const void* field, int prec, const uint64_t dims[3], int A, double* E, uint8_t* seq,
                        uint8_t* anchors_out, DevState* st, bool count_hist, cudaStream_t s, int* launches) {
  long long a[3], e[3];
  for (int i = 0; i < 3; i++) a[i] = ((long long)dims[i] + A - 1) / A, e[i] = ((long long)dims[i] + 1) / 2;
  unsigned long long na = (unsigned long long)(a[0] * a[1] * a[2]);
  unsigned blocks = (unsigned)cdiv(na, 256);
  if (prec == 4)
    k_anchor_init<float><<<blocks, 256, 0, s>>>((const float*)field, dims[0], dims[1], dims[2], A, a[1], a[2], na,
                                                A > 1 ? E : nullptr, e[1], e[2], seq, anchors_out, st, count_hist);
  else
    k_anchor_init<double><<<blocks, 256, 0, s>>>((const double*)field, dims[0], dims[1], dims[2], A, a[1], a[2], na,
                                                 A > 1 ? E : nullptr, e[1], e[2], seq, anchors_out, st, count_hist);
  (*launches)++;
}

// decompress: anchors (archive bytes, field dtype, unaligned) -> E
template <typename T>
__global__ void k_anchor_load(const uint8_t* __restrict__ anc, long long A, long long a1, long long a2,
                              unsigned long long na, double* E, long long e1, long long e2) {
  unsigned long long j = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= na) return;
  T v;
  uint8_t* b = reinterpret_cast<uint8_t*>(&v);
#pragma unroll
  for (int k = 0; k < (int)sizeof(T); k++) b[k] = anc[j * sizeof(T) + k];
  const long long az = j % a2, ay = (j / a2) % a1, ax = j / (a1 * a2);
  E[(((ax * A) >> 1) * e1 + ((ay * A) >> 1)) * e2 + ((az * A) >> 1)] = (double)v;
}

void launch_anchor_load(const uint8_t* anchors, int prec, const uint64_t dims[3], int A, double* E, cudaStream_t s,
                        int* launches) {
  long long a[3], e[3];
  for (int i = 0; i < 3; i++) a[i] = ((long long)dims[i] + A - 1) / A, e[i] = ((long long)dims[i] + 1) / 2;
  unsigned long long na = (unsigned long long)(a[0] * a[1] * a[2]);
  unsigned blocks = (unsigned)cdiv(na, 256);
  if (prec == 4)
    k_anchor_load<float><<<blocks, 256, 0, s>>>(anchors, A, a[1], a[2], na, E, e[1], e[2]);
  else
    k_anchor_load<double><<<blocks, 256, 0, s>>>(anchors, A, a[1], a[2], na, E, e[1], e[2]);
  (*launches)++;
}

// stride-1 archives (every point an anchor): anchors are the field
template <typename T>
__global__ void k_copy_anchors_out(const uint8_t* __restrict__ anc, unsigned long long n, T* out, DevState* st) {
  unsigned long long j = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  T v;
  uint8_t* b = reinterpret_cast<uint8_t*>(&v);
  for (int k = 0; k < (int)sizeof(T); k++) b[k] = anc[j * sizeof(T) + k];
  out[j] = v;
  if (!isfinite((double)v)) raise_flag(st, F_NONFINITE);
}

void launch_copy_anchors_out(const uint8_t* anchors, int prec, unsigned long long n, void* out, DevState* st,
                             cudaStream_t s, int* launches) {
  unsigned blocks = (unsigned)cdiv(n, 256);
  if (prec == 4)
    k_copy_anchors_out<float><<<blocks, 256, 0, s>>>(anchors, n, (float*)out, st);
  else
    k_copy_anchors_out<double><<<blocks, 256, 0, s>>>(anchors, n, (double*)out, st);
  (*launches)++;
}

// ---------------------------------------------------------- level tiles

// Eq. 3 sequence slot of a target of this level (ordering level L-1), in
// lattice coordinates P (ordering.py:68-84 with X,Y,Z = P).
__device__ __forceinline__ long long seq_index(const LevelGeom& g, long long P0, long long P1, long long P2) {
  const long long D1 = g.D[1], D2 = g.D[2];
  const long long ey = (D1 + 1) >> 1, ez = (D2 + 1) >> 1;
  long long r = g.prefix + (P0 * D1 + P1) * D2 + P2 - ((P0 + 1) >> 1) * ey * ez;
  if (!(P0 & 1)) {
    r -= ((P1 + 1) >> 1) * ez;
    if (!(P1 & 1)) r -= (P2 + 1) >> 1;
  }
  return r;
}

struct TileCtx {
  long long hb0[3];  // half-index of the tile origin (P0/2)
  int eoff[3];       // local index of the first owned even position (1, or 0 on size-1 axes)
  int ne[3];         // owned even positions per axis
};

// phase of a class for the scheme (1..3); 0 = not a target class
template <bool SEQ1D>
__device__ __forceinline__ int class_phase(const LevelGeom& g, int c) {
  if (c == 0) return 0;
  if (!SEQ1D) return __popc(c);
  int p = 0;
  for (int k = 0; k < 3; k++)
    if ((c >> g.seq_order[k]) & 1) p = k + 1;
  return p;
}

// compute-box of class c along axis a: [lo, lo+n) in the class's local index
template <bool SEQ1D>
__device__ __forceinline__ void class_box(const LevelGeom& g, const TileCtx& t, int c, int a, int* lo, int* n) {
  if ((c >> a) & 1) {
    *lo = 0;
    *n = g.ext[c][a];
    return;
  }
  bool halo;
  if (!SEQ1D) {
    halo = true;
  } else {
    int pc = 0, pa = 0;
    for (int k = 0; k < 3; k++) {
      if ((c >> g.seq_order[k]) & 1) pc = k;
      if (g.seq_order[k] == a) pa = k;
    }
    halo = pa > pc;
  }
  if (halo) {
    *lo = 0;
    *n = g.ext[c][a];
  } else {
    *lo = t.eoff[a];
    *n = t.ne[a];
  }
}

template <bool LINEAR, bool SEQ1D>
__device__ __forceinline__ double predict_target(const LevelGeom& g, const double* sm, int c, const int l[3],
                                                 const long long P[3]) {
  double pv[3];
  int ov[3];
  int k = 0;
  int axes[3];
  if (SEQ1D) {
    int ax = 0;
    for (int q = 0; q < 3; q++)
      if ((c >> g.seq_order[q]) & 1) ax = g.seq_order[q];
    axes[0] = ax;
    k = 1;
  } else {
    for (int a = 0; a < 3; a++)
      if ((c >> a) & 1) axes[k++] = a;
  }
  for (int i = 0; i < k; i++) {
    const int a = axes[i];
    const int cn = c & ~(1 << a);
    const int* e = g.ext[cn];
    const int st1 = e[2], st0 = e[1] * e[2];
    const int base = g.off[cn] + l[0] * st0 + l[1] * st1 + l[2];
    const int step = a == 0 ? st0 : (a == 1 ? st1 : 1);
    const int cls = classify(P[a], g.D[a], 1, LINEAR);
    const double v0 = sm[base], v1 = sm[base + step], v2 = sm[base + 2 * step], v3 = sm[base + 3 * step];
    pv[i] = apply_stencil(cls, v0, v1, v2, v3);
    ov[i] = stencil_order(cls);
  }
  if (k == 1) return pv[0];
  return combine_axes(k, pv, ov);
}

template <typename T, bool LINEAR, bool SEQ1D, bool DECOMP>
__device__ void run_tile(const LevelGeom& g, const TileCtx& t, double* sm, unsigned* shist, const T* __restrict__ field,
                         double* __restrict__ E, uint8_t* __restrict__ seq, uint32_t* __restrict__ obm,
                         const uint64_t* __restrict__ oidx, const double* __restrict__ oval, unsigned long long ocount,
                         T* __restrict__ out, double eb, double two_eb, DevState* st, bool* bad) {
  const long long d1 = g.d[1], d2 = g.d[2];
  const long long e1 = g.Ed[1], e2 = g.Ed[2];
  for (int phase = 1; phase <= 3; phase++) {
    for (int c = 1; c < 8; c++) {
      if (class_phase<SEQ1D>(g, c) != phase) continue;
      int lo[3], n[3];
      for (int a = 0; a < 3; a++) class_box<SEQ1D>(g, t, c, a, &lo[a], &n[a]);
      const int cnt = n[0] * n[1] * n[2];
      if (cnt == 0) continue;
      const int* ec = g.ext[c];
      for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) {
        int l[3];
        l[2] = lo[2] + idx % n[2];
        l[1] = lo[1] + (idx / n[2]) % n[1];
        l[0] = lo[0] + idx / (n[2] * n[1]);
        long long P[3];
        bool valid = true, owned = true;
#pragma unroll
        for (int a = 0; a < 3; a++) {
          if ((c >> a) & 1) {
            P[a] = 2 * (t.hb0[a] + l[a]) + 1;
          } else {
            P[a] = 2 * (t.hb0[a] - t.eoff[a] + l[a]);
            owned &= l[a] >= t.eoff[a] && l[a] < t.eoff[a] + t.ne[a];
          }
          valid &= P[a] >= 0 && P[a] < g.D[a];
        }
        if (!valid) continue;
        const double pred = predict_target<LINEAR, SEQ1D>(g, sm, c, l, P);
        const long long x0 = P[0] * g.s, x1 = P[1] * g.s, x2 = P[2] * g.s;
        const long long lin = (x0 * d1 + x1) * d2 + x2;
        double r;
        if (!DECOMP) {
          const double o = (double)field[lin];
          const int code = quantize<sizeof(T) == 4>(o, pred, eb, two_eb, &r);
          if (owned) {
            seq[seq_index(g, P[0], P[1], P[2])] = (uint8_t)code;
            atomicAdd(&shist[code], 1u);
            if (code == 0) atomicOr(&obm[lin >> 5], 1u << (lin & 31));
            *bad |= !isfinite(o);
            if (g.level >= 2) E[((x0 >> 1) * e1 + (x1 >> 1)) * e2 + (x2 >> 1)] = r;
          }
        } else {
          const int code = seq[seq_index(g, P[0], P[1], P[2])];
          if (code != 0) {
            r = dequantize(pred, two_eb, code);
          } else {
            unsigned long long lo2 = 0, hi2 = ocount;
            while (lo2 < hi2) {
              unsigned long long mid = (lo2 + hi2) >> 1;
              if (oidx[mid] < (unsigned long long)lin)
                lo2 = mid + 1;
              else
                hi2 = mid;
            }
            if (lo2 < ocount && oidx[lo2] == (unsigned long long)lin) {
              r = oval[lo2];
            } else {
              r = 0.0;
              *bad = true;
            }
          }
          if (owned) {
            if (g.level >= 2)
              E[((x0 >> 1) * e1 + (x1 >> 1)) * e2 + (x2 >> 1)] = r;
            else
              out[lin] = (T)r;
            if (!isfinite(r)) raise_flag(st, F_NONFINITE);
          }
        }
        if (g.off[c] >= 0) sm[g.off[c] + (l[0] * ec[1] + l[1]) * ec[2] + l[2]] = r;
      }
    }
    __syncthreads();
  }
}

template <typename T, bool DECOMP>
__global__ void __launch_bounds__(256) k_level(LevelGeom g, const T* __restrict__ field, double* __restrict__ E,
                                               uint8_t* __restrict__ seq, uint32_t* __restrict__ obm,
                                               const uint64_t* __restrict__ oidx, const double* __restrict__ oval,
                                               const unsigned long long* __restrict__ ocount_dev,
                                               T* __restrict__ out, DevState* st) {
  extern __shared__ double sm[];
  __shared__ unsigned shist[256];
  const int bx = blockIdx.x % g.ntile[2];
  const int by = (blockIdx.x / g.ntile[2]) % g.ntile[1];
  const int bz = blockIdx.x / (g.ntile[2] * g.ntile[1]);
  const int tix[3] = {bz, by, bx};
  TileCtx t;
  for (int a = 0; a < 3; a++) {
    const long long P0 = (long long)tix[a] * g.T[a];
    t.hb0[a] = P0 >> 1;
    const bool big = g.D[a] > 1;
    t.eoff[a] = big ? 1 : 0;
    t.ne[a] = big ? g.T[a] / 2 : 1;
  }
  if (!DECOMP)
    for (int i = threadIdx.x; i < 256; i += blockDim.x) shist[i] = 0;
  const double eb = st->eb, two_eb = st->two_eb;
  const unsigned long long ocount = DECOMP ? *ocount_dev : 0;
  // 1) the known 2s-lattice (class 0) from E, with halo
  {
    const int* e = g.ext[0];
    const int cnt = e[0] * e[1] * e[2];
    const long long s = g.s, E1 = g.Ed[1], E2 = g.Ed[2];
    for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) {
      const int l2 = idx % e[2], l1 = (idx / e[2]) % e[1], l0 = idx / (e[2] * e[1]);
      const long long h0 = t.hb0[0] - t.eoff[0] + l0, h1 = t.hb0[1] - t.eoff[1] + l1, h2 = t.hb0[2] - t.eoff[2] + l2;
      double v = 0.0;
      if (h0 >= 0 && 2 * h0 < g.D[0] && h1 >= 0 && 2 * h1 < g.D[1] && h2 >= 0 && 2 * h2 < g.D[2]) {
        v = E[((h0 * s) * E1 + h1 * s) * E2 + h2 * s];
        if (DECOMP && g.level == 1) {
          const bool owned = l0 >= t.eoff[0] && l0 < t.eoff[0] + t.ne[0] && l1 >= t.eoff[1] &&
                             l1 < t.eoff[1] + t.ne[1] && l2 >= t.eoff[2] && l2 < t.eoff[2] + t.ne[2];
          if (owned) out[((2 * h0) * g.d[1] + 2 * h1) * g.d[2] + 2 * h2] = (T)v;
          if (owned && !isfinite(v)) raise_flag(st, F_NONFINITE);
        }
      }
      sm[idx] = v;
    }
  }
  __syncthreads();
  const int cfg = st->cfg[g.level - 1];
  bool bad = false;
  switch (cfg & 3) {
    case 0: run_tile<T, false, false, DECOMP>(g, t, sm, shist, field, E, seq, obm, oidx, oval, ocount, out, eb, two_eb, st, &bad); break;
    case 1: run_tile<T, true, false, DECOMP>(g, t, sm, shist, field, E, seq, obm, oidx, oval, ocount, out, eb, two_eb, st, &bad); break;
    case 2: run_tile<T, false, true, DECOMP>(g, t, sm, shist, field, E, seq, obm, oidx, oval, ocount, out, eb, two_eb, st, &bad); break;
    default: run_tile<T, true, true, DECOMP>(g, t, sm, shist, field, E, seq, obm, oidx, oval, ocount, out, eb, two_eb, st, &bad); break;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) raise_flag(st, DECOMP ? F_ORPHAN : F_NONFINITE);
  if (!DECOMP) {
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
      if (shist[i]) atomicAdd(&st->hist[i], (unsigned long long)shist[i]);
  }
}

void level_kernel_smem_init() {
  static const bool done = [] {  // once per process, thread-safe
    cudaFuncSetAttribute(k_level<float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_level<double, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_level<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_level<double, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return true;
  }();
  (void)done;
}

void launch_level_compress(const LevelGeom& g, const void* field, int prec, double* E, uint8_t* seq, uint32_t* obm,
                           DevState* st, cudaStream_t s, int* launches, int cfg, double* scr) {
  if (!getenv("HB_GENERIC_LEVELS")) {  // multidim 3D levels: one marching launch (k_march.cu)
    if (const int n = launch_level_march_compress(g, field, prec, E, seq, obm, st, s, cfg)) {
      *launches += n;
      return;
    }
  }
  if (!getenv("HB_GENERIC_LEVELS")) {  // level 1 of 3D fields: TMA dependency passes (k_pass.cu)
    if (const int n = launch_level_pass_compress(g, field, prec, E, seq, obm, scr, st, s, cfg)) {
      *launches += n;
      return;
    }
  }
  if (!getenv("HB_GENERIC_LEVELS")) {
    if (const int n = launch_level_tiled_compress(g, field, prec, E, seq, obm, st, s, cfg)) {
      *launches += n;
      return;
    }
  }
  level_kernel_smem_init();
  const unsigned blocks = (unsigned)((long long)g.ntile[0] * g.ntile[1] * g.ntile[2]);
  const size_t smem = (size_t)g.smem_doubles * sizeof(double);
  if (prec == 4)
    k_level<float, false><<<blocks, 256, smem, s>>>(g, (const float*)field, E, seq, obm, nullptr, nullptr, nullptr,
                                                   nullptr, st);
  else
    k_level<double, false><<<blocks, 256, smem, s>>>(g, (const double*)field, E, seq, obm, nullptr, nullptr, nullptr,
                                                    nullptr, st);
  (*launches)++;
}

void launch_level_decompress(const LevelGeom& g, const uint8_t* seq, const uint64_t* oidx, const double* oval,
                             const unsigned long long* ocount_dev, double* E, void* out, int prec, DevState* st,
                             cudaStream_t s, int* launches, int cfg, double* scr) {
  if (!getenv("HB_GENERIC_LEVELS")) {  // multidim 3D levels: one marching launch (k_march.cu)
    if (const int n = launch_level_march_decompress(g, seq, oidx, oval, ocount_dev, E, out, prec, st, s, cfg)) {
      *launches += n;
      return;
    }
  }
  if (!getenv("HB_GENERIC_LEVELS")) {  // level 1 of 3D fields: TMA dependency passes (k_pass.cu)
    if (const int n = launch_level_pass_decompress(g, seq, oidx, oval, ocount_dev, E, out, prec, scr, st, s, cfg)) {
      *launches += n;
      return;
    }
  }
  if (!getenv("HB_GENERIC_LEVELS")) {
    if (const int n = launch_level_tiled_decompress(g, seq, oidx, oval, ocount_dev, E, out, prec, st, s, cfg)) {
      *launches += n;
      return;
    }
  }
  level_kernel_smem_init();
  const unsigned blocks = (unsigned)((long long)g.ntile[0] * g.ntile[1] * g.ntile[2]);
  const size_t smem = (size_t)g.smem_doubles * sizeof(double);
  if (prec == 4)
    k_level<float, true><<<blocks, 256, smem, s>>>(g, nullptr, E, const_cast<uint8_t*>(seq), nullptr, oidx, oval,
                                                  ocount_dev, (float*)out, st);
  else
    k_level<double, true><<<blocks, 256, smem, s>>>(g, nullptr, E, const_cast<uint8_t*>(seq), nullptr, oidx, oval,
                                                   ocount_dev, (double*)out, st);
  (*launches)++;
}

// ---------------------------------------------------- outlier compaction
// Linear-order bitmap -> ascending (u64 index, value) records written straight
// into the archive's outlier section (archive.py:65-71, packed, unaligned).
// Persistent CTAs take 8192-word tiles by ticket; a decoupled look-back gives
// each tile its record offset.

constexpr int OC_WORDS = 8192;

template <typename T>
__global__ void __launch_bounds__(256) k_outlier_compact(const uint32_t* __restrict__ bm, unsigned long long nwords,
                                                         const T* __restrict__ field, uint8_t* rec, uint64_t* oidx,
                                                         T* oval, unsigned long long* status, DevState* st) {
  __shared__ unsigned long long sh[33];
  __shared__ unsigned long long tile_sh, base_sh;
  const unsigned long long ntiles = cdiv(nwords, OC_WORDS);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) tile_sh = atomicAdd(&st->tickets[0], 1ull);
    __syncthreads();
    const unsigned long long tile = tile_sh;
    if (tile >= ntiles) break;
    const unsigned long long w0 = tile * OC_WORDS + (unsigned long long)wid * 1024;
    unsigned cnt = 0;
    for (int k = 0; k < 32; k++) {
      const unsigned long long w = w0 + k * 32 + lane;
      cnt += w < nwords ? __popc(bm[w]) : 0;
    }
    unsigned long long total;
    const unsigned long long wsum = warp_sum<unsigned long long>(cnt);
    // block scan over warps (lane 0 of each warp contributes)
    unsigned long long wexcl = block_excl_scan<unsigned long long>(lane == 0 ? wsum : 0ull, sh, &total);
    wexcl = __shfl_sync(0xffffffffu, wexcl, 0);
    if (threadIdx.x < 32) {
      const unsigned long long ex_ = lookback_warp(status, tile, total);
      if (threadIdx.x == 0) base_sh = ex_;
    }
    __syncthreads();
    unsigned long long r = base_sh + wexcl;
    if (total) {
      for (int k = 0; k < 32; k++) {
        const unsigned long long w = w0 + k * 32 + lane;
        const uint32_t bits = w < nwords ? bm[w] : 0u;
        const unsigned c = __popc(bits);
        unsigned incl = warp_incl_scan<unsigned>(c);
        unsigned long long my = r + incl - c;
        uint32_t b = bits;
        while (b) {
          const int bit = __ffs(b) - 1;
          b &= b - 1;
          const unsigned long long idx = w * 32 + bit;
          const T v = field[idx];
          if (rec) {
            uint8_t* p = rec + my * (8 + sizeof(T));
            for (int q = 0; q < 8; q++) p[q] = (uint8_t)(idx >> (8 * q));
            const uint8_t* vb = reinterpret_cast<const uint8_t*>(&v);
            for (int q = 0; q < (int)sizeof(T); q++) p[8 + q] = vb[q];
          }
          if (oidx) oidx[my] = idx;
          if (oval) oval[my] = v;
          my++;
        }
        r += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) st->outlier_count = base_sh + total;
    __syncthreads();
  }
}

void launch_outlier_compact(const uint32_t* obitmap, unsigned long long n, const void* field, int prec,
                            uint8_t* rec_out, uint64_t* oidx_out, void* oval_out, unsigned long long* lb_status,
                            DevState* st, cudaStream_t s, int* launches) {
  const unsigned long long nwords = cdiv(n, 32);
  unsigned long long tiles = cdiv(nwords, OC_WORDS);
  unsigned grid = (unsigned)(tiles < 148ull * 4 ? tiles : 148ull * 4);
  if (prec == 4)
    k_outlier_compact<float><<<grid, 256, 0, s>>>(obitmap, nwords, (const float*)field, rec_out, oidx_out,
                                                  (float*)oval_out, lb_status, st);
  else
    k_outlier_compact<double><<<grid, 256, 0, s>>>(obitmap, nwords, (const double*)field, rec_out, oidx_out,
                                                   (double*)oval_out, lb_status, st);
  (*launches)++;
}

// decompress: archive outlier records -> aligned arrays + validation
// (archive.py:139-147: idx < n, strictly ascending)
template <typename T>
__global__ void k_outliers_parse(const uint8_t* __restrict__ rec, const unsigned long long* count_dev,
                                 unsigned long long n, uint64_t* oidx, double* oval, DevState* st) {
  const unsigned long long k = *count_dev;
  bool bad = false;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint8_t* p = rec + i * (8 + sizeof(T));
    unsigned long long idx = 0;
    for (int q = 0; q < 8; q++) idx |= (unsigned long long)p[q] << (8 * q);
    T v;
    uint8_t* vb = reinterpret_cast<uint8_t*>(&v);
    for (int q = 0; q < (int)sizeof(T); q++) vb[q] = p[8 + q];
    oidx[i] = idx;
    oval[i] = (double)v;
    bad |= idx >= n;
    if (i > 0) {
      const uint8_t* pp = rec + (i - 1) * (8 + sizeof(T));
      unsigned long long prev = 0;
      for (int q = 0; q < 8; q++) prev |= (unsigned long long)pp[q] << (8 * q);
      bad |= idx <= prev;
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) raise_flag(st, F_ARCHIVE, 10);
}

void launch_outliers_parse(const uint8_t* rec, int prec, unsigned long long count_max,
                           const unsigned long long* count_dev, unsigned long long n, uint64_t* oidx, double* oval,
                           DevState* st, cudaStream_t s, int* launches) {
  unsigned long long blocks = cdiv(count_max ? count_max : 1, 256);
  if (blocks > 148ull * 8) blocks = 148ull * 8;
  if (prec == 4)
    k_outliers_parse<float><<<(unsigned)blocks, 256, 0, s>>>(rec, count_dev, n, oidx, oval, st);
  else
    k_outliers_parse<double><<<(unsigned)blocks, 256, 0, s>>>(rec, count_dev, n, oidx, oval, st);
  (*launches)++;
}

// ------------------------------------------------------------- reorder
// ordering.py:142-179 for the parity hooks (the compress/decompress path
// fuses the mapping into the level kernels).

struct LMap {
  long long d[3];
  int top;
  long long sub[5][3];
  long long prefix[5];
};

__device__ __forceinline__ long long lmap_index(const LMap& m, long long x, long long y, long long z) {
  int l = m.top;
  while (l > 0) {
    const long long msk = (1ll << l) - 1;
    if (!(x & msk) && !(y & msk) && !(z & msk)) break;
    l--;
  }
  const long long gy = m.sub[l][1], gz = m.sub[l][2];
  const long long X = x >> l, Y = y >> l, Z = z >> l;
  long long r = (X * gy + Y) * gz + Z;
  if (l < m.top) {
    const long long ey = (gy + 1) >> 1, ez = (gz + 1) >> 1;
    r -= ((X + 1) >> 1) * ey * ez;
    if (!(X & 1)) {
      r -= ((Y + 1) >> 1) * ez;
      if (!(Y & 1)) r -= (Z + 1) >> 1;
    }
  }
  return m.prefix[l] + r;
}

__global__ void k_reorder(LMap m, const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int inverse) {
  const unsigned long long n = (unsigned long long)(m.d[0] * m.d[1] * m.d[2]);
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const long long z = i % m.d[2], y = (i / m.d[2]) % m.d[1], x = i / (m.d[2] * m.d[1]);
    const long long j = lmap_index(m, x, y, z);
    if (inverse)
      out[i] = in[j];
    else
      out[j] = in[i];
  }
}

void launch_reorder(const uint8_t* in, const uint64_t dims[3], int stride, uint8_t* out, bool inverse,
                    cudaStream_t s, int* launches) {
  LMap m;
  for (int a = 0; a < 3; a++) m.d[a] = (long long)dims[a];
  m.top = ilog2i(stride);
  for (int l = 0; l <= m.top; l++)
    for (int a = 0; a < 3; a++) m.sub[l][a] = (m.d[a] + (1ll << l) - 1) >> l;
  for (int l = 0; l <= m.top; l++)
    m.prefix[l] = l == m.top ? 0 : m.sub[l + 1][0] * m.sub[l + 1][1] * m.sub[l + 1][2];
  const unsigned long long n = dims[0] * dims[1] * dims[2];
  unsigned long long blocks = cdiv(n, 256);
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  k_reorder<<<(unsigned)blocks, 256, 0, s>>>(m, in, out, inverse ? 1 : 0);
  (*launches)++;
}

}  // namespace hb
