// k_pass.cu -- level kernels as dependency passes (3D fields).
//
// A level of the interpolation predictor (predictor.py:264-304) visits the
// parity classes of its lattice in at most three dependency steps: multidim
// {1,2,4} -> {3,5,6} -> {7}; seq1d {b0} -> {b1, b0|b1} -> {b2, b0|b2, b1|b2, 7}.
// Instead of recomputing a +-3 halo inside shared-memory tiles, each step is
// one launch that computes every target of its classes exactly once and
// writes the f64 reconstruction to HBM: into the E lattice for levels >= 2
// (all their targets lie on the 2-lattice of the full grid) and into a
// per-class scratch array for level 1.  The next step reads those values back
// through L1/L2.  HBM is otherwise idle on this compute-bound path, so trading
// ~3 GB of traffic per level-1 pass set for the 1.54x halo recompute, the
// shared-memory staging and the per-phase barriers is a net win.
//
// Thread mapping: lanes walk z (consecutive in memory), warps walk y, each
// thread owns a run of RX targets along x whose x-stencil source values sit
// in a register window (RX + 3 loads for RX targets).  Blocks whose targets
// all have complete stencils take the branch-free INT path; boundary blocks
// classify per point (predictor.py:181-206).
//
// Reference: predictor.py:181-304 (prediction), :313-329 (quantize),
// :397-411 (replay), ordering.py:68-84 (Eq. 3 slot of every code).
#include "hb_common.cuh"
#include "hb_interp.cuh"
#include "hb_kernels.h"

#include <algorithm>

namespace hb {

namespace {

constexpr int PW = 4;          // warps per block (y)
constexpr int RX = 8;          // targets per thread along x
constexpr int P_THREADS = PW * 32;
#ifndef PASS_MINB
#define PASS_MINB 4
#endif

struct PassArgs {
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
  double* scr;             // level 1: class c (1..6) at scr + (c - 1) * cstride
  long long cstride;
  int ncls;
  int cls[4], axm[4];
  int nbx;                 // x blocks per class (grid.z = ncls * nbx)
};

// half-index extent of parity class `cls` along axis a of the level lattice
__device__ __forceinline__ int cdim(const LevelGeom& g, int cls, int a) {
  return ((cls >> a) & 1) ? (int)(g.D[a] >> 1) : (int)((g.D[a] + 1) >> 1);
}

// where class `cls` keeps its reconstruction: base pointer + strides per half-index
struct Src {
  const double* p;
  long long st[3];
};
__device__ __forceinline__ Src src_of(const PassArgs& A, int cls) {
  const LevelGeom& g = A.g;
  Src r;
  if (cls == 0 || g.level >= 2) {
    const long long es[3] = {g.Ed[1] * g.Ed[2], g.Ed[2], 1};
    long long off = 0;
    for (int a = 0; a < 3; a++) {
      r.st[a] = g.s * es[a];
      if ((cls >> a) & 1) off += (g.s >> 1) * es[a];
    }
    r.p = A.E + off;
  } else {
    const long long n1 = cdim(g, cls, 1), n2 = cdim(g, cls, 2);
    r.st[0] = n1 * n2, r.st[1] = n2, r.st[2] = 1;
    r.p = A.scr + (cls - 1) * A.cstride;
  }
  return r;
}

// code 0 on decompress: the outlier value at linear index `lin`
// (predictor.py:400-405; orphan -> ArchiveError).  Rare, kept out of line.
__device__ __noinline__ double pass_outlier(const PassArgs& A, unsigned long long lin, unsigned long long cnt,
                                            bool& bad) {
  unsigned long long a0 = 0, a1 = cnt;
  while (a0 < a1) {
    const unsigned long long mid = (a0 + a1) >> 1;
    if (A.oidx[mid] < lin)
      a0 = mid + 1;
    else
      a1 = mid;
  }
  if (a0 < cnt && A.oidx[a0] == lin) return A.oval[a0];
  bad = true;
  return 0.0;
}

struct Acc {
  unsigned h127, h128, h129;
  bool bad, nf;
};

// One thread: targets (x0 + i, y, z), i < nx, of class CLS interpolated along
// the K axes of AXM.  INT: every stencil is complete (no classify).  64-bit
// base pointers per thread, 32-bit steps per target.
template <typename T, bool DEC, int K, bool LINEAR, bool INT>
__device__ __forceinline__ void pass_run(const PassArgs& A, int CLS, int AXM, int x0, int nx, int y, int z,
                                         const double eb, const double two_eb, const double inv_two_eb,
                                         unsigned long long ocount, unsigned* shist, Acc& acc) {
  const LevelGeom& g = A.g;
  const int odd0 = CLS & 1, odd1 = (CLS >> 1) & 1, odd2 = (CLS >> 2) & 1;
  const long long P0 = 2ll * x0 + odd0, P1 = 2ll * y + odd1, P2 = 2ll * z + odd2;
  const long long s = g.s;
  // bases at x0 (element index, Eq. 3 slot) and 32-bit x steps
  const long long lin = ((P0 * s) * g.d[1] + P1 * s) * g.d[2] + P2 * s;
  long long slot = g.prefix + (P0 * g.D[1] + P1) * g.D[2] + P2 - ((P0 + 1) >> 1) * g.eyez;
  if (!odd0) {
    slot -= ((P1 + 1) >> 1) * g.ez;
    if (!odd1) slot -= (P2 + 1) >> 1;
  }
  const int kl0 = (int)g.kl[0], ks0 = (int)g.ks0;
  const T* fp = reinterpret_cast<const T*>(A.field) + lin;
  uint8_t* sq = A.seq + slot;
  // where this class's reconstruction goes (levels >= 2: E; level 1: scratch, class 7 nowhere)
  const Src dst = src_of(A, CLS);
  double* dp = const_cast<double*>(dst.p) + x0 * dst.st[0] + y * dst.st[1] + z * dst.st[2];
  const int dst0 = (int)dst.st[0];
  const bool wr = g.level >= 2 || CLS != 7;

  // ---- loads of the run (issued together)
  T o[RX];
  uint8_t cd[RX];
#pragma unroll
  for (int i = 0; i < RX; i++) {
    if (i < nx) {
      if (!DEC)
        o[i] = __ldg(fp + i * kl0);
      else
        cd[i] = __ldg(sq + i * ks0);
    }
  }
  // ---- stencil sources of the K axes (ascending axis order, predictor.py:247-256)
  const double* sp[K];
  int sst[K], sx[K], sax[K], scls[K];
  double w[RX + 3];  // x-stencil window (axis 0 is always the first axis when present)
  {
    int m = AXM;
#pragma unroll
    for (int j = 0; j < K; j++) {
      const int a = __ffs(m) - 1;
      m &= m - 1;
      const int cn = CLS & ~(1 << a);
      const Src S = src_of(A, cn);
      sax[j] = a;
      sst[j] = (int)S.st[a];
      sx[j] = (int)S.st[0];
      const double* base = S.p + y * S.st[1] + z * S.st[2];
      if (a == 0) {
        // window: source x indices x0-1 .. x0+RX+1, clamped into the array
        const int na = cdim(g, cn, 0);
#pragma unroll
        for (int k = 0; k < RX + 3; k++) {
          const int xi = min(max(x0 - 1 + k, 0), na - 1);
          w[k] = __ldg(base + xi * sx[j]);
        }
        sp[j] = base;
      } else {
        sp[j] = base + x0 * S.st[0] - sst[j];  // first stencil point (offset -1 along a)
      }
      if (!INT && a != 0) {
        scls[j] = classify(a == 1 ? P1 : P2, g.D[a], 1, LINEAR);
      } else {
        scls[j] = LINEAR ? ST_MID : ST_CUBIC;
      }
    }
  }
  // clamped y / z stencil loads: indices outside the source array are never
  // used by the (boundary) stencil class, they only must not fault
  int lo1 = 0, hi1 = 3, lo2 = 0, hi2 = 3;
  if (!INT) {
    const int n1s = cdim(g, CLS & ~2, 1), n2s = cdim(g, CLS & ~4, 2);
    lo1 = y - 1 < 0 ? 1 : 0, hi1 = (y + 2 >= n1s) ? n1s - 1 - (y - 1) : 3;
    lo2 = z - 1 < 0 ? 1 : 0, hi2 = (z + 2 >= n2s) ? n2s - 1 - (z - 1) : 3;
  }

#pragma unroll
  for (int i = 0; i < RX; i++) {
    if (i >= nx) break;
    double pv[K];
    int ov[K];
#pragma unroll
    for (int j = 0; j < K; j++) {
      const int a = sax[j];
      int cls = scls[j];
      double v0, v1, v2, v3;
      if (a == 0) {
        if (!INT) cls = classify(P0 + 2 * i, g.D[0], 1, LINEAR);
        v0 = w[i], v1 = w[i + 1], v2 = w[i + 2], v3 = w[i + 3];
      } else {
        const double* q = sp[j] + i * sx[j];
        const int t = sst[j];
        if (INT && LINEAR) {
          v0 = 0.0, v1 = q[t], v2 = q[2 * t], v3 = 0.0;
        } else if (INT) {
          v0 = q[0], v1 = q[t], v2 = q[2 * t], v3 = q[3 * t];
        } else {
          const int lo = a == 1 ? lo1 : lo2, hi = a == 1 ? hi1 : hi2;
          v0 = q[min(max(0, lo), hi) * t];
          v1 = q[min(max(1, lo), hi) * t];
          v2 = q[min(max(2, lo), hi) * t];
          v3 = q[min(max(3, lo), hi) * t];
        }
      }
      pv[j] = apply_stencil(INT ? (LINEAR ? ST_MID : ST_CUBIC) : cls, v0, v1, v2, v3);
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
        r = pass_outlier(A, (unsigned long long)(lin + (long long)i * kl0), ocount, acc.bad);
      if (g.level == 1) {
        reinterpret_cast<T*>(A.out)[lin + (long long)i * kl0] = (T)r;
        acc.nf |= !isfinite(r);
      }
    }
    if (wr) dp[i * dst0] = r;
  }
}

// ------------------------------------------------------------------ kernel
template <typename T, bool DEC, int K, bool LINEAR>
__global__ void __launch_bounds__(P_THREADS, PASS_MINB) k_pass(PassArgs A) {
  __shared__ unsigned shist[256];
  const LevelGeom& g = A.g;
  if (!DEC)
    for (int i = threadIdx.x; i < 256; i += P_THREADS) shist[i] = 0;
  // grid: (z blocks, y blocks, class-major x blocks); blocks past a class's extent idle
  int k = 0, bx = blockIdx.z;
  while (k + 1 < A.ncls && bx >= A.nbx) bx -= A.nbx, k++;
  const int CLS = A.cls[k], AXM = A.axm[k];
  const int bz = blockIdx.x, by = blockIdx.y;
  const int n0 = cdim(g, CLS, 0), n1 = cdim(g, CLS, 1), n2 = cdim(g, CLS, 2);
  const int x0 = bx * RX, y = by * PW + (threadIdx.x >> 5), z = bz * 32 + (threadIdx.x & 31);
  const int nx = n0 - x0 < RX ? n0 - x0 : RX;
  // complete stencils for every target of the block along every axis of AXM
  // (cubic: P >= 3 and P + 3 < D; linear: P + 1 < D; predictor.py:181-206)
  bool full = true;
  {
    const int lo[3] = {x0, by * PW, bz * 32};
    const int hi[3] = {x0 + nx - 1, min(by * PW + PW, n1) - 1, min(bz * 32 + 32, n2) - 1};
#pragma unroll
    for (int a = 0; a < 3; a++)
      if ((AXM >> a) & 1) {
        const long long Plo = 2ll * lo[a] + 1, Phi = 2ll * hi[a] + 1;
        full &= LINEAR ? (Phi + 1 < g.D[a]) : (Plo >= 3 && Phi + 3 < g.D[a]);
      }
  }
  const double eb = A.st->eb, two_eb = A.st->two_eb;
  const double inv_two_eb = __ddiv_rn(1.0, two_eb);
  const unsigned long long ocount = DEC ? *A.ocount : 0;
  if (!DEC) __syncthreads();
  Acc acc{0u, 0u, 0u, false, false};
  if (y < n1 && z < n2 && nx > 0) {
    if (full)
      pass_run<T, DEC, K, LINEAR, true>(A, CLS, AXM, x0, nx, y, z, eb, two_eb, inv_two_eb, ocount, shist, acc);
    else
      pass_run<T, DEC, K, LINEAR, false>(A, CLS, AXM, x0, nx, y, z, eb, two_eb, inv_two_eb, ocount, shist, acc);
  }
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
    for (int i = threadIdx.x; i < 256; i += P_THREADS)
      if (shist[i]) atomicAdd(&A.st->hist[i], (unsigned long long)shist[i]);
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

template <typename T, bool DEC, int K, bool LINEAR>
void launch_pass(PassArgs& A, const int* cls, const int* axm, int n, cudaStream_t s, int* launches) {
  A.ncls = n;
  long long mz = 0, my = 0, mx = 0;
  for (int k = 0; k < n; k++) {
    A.cls[k] = cls[k];
    A.axm[k] = axm[k];
    long long nd[3];
    for (int a = 0; a < 3; a++) nd[a] = ((cls[k] >> a) & 1) ? A.g.D[a] >> 1 : (A.g.D[a] + 1) >> 1;
    mz = std::max(mz, (nd[2] + 31) / 32);
    my = std::max(my, (nd[1] + PW - 1) / PW);
    mx = std::max(mx, (nd[0] + RX - 1) / RX);
  }
  if (!mz || !my || !mx) return;
  A.nbx = (int)mx;
  const dim3 grid((unsigned)mz, (unsigned)my, (unsigned)(mx * n));
  k_pass<T, DEC, K, LINEAR><<<grid, P_THREADS, 0, s>>>(A);
  (*launches)++;
}

template <typename T, bool DEC, bool LINEAR>
void run_level_passes(PassArgs& A, int cfg, cudaStream_t s, int* launches) {
  if ((cfg & 2) == 0) {  // multidim: a class interpolates along all its odd axes
    const int c1[3] = {1, 2, 4}, c2[3] = {3, 5, 6}, c3[1] = {7};
    launch_pass<T, DEC, 1, LINEAR>(A, c1, c1, 3, s, launches);
    launch_pass<T, DEC, 2, LINEAR>(A, c2, c2, 3, s, launches);
    launch_pass<T, DEC, 3, LINEAR>(A, c3, c3, 1, s, launches);
  } else {  // seq1d along seq_order (predictor.py:267-280)
    const int b0 = 1 << A.g.seq_order[0], b1 = 1 << A.g.seq_order[1], b2 = 1 << A.g.seq_order[2];
    const int p1c[1] = {b0}, p1a[1] = {b0};
    const int p2c[2] = {b1, b0 | b1}, p2a[2] = {b1, b1};
    const int p3c[4] = {b2, b0 | b2, b1 | b2, 7}, p3a[4] = {b2, b2, b2, b2};
    launch_pass<T, DEC, 1, LINEAR>(A, p1c, p1a, 1, s, launches);
    launch_pass<T, DEC, 1, LINEAR>(A, p2c, p2a, 2, s, launches);
    launch_pass<T, DEC, 1, LINEAR>(A, p3c, p3a, 4, s, launches);
  }
}

template <typename T, bool DEC>
void run_level(PassArgs& A, int cfg, cudaStream_t s, int* launches) {
  if (cfg & 1)
    run_level_passes<T, DEC, true>(A, cfg, s, launches);
  else
    run_level_passes<T, DEC, false>(A, cfg, s, launches);
}

}  // namespace

size_t level_scratch_bytes(const uint64_t dims[3]) {
  unsigned long long ne = 1;
  for (int a = 0; a < 3; a++) ne *= (dims[a] + 1) / 2;
  return (size_t)6 * ne * 8 + 256;
}

bool pass_supported(const LevelGeom& g) { return g.d[0] > 1 && g.d[1] > 1 && g.d[2] > 1; }

int launch_level_pass_compress(const LevelGeom& g, const void* field, int prec, double* E, uint8_t* seq, uint32_t* obm,
                               double* scr, DevState* st, cudaStream_t s, int cfg) {
  if (cfg < 0 || !pass_supported(g) || !scr) return 0;
  PassArgs A{};
  A.g = g;
  A.field = field;
  A.E = E;
  A.seq = seq;
  A.obm = obm;
  A.st = st;
  A.scr = scr;
  A.cstride = (long long)((g.d[0] + 1) / 2) * ((g.d[1] + 1) / 2) * ((g.d[2] + 1) / 2);
  int n = 0;
  if (prec == 4)
    run_level<float, false>(A, cfg, s, &n);
  else
    run_level<double, false>(A, cfg, s, &n);
  return n;
}

int launch_level_pass_decompress(const LevelGeom& g, const uint8_t* seq, const uint64_t* oidx, const double* oval,
                                 const unsigned long long* ocount_dev, double* E, void* out, int prec, double* scr,
                                 DevState* st, cudaStream_t s, int cfg) {
  if (cfg < 0 || !pass_supported(g) || !scr) return 0;
  PassArgs A{};
  A.g = g;
  A.E = E;
  A.seq = const_cast<uint8_t*>(seq);
  A.oidx = oidx;
  A.oval = oval;
  A.ocount = ocount_dev;
  A.out = out;
  A.st = st;
  A.scr = scr;
  A.cstride = (long long)((g.d[0] + 1) / 2) * ((g.d[1] + 1) / 2) * ((g.d[2] + 1) / 2);
  int n = 0;
  if (g.level == 1) {
    const long long ne = g.Ed[0] * g.Ed[1] * g.Ed[2];
    const unsigned blocks = (unsigned)std::min<long long>((ne + 255) / 256, 148 * 16);
    if (prec == 4)
      k_even_out<float><<<blocks, 256, 0, s>>>(E, g, reinterpret_cast<float*>(out), st);
    else
      k_even_out<double><<<blocks, 256, 0, s>>>(E, g, reinterpret_cast<double*>(out), st);
    n++;
  }
  if (prec == 4)
    run_level<float, true>(A, cfg, s, &n);
  else
    run_level<double, true>(A, cfg, s, &n);
  return n;
}

}  // namespace hb
