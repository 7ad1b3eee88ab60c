// hb_interp.cuh -- bit-exact f64 spline stencils and the error-bounded
// quantizer, shared by the level kernels (k_predict.cu) and the tuner
// (k_tune.cu).
//
// Every product and sum is an explicitly rounded __dmul_rn/__dadd_rn so no
// FMA contraction can occur (the reference evaluates numpy ufuncs one rounded
// op at a time: predictor.py:221-226, :320-328).  The library is also built
// with --fmad=false as a second line of defence.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

namespace hb {

// stencil classes (predictor.py:47-52); numbering is internal
enum : int { ST_CUBIC = 0, ST_QLO = 1, ST_QHI = 2, ST_MID = 3, ST_TRAIL = 4, ST_COPY = 5 };

// predictor.py:181-206 with the target at lattice position `pos` along an
// axis of `d` points and stencil step `s` (pos, d in the same units).
__device__ __forceinline__ int classify(long long pos, long long d, long long s, bool linear) {
  const bool p1 = pos + s < d, m3 = pos >= 3 * s;
  if (linear) return p1 ? ST_MID : (m3 ? ST_TRAIL : ST_COPY);
  const bool p3 = pos + 3 * s < d;
  if (m3 && p3) return ST_CUBIC;
  if (!m3 && p3) return ST_QLO;
  if (m3 && p1) return ST_QHI;
  if (p1) return ST_MID;
  if (m3) return ST_TRAIL;
  return ST_COPY;
}

__device__ __forceinline__ int stencil_order(int cls) {
  return cls == ST_CUBIC ? 4 : (cls <= ST_QHI ? 3 : (cls == ST_COPY ? 1 : 2));
}

// v0..v3 are the samples at offsets -3, -1, +1, +3 (units of the stencil
// step); only the ones the class uses are read.  Evaluation order is the
// reference's: acc = v*w (first offset), then acc = acc + v*w in offset order.
__device__ __forceinline__ double apply_stencil(int cls, double v0, double v1, double v2, double v3) {
  switch (cls) {
    case ST_CUBIC:
      return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(v0, -0.0625), __dmul_rn(v1, 0.5625)), __dmul_rn(v2, 0.5625)),
                       __dmul_rn(v3, -0.0625));
    case ST_QLO:
      return __dadd_rn(__dadd_rn(__dmul_rn(v1, 0.375), __dmul_rn(v2, 0.75)), __dmul_rn(v3, -0.125));
    case ST_QHI:
      return __dadd_rn(__dadd_rn(__dmul_rn(v0, -0.125), __dmul_rn(v1, 0.75)), __dmul_rn(v2, 0.375));
    case ST_MID:
      return __dadd_rn(__dmul_rn(v1, 0.5), __dmul_rn(v2, 0.5));
    case ST_TRAIL:
      return __dadd_rn(__dmul_rn(v0, -0.5), __dmul_rn(v1, 1.5));
    default:
      return __dmul_rn(v1, 1.0);
  }
}

// predictor.py:247-256: average of the axis predictions that reach the best
// order, accumulated in ascending axis order from +0.0, then num/den.
__device__ __forceinline__ double combine_axes(int k, const double* p, const int* o) {
  int best = o[0];
  for (int i = 1; i < k; i++) best = o[i] > best ? o[i] : best;
  double num = 0.0;
  int den = 0;
  for (int i = 0; i < k; i++)
    if (o[i] == best) {
      num = __dadd_rn(num, p[i]);
      den++;
    }
  if (den == 1) return num;
  if (den == 2) return __dmul_rn(num, 0.5);  // exact: x/2 == x*0.5 in IEEE
  return __ddiv_rn(num, (double)den);
}

// predictor.py:313-329 for one element.  Returns the code byte (0 = outlier)
// and writes the value the working grid keeps.
template <bool CAST32>
__device__ __forceinline__ int quantize(double o, double p, double eb, double two_eb, double* recon) {
  const double err = __dsub_rn(o, p);
  const double q = copysign(floor(__dadd_rn(__ddiv_rn(fabs(err), two_eb), 0.5)), err);
  const bool small = fabs(q) <= 127.0;
  const double r = __dadd_rn(p, __dmul_rn(two_eb, q));
  const double stored = CAST32 ? (double)__double2float_rn(r) : r;
  const bool ok = small && (fabs(__dsub_rn(o, stored)) <= eb);
  *recon = ok ? r : o;
  return ok ? (int)__dadd_rn(q, 128.0) : 0;
}

// Same result as quantize<>, with the IEEE quotient |err|/two_eb replaced by a
// multiplication with the rounded reciprocal whenever that cannot change
// floor(q + 0.5).  For x = |err|/two_eb < 200 the product differs from the
// correctly rounded quotient by < 2^-43 after the +0.5, so a fractional part
// at least 2^-40 away from an integer proves both floors agree; otherwise
// (or for non-finite values) the exact division is evaluated.  For x >= 200
// the code is an outlier either way (|q| > 127) and the stored value is the
// original, so an off-by-one q cannot change the result.
template <bool CAST32>
__device__ __forceinline__ int quantize_fast(double o, double p, double eb, double two_eb, double inv_two_eb,
                                             double* recon) {
  const double err = __dsub_rn(o, p);
  const double ae = fabs(err);
  double u = __dadd_rn(__dmul_rn(ae, inv_two_eb), 0.5);
  double f = floor(u);
  const double fr = __dsub_rn(u, f);
  if (!(fr > 0x1p-40 && fr < 1.0 - 0x1p-40) && !(u >= 200.5)) {  // NaN lands here too
    u = __dadd_rn(__ddiv_rn(ae, two_eb), 0.5);
    f = floor(u);
  }
  const double q = copysign(f, err);
  const bool small = fabs(q) <= 127.0;
  const double r = __dadd_rn(p, __dmul_rn(two_eb, q));
  const double stored = CAST32 ? (double)__double2float_rn(r) : r;
  const bool ok = small && (fabs(__dsub_rn(o, stored)) <= eb);
  *recon = ok ? r : o;
  return ok ? (int)__dadd_rn(q, 128.0) : 0;
}

// predictor.py:399: replay of a stored code
__device__ __forceinline__ double dequantize(double p, double two_eb, int code) {
  return __dadd_rn(p, __dmul_rn(two_eb, __dsub_rn((double)code, 128.0)));
}

}  // namespace hb
