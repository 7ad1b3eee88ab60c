// k_quality.cu -- reconstruction quality metrics in one HBM pass
// (reference field.py:145-187: mse, max_abs_error, psnr's value range).
//
// One read of the original and the reconstruction produces
//   sum((o - r)^2)   in numpy's pairwise summation order, so mse = sum / N is
//                    bit-identical to np.mean(d * d) (field.py:148-149)
//   max |o - r|      (field.py:155, order-free)
//   min / max of o   in the field dtype (value_range, field.py:129-132)
//
// numpy's pairwise sum of n contiguous doubles (umath loops, PW_BLOCKSIZE
// 128): n < 8 sequential from 0.0; n <= 128 eight strided accumulators
// combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail;
// otherwise split at n2 = n/2 - (n/2)%8 and add the halves.  Every node of
// that recursion tree above ~512 elements is internal, so depth D (N/2^D in
// [256, 512)) is a complete level of 2^D nodes: thread t walks from the root
// to node t (D splits), sums its node with the exact recursion, and the 2^D
// node sums are combined as the perfect binary tree they form -- in shared
// memory per CTA, then across CTAs by the last CTA to finish.
#include <cuda_runtime.h>
#include <stdint.h>

#include "hb_common.cuh"
#include "hb_kernels.h"

namespace hb {

namespace {

constexpr int QT = 256;

template <typename T>
struct QAcc {
  double mx;  // max |o - r|
  T lo, hi;   // min / max of the original
};

template <typename T>
__device__ __forceinline__ double sq(const T* __restrict__ o, const T* __restrict__ r, long long i, QAcc<T>& a) {
  const T ov = o[i];
  const double d = __dsub_rn((double)ov, (double)r[i]);
  a.mx = fmax(a.mx, fabs(d));
  a.lo = ov < a.lo ? ov : a.lo;
  a.hi = ov > a.hi ? ov : a.hi;
  return __dmul_rn(d, d);
}

// numpy pairwise_sum_DOUBLE on the squared differences of [i0, i0 + n);
// DEPTH bounds the remaining recursion (nodes handed to a thread are < 544)
template <typename T, int DEPTH>
__device__ double pw(const T* __restrict__ o, const T* __restrict__ r, long long i0, long long n, QAcc<T>& a) {
  if (n < 8) {
    double s = 0.0;
    for (long long i = 0; i < n; i++) s = __dadd_rn(s, sq(o, r, i0 + i, a));
    return s;
  }
  if (DEPTH == 0 || n <= 128) {
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; j++) acc[j] = sq(o, r, i0 + j, a);
    long long i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; j++) acc[j] = __dadd_rn(acc[j], sq(o, r, i0 + i + j, a));
    double s = __dadd_rn(__dadd_rn(__dadd_rn(acc[0], acc[1]), __dadd_rn(acc[2], acc[3])),
                         __dadd_rn(__dadd_rn(acc[4], acc[5]), __dadd_rn(acc[6], acc[7])));
    for (; i < n; i++) s = __dadd_rn(s, sq(o, r, i0 + i, a));
    return s;
  }
  long long n2 = n / 2;
  n2 -= n2 % 8;
  const double left = pw<T, (DEPTH > 0 ? DEPTH - 1 : 0)>(o, r, i0, n2, a);
  return __dadd_rn(left, pw<T, (DEPTH > 0 ? DEPTH - 1 : 0)>(o, r, i0 + n2, n - n2, a));
}

// pairwise-combine w values of s[] (w a power of two) into s[0], in index order
__device__ void tree_combine(double* s, int w) {
  for (; w > 1; w >>= 1) {
    double v = 0.0;
    if ((int)threadIdx.x < w / 2) v = __dadd_rn(s[2 * threadIdx.x], s[2 * threadIdx.x + 1]);
    __syncthreads();
    if ((int)threadIdx.x < w / 2) s[threadIdx.x] = v;
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(QT) k_quality(const T* __restrict__ o, const T* __restrict__ r, long long n,
                                                int depth, double* __restrict__ part, unsigned* ticket,
                                                double* __restrict__ out) {
  __shared__ double s[QT];
  __shared__ double smx[QT / 32], slo[QT / 32], shi[QT / 32];
  __shared__ bool last;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // root -> node t at depth `depth`
  long long i0 = 0, len = n;
  for (int b = depth - 1; b >= 0; b--) {
    long long n2 = len / 2;
    n2 -= n2 % 8;
    if ((t >> b) & 1) {
      i0 += n2;
      len -= n2;
    } else {
      len = n2;
    }
  }
  QAcc<T> a{0.0, (T)INFINITY, (T)-INFINITY};
  const long long nodes = 1ll << depth;  // < blockDim.x only for tiny fields (one CTA of 32)
  s[threadIdx.x] = t < nodes ? pw<T, 3>(o, r, i0, len, a) : 0.0;
  __syncthreads();
  tree_combine(s, nodes < (long long)blockDim.x ? (int)nodes : (int)blockDim.x);
  double mx = a.mx, lo = (double)a.lo, hi = (double)a.hi;
  for (int k = 16; k > 0; k >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, k));
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, k));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, k));
  }
  if ((threadIdx.x & 31) == 0) {
    smx[threadIdx.x >> 5] = mx;
    slo[threadIdx.x >> 5] = lo;
    shi[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x + 31) / 32; w++) {
      mx = fmax(mx, smx[w]);
      lo = fmin(lo, slo[w]);
      hi = fmax(hi, shi[w]);
    }
    const int B = gridDim.x;
    part[blockIdx.x] = s[0];
    part[B + blockIdx.x] = mx;
    part[2 * B + blockIdx.x] = lo;
    part[3 * B + blockIdx.x] = hi;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the last CTA: perfect-tree combine of the per-CTA sums (gridDim.x is a
  // power of two), order-free reductions of the rest
  const int B = gridDim.x;
  // chunks of QT leaves form complete subtrees: combine each chunk, then the
  // chunk results (<= QT of them: n < 2^33, checked by the caller)
  const int chunks = B > QT ? B / QT : 1;
  const int w = B > QT ? QT : B;
  double mxa = 0.0, loa = INFINITY, hia = -INFINITY;
  for (int c = 0; c < chunks; c++) {
    const int k = c * w + threadIdx.x;
    if ((int)threadIdx.x < w) {
      s[threadIdx.x] = __ldcg(&part[k]);
      mxa = fmax(mxa, __ldcg(&part[B + k]));
      loa = fmin(loa, __ldcg(&part[2 * B + k]));
      hia = fmax(hia, __ldcg(&part[3 * B + k]));
    }
    __syncthreads();
    tree_combine(s, w);
    if (threadIdx.x == 0) part[4 * B + c] = s[0];
    __syncthreads();
  }
  if (chunks > 1) {
    for (int c = threadIdx.x; c < chunks; c += blockDim.x) s[c] = part[4 * B + c];
    __syncthreads();
    tree_combine(s, chunks);
  }
  const double psum = s[0];
  for (int k = 16; k > 0; k >>= 1) {
    mxa = fmax(mxa, __shfl_xor_sync(0xffffffffu, mxa, k));
    loa = fmin(loa, __shfl_xor_sync(0xffffffffu, loa, k));
    hia = fmax(hia, __shfl_xor_sync(0xffffffffu, hia, k));
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    smx[threadIdx.x >> 5] = mxa;
    slo[threadIdx.x >> 5] = loa;
    shi[threadIdx.x >> 5] = hia;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x + 31) / 32; q++) {
      mxa = fmax(mxa, smx[q]);
      loa = fmin(loa, slo[q]);
      hia = fmax(hia, shi[q]);
    }
    out[0] = psum;
    out[1] = mxa;
    out[2] = loa;
    out[3] = hia;
    *ticket = 0;  // ready for the next call
  }
}

}  // namespace

int quality_depth(unsigned long long n) {
  int d = 0;
  while ((n >> (d + 1)) >= 256) d++;
  return d;
}

size_t quality_scratch_bytes(unsigned long long n) {
  const int d = quality_depth(n);
  const long long threads = 1ll << d;
  const long long B = threads > QT ? threads / QT : 1;
  return (size_t)(5 * B + 8) * sizeof(double) + 64;
}

void launch_quality(const void* orig, const void* recon, int prec, unsigned long long n, void* scratch,
                    double* out_dev, cudaStream_t s, int* launches) {
  const int d = quality_depth(n);
  const long long threads = 1ll << d;
  const int bs = threads > QT ? QT : (threads < 32 ? 32 : (int)threads);
  const unsigned B = (unsigned)(threads > bs ? threads / bs : 1);
  unsigned* ticket = reinterpret_cast<unsigned*>(scratch);
  double* part = reinterpret_cast<double*>(static_cast<char*>(scratch) + 64);
  cudaMemsetAsync(ticket, 0, sizeof(unsigned), s);
  if (prec == 4)
    k_quality<float><<<B, bs, 0, s>>>((const float*)orig, (const float*)recon, (long long)n, d, part, ticket, out_dev);
  else
    k_quality<double><<<B, bs, 0, s>>>((const double*)orig, (const double*)recon, (long long)n, d, part, ticket,
                                       out_dev);
  (*launches)++;
}

}  // namespace hb
