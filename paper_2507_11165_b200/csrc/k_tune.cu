// k_tune.cu -- sampling auto-tuner (tuning.py:66-170) on the GPU.
//
// One CTA per (config, sample block): the block's f64 state (17^3 = 39 KB)
// and its original values live in shared memory; the level's sub-steps run in
// the reference order, each sub-step's |orig - pred| array is reduced with
// numpy's pairwise summation (leaves of <= 128 elements with 8 strided
// accumulators) and accumulated sequentially, exactly like
// `total += float(np.fabs(ob - pred).sum())` (tuning.py:160).  A 4-thread
// select kernel then sums block errors with CPython 3.12's Neumaier `sum`
// (tuning.py:135), takes the (err, index) argmin (:137) and records the
// winner whose trial grids seed the next level (:140).
#include <cuda_runtime.h>

#include <utility>
#include <vector>

#include "hb_common.cuh"
#include "hb_interp.cuh"
#include "hb_kernels.h"

namespace hb {

constexpr int TUNE_THREADS = 512;
// CONFIG_CHOICES (tuning.py:29) as InterpConfig bytes: bit0 linear, bit1 seq1d
__constant__ uint8_t c_choice[4] = {0x0, 0x2, 0x1, 0x3};

struct SubStep {
  int start[3], step[3], count[3];
  int axes[3];
  int k;
};

// predictor.py:264-296 on block-local dims
__device__ int block_steps(const int d[3], int level, bool seq1d, SubStep* out) {
  const int s = 1 << (level - 1);
  int n = 0;
  if (seq1d) {
    int o[3] = {0, 1, 2};
    for (int i = 0; i < 3; i++)
      for (int j = i + 1; j < 3; j++)
        if (d[o[j]] > d[o[i]] || (d[o[j]] == d[o[i]] && o[j] < o[i])) {
          int t = o[i];
          o[i] = o[j];
          o[j] = t;
        }
    for (int k = 0; k < 3; k++) {
      const int a = o[k];
      SubStep ss;
      for (int j = 0; j < 3; j++) {
        bool earlier = false;
        for (int m = 0; m < k; m++) earlier |= o[m] == j;
        ss.start[j] = j == a ? s : 0;
        ss.step[j] = j == a ? 2 * s : (earlier ? s : 2 * s);
        ss.count[j] = d[j] > ss.start[j] ? (d[j] - ss.start[j] + ss.step[j] - 1) / ss.step[j] : 0;
      }
      ss.axes[0] = a;
      ss.k = 1;
      if (ss.count[a] > 0) out[n++] = ss;
    }
  } else {
    const int sets[7] = {1, 2, 4, 3, 5, 6, 7};
    for (int t = 0; t < 7; t++) {
      SubStep ss;
      bool empty = false;
      ss.k = 0;
      for (int j = 0; j < 3; j++) {
        const bool odd = (sets[t] >> j) & 1;
        ss.start[j] = odd ? s : 0;
        ss.step[j] = 2 * s;
        ss.count[j] = d[j] > ss.start[j] ? (d[j] - ss.start[j] + ss.step[j] - 1) / ss.step[j] : 0;
        if (odd) {
          if (ss.count[j] == 0) empty = true;
          ss.axes[ss.k++] = j;
        }
      }
      if (!empty) out[n++] = ss;
    }
  }
  return n;
}

// numpy pairwise_sum leaf (n <= 128)
__device__ double pw_leaf(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; i++) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = a[j];
  int i;
  for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; i++) res = __dadd_rn(res, a[i]);
  return res;
}

// enumerate leaves of the pairwise recursion in order (explicit stack)
template <typename I>
__device__ int pw_leaves(int n, I* ls, I* ln) {
  int stk_s[32], stk_n[32], sp = 0, nl = 0;
  stk_s[sp] = 0, stk_n[sp] = n, sp++;
  while (sp) {
    sp--;
    const int s0 = stk_s[sp], n0 = stk_n[sp];
    if (n0 <= 128) {
      ls[nl] = (I)s0, ln[nl] = (I)n0, nl++;
    } else {
      int n2 = n0 / 2;
      n2 -= n2 % 8;
      stk_s[sp] = s0 + n2, stk_n[sp] = n0 - n2, sp++;  // right pushed first -> left popped first
      stk_s[sp] = s0, stk_n[sp] = n2, sp++;
    }
  }
  return nl;
}

// combine leaf sums along the same recursion (post-order)
__device__ double pw_combine(int n, const double* leaf, int* cursor) {
  if (n <= 128) return leaf[(*cursor)++];
  int n2 = n / 2;
  n2 -= n2 % 8;
  const double a = pw_combine(n2, leaf, cursor);
  const double b = pw_combine(n - n2, leaf, cursor);
  return __dadd_rn(a, b);
}

// a / b for 0 <= a < 2^22, 0 < b < 2^12 through the float reciprocal rb = 1/b
// (one correction step each way makes it exact)
__device__ __forceinline__ int qdiv(int a, int b, float rb) {
  int q = __float2int_rz(__int2float_rn(a) * rb);
  int r = a - q * b;
  if (r < 0) q--, r += b;
  if (r >= b) q++;
  return q;
}

// tuning.py:135-140 for one level, run by the first warp of the CTA that
// finishes the level last (k_tune_level): Neumaier sum of the block errors per
// config, (err, index) argmin, winner handed to the next level.
// `x` holds the 4 x nb block errors (staged in shared memory by the caller:
// a serial loop of dependent L2 loads cost ~20 us per level).
__device__ void tune_select(int nb, int level, const double* berr, bool staged, DevState* st, uint8_t* host_cfg,
                            cudaGraphConditionalHandle cond) {
  __shared__ double e[4];
  const int ci = threadIdx.x;
  if (ci < 4) {
    const double* x = berr + ci * nb;
    double f = __dadd_rn(0.0, staged ? x[0] : __ldcg(&x[0])), c = 0.0;  // sum() starts from int 0
    for (int i = 1; i < nb; i++) {
      const double xi = staged ? x[i] : __ldcg(&x[i]);
      const double t = __dadd_rn(f, xi);
      if (fabs(f) >= fabs(xi))
        c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), xi));
      else
        c = __dadd_rn(c, __dadd_rn(__dsub_rn(xi, t), f));
      f = t;
    }
    if (c != 0.0 && isfinite(c)) f = __dadd_rn(f, c);
    e[ci] = f;
    st->tune_errs[(level - 1) * 4 + ci] = f;
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    int best = 0;
    for (int i = 1; i < 4; i++)
      if (e[i] < e[best]) best = i;
    st->tune_winner[level - 1] = best;
    st->cfg[level - 1] = c_choice[best];
    __threadfence();
    // inside the compress graph: the level's switch node runs body `best`
    // (the level passes of that config) -- no host round trip
    if (cond) cudaGraphSetConditional(cond, (unsigned)best);
    if (host_cfg) {  // mapped pinned memory: the host reads it once an event after this kernel completes
      host_cfg[level - 1] = c_choice[best];
      __threadfence_system();
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(TUNE_THREADS)
    k_tune_level(const T* __restrict__ field, long long fd1, long long fd2, const unsigned long long* origins, int nb,
                 int b0, int b1, int b2, int top, int level, double* trials, double* berr, DevState* st,
                 T* borig, unsigned* done, uint8_t* host_cfg, cudaGraphConditionalHandle cond) {
  extern __shared__ double tsm[];
  const int bn = b0 * b1 * b2;
  double* g = tsm;
  double* diff = tsm + bn;  // two halves: sub-steps alternate (a sub-step has <= bn/2 targets)
  T* orig = reinterpret_cast<T*>(diff + bn);
  // pairwise-sum leaves of every sub-step (a sub-step has <= bn/2 <= 5120
  // targets and leaves of >= 57, so <= 90 leaves)
  constexpr int TL = 96;
  __shared__ uint16_t lstart[7][TL], llen[7][TL];
  __shared__ double leafv[7][TL];
  __shared__ int nleaf[7];
  const int ci = blockIdx.x / nb, b = blockIdx.x % nb;
  // original block values (tuning.py:111-112): gathered from the field at the
  // top level (and kept compact in borig), read back contiguously below it.
  // Loads are issued in batches of GB per thread (one memory latency per batch).
  constexpr int GB = 8;
  const size_t set_stride = (size_t)4 * nb * bn;
  if (level == top) {
    const unsigned long long ox = origins[3 * b], oy = origins[3 * b + 1], oz = origins[3 * b + 2];
    const float r2 = 1.0f / (float)b2, r12 = 1.0f / (float)(b1 * b2);
    for (int i0 = threadIdx.x; i0 < bn; i0 += GB * blockDim.x) {
      T v[GB];
#pragma unroll
      for (int k = 0; k < GB; k++) {
        const int i = i0 + k * blockDim.x;
        if (i < bn) {
          const int x = qdiv(i, b1 * b2, r12), yz = i - x * b1 * b2, y = qdiv(yz, b2, r2), z = yz - y * b2;
          v[k] = field[((ox + x) * fd1 + oy + y) * fd2 + oz + z];
        }
      }
#pragma unroll
      for (int k = 0; k < GB; k++) {
        const int i = i0 + k * blockDim.x;
        if (i < bn) {
          orig[i] = v[k];
          g[i] = (double)v[k];
          if (ci == 0) borig[(size_t)b * bn + i] = v[k];
        }
      }
    }
  } else {
    // state carried from the previous level's winner (tuning.py:140)
    const int w = st->tune_winner[level];  // winner of level+1
    const double* src = trials + (size_t)((level + 1) & 1) * set_stride + ((size_t)w * nb + b) * bn;
    const T* bo = borig + (size_t)b * bn;
    for (int i0 = threadIdx.x; i0 < bn; i0 += GB * blockDim.x) {
      T v[GB];
      double u[GB];
#pragma unroll
      for (int k = 0; k < GB; k++) {
        const int i = i0 + k * blockDim.x;
        if (i < bn) v[k] = bo[i], u[k] = src[i];
      }
#pragma unroll
      for (int k = 0; k < GB; k++) {
        const int i = i0 + k * blockDim.x;
        if (i < bn) orig[i] = v[k], g[i] = u[k];
      }
    }
  }
  const uint8_t cb = c_choice[ci];
  const bool linear = cb & 1, seq1d = (cb >> 1) & 1;
  const double eb = st->eb, two_eb = st->two_eb, inv_two_eb = __ddiv_rn(1.0, two_eb);
  const int dims[3] = {b0, b1, b2};
  // the level's sub-steps, computed once per CTA into shared memory (a
  // per-thread table lived in local memory: 688 B of stack per thread that
  // the 98 KB shared-memory carve-out pushed out of L1)
  __shared__ SubStep s_ss[7];
  __shared__ int s_nss;
  if (threadIdx.x == 0) s_nss = block_steps(dims, level, seq1d, s_ss);
  __syncthreads();
  const int nss = s_nss;
  // leaf tables, one thread per sub-step (read after the first sub-step's barrier)
  if (threadIdx.x < nss) {
    const SubStep& S = s_ss[threadIdx.x];
    nleaf[threadIdx.x] = pw_leaves(S.count[0] * S.count[1] * S.count[2], lstart[threadIdx.x], llen[threadIdx.x]);
  }
  const int s = 1 << (level - 1);
  // One barrier per sub-step: it publishes the sub-step's reconstructions
  // (the next sub-step's stencil taps) and its |orig - pred| half.  The leaf
  // sums of sub-step t run before the barrier of t+1, which precedes the next
  // write of that half (sub-step t+2); the pairwise combines run at the end.
  for (int t = 0; t < nss; t++) {
    const SubStep S = s_ss[t];
    const int n = S.count[0] * S.count[1] * S.count[2];
    const int c12 = S.count[1] * S.count[2];
    const float r2 = 1.0f / (float)S.count[2], r12 = 1.0f / (float)c12;
    double* dd = diff + (t & 1) * (bn / 2);
    for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
      int c[3];
      const int q0 = qdiv(idx, c12, r12), rem = idx - q0 * c12, q1 = qdiv(rem, S.count[2], r2);
      c[2] = S.start[2] + (rem - q1 * S.count[2]) * S.step[2];
      c[1] = S.start[1] + q1 * S.step[1];
      c[0] = S.start[0] + q0 * S.step[0];
      const int lin = (c[0] * b1 + c[1]) * b2 + c[2];
      double pv[3] = {0.0, 0.0, 0.0};
      int ov[3] = {0, 0, 0};
#pragma unroll
      for (int i = 0; i < 3; i++) {
        if (i >= S.k) break;
        const int a = S.axes[i];
        const int ca = a == 0 ? c[0] : (a == 1 ? c[1] : c[2]), da = a == 0 ? b0 : (a == 1 ? b1 : b2);
        const int stp = (a == 0 ? b1 * b2 : (a == 1 ? b2 : 1)) * s;
        const int cls = classify(ca, da, s, linear);
        // samples at -3s, -1s, +1s, +3s; only in-range ones are used by cls
        const double v0 = ca >= 3 * s ? g[lin - 3 * stp] : 0.0;
        const double v1 = g[lin - stp];
        const double v2 = ca + s < da ? g[lin + stp] : 0.0;
        const double v3 = ca + 3 * s < da ? g[lin + 3 * stp] : 0.0;
        pv[i] = apply_stencil(cls, v0, v1, v2, v3);
        ov[i] = stencil_order(cls);
      }
      const double pred = S.k == 1 ? pv[0] : combine_axes(S.k, pv, ov);
      const double o = (double)orig[lin];
      dd[idx] = fabs(__dsub_rn(o, pred));
      double r;
      quantize_fast<sizeof(T) == 4>(o, pred, eb, two_eb, inv_two_eb, &r);
      g[lin] = r;
    }
    __syncthreads();
    // each leaf on 8 lanes: lane j owns numpy's accumulator r[j] (column j)
    const int nl = nleaf[t];
    for (int base = 0; base < nl; base += TUNE_THREADS / 8) {
      const int li = base + (int)(threadIdx.x >> 3), j = threadIdx.x & 7;
      double r = 0.0;
      int ln = 0;
      const double* a = dd;
      if (li < nl) {
        ln = llen[t][li];
        a = dd + lstart[t][li];
        if (ln >= 8) {
          r = a[j];
          for (int i = 8; i < ln - (ln % 8); i += 8) r = __dadd_rn(r, a[i + j]);
        }
      }
      double rr[8];
#pragma unroll
      for (int q = 0; q < 8; q++) rr[q] = __shfl_sync(0xffffffffu, r, (threadIdx.x & 24) + q);
      if (li < nl && j == 0) {
        double res;
        if (ln < 8) {
          res = 0.0;
          for (int i = 0; i < ln; i++) res = __dadd_rn(res, a[i]);
        } else {
          res = __dadd_rn(__dadd_rn(__dadd_rn(rr[0], rr[1]), __dadd_rn(rr[2], rr[3])),
                          __dadd_rn(__dadd_rn(rr[4], rr[5]), __dadd_rn(rr[6], rr[7])));
          for (int i = ln - (ln % 8); i < ln; i++) res = __dadd_rn(res, a[i]);
        }
        leafv[t][li] = res;
      }
    }
  }
  double* dst = trials + (size_t)(level & 1) * set_stride + ((size_t)ci * nb + b) * bn;
  for (int i = threadIdx.x; i < bn; i += blockDim.x) dst[i] = g[i];
  // the CTA that finishes the level last selects its config (no extra launch)
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    // the block's error: sum over sub-steps (in order) of numpy's pairwise sum
    double total = 0.0;
    for (int t = 0; t < nss; t++) {
      int cur = 0;
      total = __dadd_rn(total, pw_combine(s_ss[t].count[0] * s_ss[t].count[1] * s_ss[t].count[2], leafv[t], &cur));
    }
    berr[ci * nb + b] = total;
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // every CTA's block errors into shared memory with parallel loads (the
  // trial grid is no longer needed), then one warp runs the ordered sums
  const bool staged = (size_t)4 * nb * 8 <= (size_t)bn * (16 + sizeof(T));
  if (staged) {
    for (int i = threadIdx.x; i < 4 * nb; i += blockDim.x) tsm[i] = __ldcg(&berr[i]);
    __syncthreads();
  }
  if (threadIdx.x < 32) tune_select(nb, level, staged ? tsm : berr, staged, st, host_cfg, cond);
  if (threadIdx.x == 0) *done = 0;  // ready for the next level / call
}

static size_t tune_smem(const TunePlan& p, int prec) {
  return (size_t)p.bn * 8 * 2 + (size_t)p.bn * prec;
}

bool tune_supported(const TunePlan& p) { return tune_smem(p, 8) <= 200 * 1024; }

size_t tune_ws_bytes(const TunePlan& p) {
  // trials (two level sets of 4 configs) | compact block originals | level counter
  return (size_t)2 * 4 * p.nb * p.bn * 8 + (size_t)p.nb * p.bn * 8 + 64;
}

void launch_tune_level(const TunePlan& p, const void* field, int prec, const uint64_t dims[3],
                       const unsigned long long* origins, int level, double* trials, double* berr, DevState* st,
                       cudaStream_t s, int* launches, uint8_t* host_cfg, cudaGraphConditionalHandle cond) {
  const size_t smem = tune_smem(p, prec);
  double* borig = trials + (size_t)2 * 4 * p.nb * p.bn;
  unsigned* done = reinterpret_cast<unsigned*>(borig + (size_t)p.nb * p.bn);
  if (level == p.top) cudaMemsetAsync(done, 0, sizeof(unsigned), s);
  // the attribute is process-wide: set once to the largest plan tune_supported
  // admits (a per-launch value raced between threads compressing different
  // shapes, failing the other thread's launch)
  static const bool attr = [] {
    cudaFuncSetAttribute(k_tune_level<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_tune_level<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return true;
  }();
  (void)attr;
  if (prec == 4) {
    k_tune_level<float><<<4 * p.nb, TUNE_THREADS, smem, s>>>((const float*)field, dims[1], dims[2], origins, p.nb,
                                                             p.shape[0], p.shape[1], p.shape[2], p.top, level, trials,
                                                             berr, st, reinterpret_cast<float*>(borig), done,
                                                             host_cfg, cond);
  } else {
    k_tune_level<double><<<4 * p.nb, TUNE_THREADS, smem, s>>>((const double*)field, dims[1], dims[2], origins, p.nb,
                                                              p.shape[0], p.shape[1], p.shape[2], p.top, level,
                                                              trials, berr, st, borig, done, host_cfg, cond);
  }
  (*launches)++;
}

// ------------------------------------------------ whole-field (thin) tuner
// plan_blocks returns the whole field as the single sample block when its
// smallest non-degenerate dim is < 17 (tuning.py:74-75).  Blocks too large for
// shared memory run here on global-memory grids: one launch per sub-step, the
// |orig - pred| array of each sub-step materialised in C order, numpy's
// pairwise sum over it (parallel leaves, recursive combine), and the same
// argmin / winner hand-over as the tiled path (nb = 1, so Python's sum over
// blocks is the single total).

struct HSub {  // host copy of one sub-step
  int start[3], step[3], count[3];
  int axes[3];
  int k;
};

static int host_steps(const int d[3], int level, bool seq1d, HSub* out) {
  const int s = 1 << (level - 1);
  int n = 0;
  if (seq1d) {
    int o[3] = {0, 1, 2};
    for (int i = 0; i < 3; i++)
      for (int j = i + 1; j < 3; j++)
        if (d[o[j]] > d[o[i]] || (d[o[j]] == d[o[i]] && o[j] < o[i])) std::swap(o[i], o[j]);
    for (int k = 0; k < 3; k++) {
      const int a = o[k];
      HSub ss;
      for (int j = 0; j < 3; j++) {
        bool earlier = false;
        for (int m = 0; m < k; m++) earlier |= o[m] == j;
        ss.start[j] = j == a ? s : 0;
        ss.step[j] = j == a ? 2 * s : (earlier ? s : 2 * s);
        ss.count[j] = d[j] > ss.start[j] ? (d[j] - ss.start[j] + ss.step[j] - 1) / ss.step[j] : 0;
      }
      ss.axes[0] = a;
      ss.k = 1;
      if (ss.count[a] > 0) out[n++] = ss;
    }
  } else {
    const int sets[7] = {1, 2, 4, 3, 5, 6, 7};
    for (int t = 0; t < 7; t++) {
      HSub ss;
      bool empty = false;
      ss.k = 0;
      for (int j = 0; j < 3; j++) {
        const bool odd = (sets[t] >> j) & 1;
        ss.start[j] = odd ? s : 0;
        ss.step[j] = 2 * s;
        ss.count[j] = d[j] > ss.start[j] ? (d[j] - ss.start[j] + ss.step[j] - 1) / ss.step[j] : 0;
        if (odd) {
          if (ss.count[j] == 0) empty = true;
          ss.axes[ss.k++] = j;
        }
      }
      if (!empty) out[n++] = ss;
    }
  }
  return n;
}

template <typename T>
__global__ void k_tg_init(const T* __restrict__ f, unsigned long long n, double* g) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    g[i] = (double)f[i];
}

__global__ void k_tg_copy(const double* __restrict__ src_base, unsigned long long stride, const DevState* st,
                          int level, unsigned long long n, double* dst) {
  const double* src = src_base + (size_t)st->tune_winner[level - 1] * stride;  // winner of `level`
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

template <typename T>
__global__ void k_tg_step(const T* __restrict__ f, HSub S, int d0, int d1, int d2, int level, int linear,
                          double* g, double* diff, DevState* st) {
  const unsigned long long n = (unsigned long long)S.count[0] * S.count[1] * S.count[2];
  const int s = 1 << (level - 1);
  const int dims[3] = {d0, d1, d2};
  const double eb = st->eb, two_eb = st->two_eb, inv_two_eb = __ddiv_rn(1.0, two_eb);
  for (unsigned long long idx = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (unsigned long long)gridDim.x * blockDim.x) {
    long long c[3];
    c[2] = S.start[2] + (long long)(idx % S.count[2]) * S.step[2];
    c[1] = S.start[1] + (long long)((idx / S.count[2]) % S.count[1]) * S.step[1];
    c[0] = S.start[0] + (long long)(idx / ((unsigned long long)S.count[2] * S.count[1])) * S.step[0];
    const long long lin = (c[0] * d1 + c[1]) * d2 + c[2];
    double pv[3];
    int ov[3];
    for (int i = 0; i < S.k; i++) {
      const int a = S.axes[i];
      const long long stp = (a == 0 ? (long long)d1 * d2 : (a == 1 ? (long long)d2 : 1ll)) * s;
      const int cls = classify(c[a], dims[a], s, linear);
      const double v0 = c[a] >= 3 * s ? g[lin - 3 * stp] : 0.0;
      const double v1 = g[lin - stp];
      const double v2 = c[a] + s < dims[a] ? g[lin + stp] : 0.0;
      const double v3 = c[a] + 3 * s < dims[a] ? g[lin + 3 * stp] : 0.0;
      pv[i] = apply_stencil(cls, v0, v1, v2, v3);
      ov[i] = stencil_order(cls);
    }
    const double pred = S.k == 1 ? pv[0] : combine_axes(S.k, pv, ov);
    const double o = (double)f[lin];
    diff[idx] = fabs(__dsub_rn(o, pred));
    double r;
    quantize_fast<sizeof(T) == 4>(o, pred, eb, two_eb, inv_two_eb, &r);
    g[lin] = r;
  }
}

__global__ void k_tg_leaves(const double* __restrict__ diff, const int2* __restrict__ leaves, int nleaf,
                            double* leafsum) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nleaf; i += gridDim.x * blockDim.x)
    leafsum[i] = pw_leaf(diff + leaves[i].x, leaves[i].y);
}

// total += pairwise(n) from the leaf sums (recursion of numpy's pairwise_sum)
__device__ double tg_combine(unsigned long long n, const double* leaf, unsigned long long* cur) {
  if (n <= 128) return leaf[(*cur)++];
  unsigned long long n2 = n / 2;
  n2 -= n2 % 8;
  const double a = tg_combine(n2, leaf, cur);
  const double b = tg_combine(n - n2, leaf, cur);
  return __dadd_rn(a, b);
}

__global__ void k_tg_accum(unsigned long long n, const double* leafsum, double* total) {
  unsigned long long cur = 0;
  *total = __dadd_rn(*total, tg_combine(n, leafsum, &cur));
}

// tuning.py:135-140 for a single block: errs[c] = 0 + total[c]
__global__ void k_tg_select(int level, double* totals, DevState* st) {
  int best = 0;
  for (int i = 0; i < 4; i++) {
    const double e = __dadd_rn(0.0, totals[i]);
    st->tune_errs[(level - 1) * 4 + i] = e;
    if (i > 0 && e < __dadd_rn(0.0, totals[best])) best = i;
  }
  st->tune_winner[level - 1] = best;
  st->cfg[level - 1] = c_choice[best];
  for (int i = 0; i < 4; i++) totals[i] = 0.0;
}

size_t tune_global_bytes(unsigned long long bn) { return bn * 8 * 6 + 4096 * 16 + (bn / 32 + 64) * 16; }

// scratch: [state | 4 trials | diff | leaf sums | totals]
int launch_tune_global(const void* field, int prec, const uint64_t dims[3], int top, uint8_t* scratch,
                       DevState* st, cudaStream_t s, int* launches,
                       int (*upload)(void* ctx, void* dev, const void* src, size_t n), void* up_ctx) {
  const unsigned long long bn = dims[0] * dims[1] * dims[2];
  double* state = reinterpret_cast<double*>(scratch);
  double* trial = state + bn;
  double* diff = trial + 4 * bn;
  double* leafsum = diff + bn;
  double* totals = leafsum + (bn / 32 + 64);
  int2* leaves = reinterpret_cast<int2*>(totals + 8);
  const int d[3] = {(int)dims[0], (int)dims[1], (int)dims[2]};
  const unsigned grid = 148 * 8;
  if (prec == 4)
    k_tg_init<float><<<grid, 256, 0, s>>>((const float*)field, bn, state);
  else
    k_tg_init<double><<<grid, 256, 0, s>>>((const double*)field, bn, state);
  (*launches)++;
  cudaMemsetAsync(totals, 0, 8 * sizeof(double), s);
  for (int level = top; level >= 1; level--) {
    for (int ci = 0; ci < 4; ci++) {
      const uint8_t cb = ci == 0 ? 0 : (ci == 1 ? 2 : (ci == 2 ? 1 : 3));
      double* g = trial + (size_t)ci * bn;
      cudaMemcpyAsync(g, state, bn * 8, cudaMemcpyDeviceToDevice, s);
      HSub ss[7];
      const int nss = host_steps(d, level, (cb >> 1) & 1, ss);
      for (int t = 0; t < nss; t++) {
        const unsigned long long n = (unsigned long long)ss[t].count[0] * ss[t].count[1] * ss[t].count[2];
        if (prec == 4)
          k_tg_step<float><<<grid, 256, 0, s>>>((const float*)field, ss[t], d[0], d[1], d[2], level, cb & 1, g,
                                                diff, st);
        else
          k_tg_step<double><<<grid, 256, 0, s>>>((const double*)field, ss[t], d[0], d[1], d[2], level, cb & 1, g,
                                                 diff, st);
        // leaves of the recursion in order (host, depends on n only)
        std::vector<int2> lv;
        std::vector<std::pair<unsigned long long, unsigned long long>> stk{{0ull, n}};
        while (!stk.empty()) {
          auto [s0, n0] = stk.back();
          stk.pop_back();
          if (n0 <= 128) {
            lv.push_back(make_int2((int)s0, (int)n0));
          } else {
            unsigned long long n2 = n0 / 2;
            n2 -= n2 % 8;
            stk.push_back({s0 + n2, n0 - n2});
            stk.push_back({s0, n2});
          }
        }
        const int rc = upload(up_ctx, leaves, lv.data(), lv.size() * sizeof(int2));
        if (rc) return rc;
        k_tg_leaves<<<(unsigned)((lv.size() + 255) / 256), 256, 0, s>>>(diff, leaves, (int)lv.size(), leafsum);
        k_tg_accum<<<1, 1, 0, s>>>(n, leafsum, totals + ci);
        *launches += 3;
        cudaStreamSynchronize(s);  // the leaf table in pinned memory is reused by the next sub-step
      }
    }
    k_tg_select<<<1, 1, 0, s>>>(level, totals, st);
    k_tg_copy<<<grid, 256, 0, s>>>(trial, bn, st, level, bn, state);
    *launches += 2;
  }
  return 0;
}

}  // namespace hb
