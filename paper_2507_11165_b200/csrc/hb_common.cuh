// hb_common.cuh -- shared types and device utilities for the B200 hibound path.
//
// All kernels are written for sm_100a (B200): 148 SMs, 32-wide warps, up to
// 227 KB of shared memory per CTA.  The path is HBM/latency bound integer and
// f64 work, so no tensor cores are involved; see DESIGN.md for the roofline.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hibound_b200.h"

namespace hb {

constexpr int kSMs = 148;

// error bits accumulated on the device; the host maps them to HB_E* codes
enum : uint32_t {
  F_NONFINITE = 1u << 0,   // FieldError (field.py:51-52)
  F_DEGENERATE = 1u << 1,  // DegenerateBoundError (field.py:141, predictor.py:333)
  F_ARCHIVE = 1u << 2,     // ArchiveError
  F_STAGE = 1u << 3,       // StageError
  F_CAPACITY = 1u << 4,    // internal buffer too small (bug guard)
  F_ORPHAN = 1u << 5,      // code 0 without outlier (predictor.py:402-405) -> ArchiveError
  F_ZEROCOUNT = 1u << 6,   // #code0 != outlier count (archive.py:168-169) -> ArchiveError
  F_UNSUPPORTED = 1u << 7,
};

// Reducer (RRE/RZE) bookkeeping for one nesting level (stages.py:165-221)
struct BmLevel {
  unsigned long long orig;    // bytes of input to this level
  unsigned long long nwords;  // padded word count
  unsigned long long bm_len;  // raw bitmap bytes
  unsigned long long kept;    // kept words
  unsigned long long rec_len; // encoded record length (after nesting decision)
  int flag;                   // bitmap section is a nested record
  int active;                 // level was computed
  unsigned long long tiles_done;  // k_reduce_tail: completed tiles of this level
};

struct BmState {
  BmLevel lv[4];
};

// Device-resident state of one compress/decompress call.  Everything that
// decides buffer offsets lives here so the whole call stays asynchronous and
// graph-capturable; the host reads it back once at the end.
struct DevState {
  double eb, two_eb;
  unsigned long long vmin_bits, vmax_bits;  // order-preserving encodings
  uint32_t flags;
  uint32_t detail;
  uint8_t cfg[4];
  int tune_winner[4];
  double tune_errs[16];
  unsigned long long hist[256];
  unsigned long long outlier_count;
  unsigned long long zero_count;
  // Huffman (stages.py:246-329)
  unsigned long long hf_nbits;
  unsigned long long hf_rec_len;
  unsigned long long hf_code[256];
  uint8_t hf_len[256];
  // reducer chains: [0] RRE4 over HF (CR), [1] RZE1 over TCMS8 (CR), [2] RRE1 over BIT1 (TP)
  BmState bm[3];
  unsigned long long tcms_rec_len;
  unsigned long long stream_len;
  unsigned long long seq_len;
  unsigned long long archive_len;
  int escape;
  // decompress
  unsigned long long hd_nsym, hd_nbits;
  int hd_maxlen;
  unsigned long long tickets[16];
  unsigned long long scratch[32];
  double inv_two_eb;  // __ddiv_rn(1.0, two_eb), set with eb (one IEEE division per call, not per block)
};

__device__ __forceinline__ void raise_flag(DevState* st, uint32_t f, uint32_t detail = 0) {
  atomicOr(&st->flags, f);
  if (detail) atomicCAS(&st->detail, 0u, detail);
}

// ------------------------------------------------------------ scans

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v += n;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan; returns the exclusive prefix for this thread and
// the block total in *total.  `sh` must hold >= 33 elements.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* sh, T* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) sh[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T s = lane < nw ? sh[lane] : T(0);
    T si = warp_incl_scan(s);
    if (lane < nw) sh[lane] = si - s;
    if (lane == nw - 1) sh[32] = si;
  }
  __syncthreads();
  T res = sh[wid] + inc - v;
  *total = sh[32];
  __syncthreads();
  return res;
}

// ------------------------------------------------- decoupled look-back
// status word: bits 62-63 flag (1 = aggregate, 2 = inclusive prefix), 0-61 value
constexpr unsigned long long LB_AGG = 1ull << 62, LB_INC = 2ull << 62, LB_MASK = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
  return *(volatile const unsigned long long*)p;
}

// Called by ONE thread of tile `t`; returns the exclusive prefix of tile t.
__device__ __forceinline__ unsigned long long lookback(unsigned long long* status, unsigned long long t,
                                                       unsigned long long agg) {
  if (t == 0) {
    __threadfence();
    atomicExch(&status[0], LB_INC | agg);
    return 0;
  }
  atomicExch(&status[t], LB_AGG | agg);
  __threadfence();
  unsigned long long excl = 0;
  long long j = (long long)t - 1;
  while (true) {
    unsigned long long s = ld_volatile(&status[j]);
    if ((s >> 62) == 0) continue;
    excl += s & LB_MASK;
    if ((s >> 62) == 2) break;
    j--;
  }
  __threadfence();
  atomicExch(&status[t], LB_INC | (excl + agg));
  return excl;
}

// Warp-parallel variant: called by all 32 lanes of ONE warp of tile `t`;
// inspects 32 predecessors per round (one status word per lane), so the walk
// costs ~t/32 L2 round trips even when no predecessor has its inclusive
// prefix yet.  Returns the exclusive prefix on every lane.
__device__ __forceinline__ unsigned long long lookback_warp(unsigned long long* status, unsigned long long t,
                                                            unsigned long long agg) {
  const int lane = threadIdx.x & 31;
  if (t == 0) {
    if (lane == 0) {
      __threadfence();
      atomicExch(&status[0], LB_INC | agg);
    }
    return 0;
  }
  if (lane == 0) atomicExch(&status[t], LB_AGG | agg);
  unsigned long long excl = 0;
  long long base = (long long)t - 1;
  while (true) {
    const long long j = base - lane;
    unsigned long long s = j >= 0 ? ld_volatile(&status[j]) : LB_INC;
    while (__any_sync(0xffffffffu, (s >> 62) == 0))
      if ((s >> 62) == 0) s = ld_volatile(&status[j]);
    const unsigned inc = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    if (inc) {
      const int first = __ffs(inc) - 1;
      excl += warp_sum<unsigned long long>(lane <= first ? (s & LB_MASK) : 0ull);
      break;
    }
    excl += warp_sum<unsigned long long>(s & LB_MASK);
    base -= 32;
  }
  if (lane == 0) {
    __threadfence();
    atomicExch(&status[t], LB_INC | (excl + agg));
  }
  return excl;
}

// The wait half of lookback_warp for a tile that already published its
// aggregate (t > 0): whole warp, returns the exclusive prefix and publishes
// the inclusive one.
__device__ __forceinline__ unsigned long long lookback_wait(unsigned long long* status, unsigned long long t,
                                                            unsigned long long agg) {
  const int lane = threadIdx.x & 31;
  unsigned long long excl = 0;
  long long base = (long long)t - 1;
  while (true) {
    const long long j = base - lane;
    unsigned long long s = j >= 0 ? ld_volatile(&status[j]) : LB_INC;
    while (__any_sync(0xffffffffu, (s >> 62) == 0)) {
      __nanosleep(32);  // back off: spinning warps steal issue slots from the producers
      if ((s >> 62) == 0) s = ld_volatile(&status[j]);
    }
    const unsigned inc = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    if (inc) {
      const int first = __ffs(inc) - 1;
      excl += warp_sum<unsigned long long>(lane <= first ? (s & LB_MASK) : 0ull);
      break;
    }
    excl += warp_sum<unsigned long long>(s & LB_MASK);
    base -= 32;
  }
  if (lane == 0) {
    __threadfence();
    atomicExch(&status[t], LB_INC | (excl + agg));
  }
  return excl;
}

// ordered encodings for float min/max atomics
__device__ __forceinline__ unsigned long long ord_bits(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | (1ull << 63));
}
__device__ __forceinline__ double from_ord_bits(unsigned long long o) {
  unsigned long long b = (o >> 63) ? (o & ~(1ull << 63)) : ~o;
  return __longlong_as_double((long long)b);
}

__host__ __device__ __forceinline__ unsigned long long cdiv(unsigned long long a, unsigned long long b) {
  return (a + b - 1) / b;
}

}  // namespace hb
