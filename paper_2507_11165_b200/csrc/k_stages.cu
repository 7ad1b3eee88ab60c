// k_stages.cu -- the lossless stages of both pipelines on the GPU
// (stages.py:94-435): bitmap reducers RRE/RZE with <= 3 nested RRE1 bitmaps,
// TCMS zigzag, BIT bit-plane transpose and canonical Huffman, encode and
// decode.
//
// Every data-dependent size stays on the device (DevState / BmState), so a
// whole compress or decompress is one asynchronous launch sequence.  Kernels
// whose work depends on a device-side size are persistent: grid = a few CTAs
// per SM, tiles handed out by an atomic ticket, and a decoupled look-back
// (hb_common.cuh) provides each tile's exclusive prefix (kept words, code
// bits, decoded symbols) in a single pass.
#include <cuda_runtime.h>
#include <stdio.h>

#include <vector>
#include <cstdio>
#include <cstdlib>

#include "hb_common.cuh"
#include "hb_kernels.h"

namespace hb {

constexpr int RD_THREADS = 256;
constexpr int RD_TILE = RD_THREADS * 32;  // words per tile (8 warps x 32 steps x 32 lanes)
constexpr unsigned PERSIST_CTAS = 148 * 4;

__device__ __forceinline__ uint64_t ld_bytes(const uint8_t* p, int n) {
  uint64_t v = 0;
  for (int i = 0; i < n; i++) v |= (uint64_t)p[i] << (8 * i);
  return v;
}
__device__ __forceinline__ void st_bytes(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; i++) p[i] = (uint8_t)(v >> (8 * i));
}
__device__ __forceinline__ uint64_t zz(uint64_t u, int w) {  // stages.py:106-107
  const int top = 8 * w - 1;
  const uint64_t m = w == 8 ? ~0ull : ((1ull << (8 * w)) - 1);
  return ((u << 1) ^ (0ull - (u >> top))) & m;
}
__device__ __forceinline__ uint64_t unzz(uint64_t u, int w) {  // stages.py:117
  const uint64_t m = w == 8 ? ~0ull : ((1ull << (8 * w)) - 1);
  return ((u >> 1) ^ (0ull - (u & 1))) & m;
}
// byte-wise zigzag of 8 packed bytes (TCMS w=1, SWAR)
__device__ __forceinline__ uint64_t zz8x1(uint64_t u) {
  const uint64_t hi = (u >> 7) & 0x0101010101010101ull;
  return ((u << 1) & 0xFEFEFEFEFEFEFEFEull) ^ (hi * 0xFFull);
}
__device__ __forceinline__ uint64_t unzz8x1(uint64_t u) {
  const uint64_t lo = u & 0x0101010101010101ull;
  return ((u >> 1) & 0x7F7F7F7F7F7F7F7Full) ^ (lo * 0xFFull);
}
// plane byte k of an 8-byte BIT1 tile held little-endian in g (stages.py:139-140)
__device__ __forceinline__ uint8_t bit_plane(uint64_t g, int k) {
  return (uint8_t)((((g >> (7 - k)) & 0x0101010101010101ull) * 0x8040201008040201ull) >> 56);
}

// ------------------------------------------------------------- sources
// A reducer source yields little-endian words of `width` bytes of a (virtual)
// byte record, zero padded past its length.

struct MemSrc {  // plain bytes
  const uint8_t* p;
  unsigned long long len;
  int w;
  __device__ uint64_t word(unsigned long long i) const {
    const unsigned long long o = i * w;
    if (o + w <= len) {
      if (w == 4 && !((uintptr_t)(p + o) & 3)) return *reinterpret_cast<const uint32_t*>(p + o);
      if (w == 8 && !((uintptr_t)(p + o) & 7)) return *reinterpret_cast<const uint64_t*>(p + o);
      return ld_bytes(p + o, w);
    }
    uint64_t v = 0;
    for (int k = 0; k < w; k++)
      if (o + k < len) v |= (uint64_t)p[o + k] << (8 * k);
    return v;
  }
  // words [i0, i0+32) (i0 % 32 == 0), zero past the end
  template <typename T>
  __device__ void load32(unsigned long long i0, T* v) const {
    const unsigned long long o = i0 * w;
    if (o + 32ull * w <= len && !((uintptr_t)(p + o) & 15)) {
      const uint4* q = reinterpret_cast<const uint4*>(p + o);
      if (w == 1) {
        const uint4 a = q[0], b = q[1];
        const uint32_t u[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int j = 0; j < 32; j++) v[j] = (u[j >> 2] >> (8 * (j & 3))) & 0xFF;
        return;
      }
      if (w == 4) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const uint4 a = q[k];
          v[4 * k] = a.x, v[4 * k + 1] = a.y, v[4 * k + 2] = a.z, v[4 * k + 3] = a.w;
        }
        return;
      }
    }
#pragma unroll
    for (int j = 0; j < 32; j++) v[j] = (T)word(i0 + j);
  }
};

// TCMS(width tw) record of a byte buffer, read as bytes (feeds RZE1 in CR)
struct TcmsSrc {
  const uint8_t* p;  // underlying data
  unsigned long long n;  // underlying length
  int tw;
  __device__ uint64_t word(unsigned long long j) const {  // width-1 words
    if (j < 10) {
      if (j == 0) return 4;
      if (j == 1) return (uint64_t)tw;
      return (n >> (8 * (j - 2))) & 0xFF;
    }
    const unsigned long long q = (j - 10) / tw, r = (j - 10) % tw;
    const unsigned long long o = q * tw;
    uint64_t u = 0;
    if (o + tw <= n && tw == 8 && !((uintptr_t)(p + o) & 7))
      u = *reinterpret_cast<const uint64_t*>(p + o);
    else
      for (int k = 0; k < tw; k++)
        if (o + k < n) u |= (uint64_t)p[o + k] << (8 * k);
    return (zz(u, tw) >> (8 * r)) & 0xFF;
  }
  __device__ unsigned long long len() const { return 10 + cdiv(n, tw) * tw; }
  template <typename T>
  __device__ void load32(unsigned long long i0, T* v) const {
    if (tw == 8 && i0 >= 32) {  // bytes [i0, i0+32) = words (i0-10)/8 .. +4 of zz(data)
      const unsigned long long q0 = (i0 - 10) >> 3;  // (i0-10) % 8 == 6
      uint64_t z[5];
#pragma unroll
      for (int k = 0; k < 5; k++) {
        const unsigned long long o = (q0 + k) * 8;
        uint64_t u = 0;
        if (o + 8 <= n)
          u = *reinterpret_cast<const uint64_t*>(p + o);
        else
          for (int b = 0; b < 8; b++)
            if (o + b < n) u |= (uint64_t)p[o + b] << (8 * b);
        z[k] = o < n ? zz(u, 8) : 0;
      }
#pragma unroll
      for (int j = 0; j < 32; j++) {
        const int b = 6 + j;  // byte position from word q0
        v[j] = (T)((z[b >> 3] >> (8 * (b & 7))) & 0xFF);
      }
      return;
    }
#pragma unroll
    for (int j = 0; j < 32; j++) v[j] = (T)word(i0 + j);
  }
};

// BIT1(TCMS1(seq)) record bytes (feeds RRE1 in TP): stages.py:430-431
struct TpSrc {
  const uint8_t* seq;
  unsigned long long n;
  // byte m of the TCMS1 record: header [4,1,n] then zigzag(seq), 0 past end
  __device__ uint64_t tcms_group(unsigned long long t) const {  // bytes [8t, 8t+8)
    uint64_t g = 0;
    if (t <= 1) {
      for (int k = 0; k < 8; k++) {
        const unsigned long long m = 8 * t + k;
        uint64_t b;
        if (m == 0)
          b = 4;
        else if (m == 1)
          b = 1;
        else if (m < 10)
          b = (n >> (8 * (m - 2))) & 0xFF;
        else
          b = (m - 10 < n) ? (uint64_t)seq[m - 10] : 0;
        g |= b << (8 * k);
      }
      return t == 1 ? (g & 0xFFFFull) | (zz8x1(g & ~0xFFFFull)) : g;
    }
    const unsigned long long o = 8 * t - 10;  // seq offset, o % 8 == 6
    if (o + 8 <= n) {
      const uint64_t* w = reinterpret_cast<const uint64_t*>(seq + (o - 6));
      g = (w[0] >> 48) | (w[1] << 16);
    } else {
      for (int k = 0; k < 8; k++)
        if (o + k < n) g |= (uint64_t)seq[o + k] << (8 * k);
    }
    return zz8x1(g);
  }
  __device__ uint64_t word(unsigned long long j) const {
    if (j < 10) {
      if (j == 0) return 5;
      if (j == 1) return 1;
      return ((n + 10) >> (8 * (j - 2))) & 0xFF;
    }
    const unsigned long long t = (j - 10) >> 3;
    return bit_plane(tcms_group(t), (int)((j - 10) & 7));
  }
  __device__ unsigned long long len() const { return 10 + cdiv(n + 10, 8) * 8; }
  template <typename T>
  __device__ void load32(unsigned long long i0, T* v) const {
    if (i0 >= 32) {  // record bytes [i0, i0+32) = planes of tiles (i0-10)/8 .. +4
      const unsigned long long t0 = (i0 - 10) >> 3;  // (i0-10) % 8 == 6
      uint64_t g[5];
#pragma unroll
      for (int k = 0; k < 5; k++) g[k] = tcms_group(t0 + k);
#pragma unroll
      for (int j = 0; j < 32; j++) {
        const int b = 6 + j;
        v[j] = (T)bit_plane(g[b >> 3], b & 7);
      }
      return;
    }
#pragma unroll
    for (int j = 0; j < 32; j++) v[j] = (T)word(i0 + j);
  }
};

// ------------------------------------------------------- reducer encode
// stages.py:165-184.  stage 2 = RRE (keep w[i] != w[i-1]), 3 = RZE (w != 0).

// WT: register word type (32-bit for widths <= 4: half the registers).
// stg: shared staging for the tile's kept words (widths <= 4), written out
// with coalesced stores once the tile's base is known; null = direct stores.
// ST / W: compile-time stage / width (0 = take the runtime argument); the
// chains the compressor runs are instantiated with both fixed, so each kernel
// holds only its own width's load/store code.
// done != null: each completed tile (all its stores fenced) bumps *done, and
// the CTA holding the last tile also publishes the level's sizes (k_reduce_tail).
template <class Src, typename WT, int ST = 0, int W = 0>
__device__ void reduce_tiles(const Src& src, unsigned long long nw, int stage_rt, int width_rt, uint8_t* bitmap,
                             uint8_t* payload, unsigned long long* lb, BmLevel* lv, uint8_t* stg,
                             unsigned long long* done = nullptr) {
  const int stage = ST ? ST : stage_rt;
  const int width = W ? W : width_rt;
  __shared__ unsigned long long sh[33];
  __shared__ unsigned long long tile_sh, base_sh;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned long long ntiles = cdiv(nw, RD_TILE);
  unsigned long long* ticket = lb;
  unsigned long long* status = lb + 1;
  for (;;) {
    if (threadIdx.x == 0) tile_sh = atomicAdd(ticket, 1ull);
    __syncthreads();
    const unsigned long long tile = tile_sh;
    if (tile >= ntiles) break;
    // each lane owns 32 consecutive words: independent loads, one bitmap word
    const unsigned long long i0 = tile * RD_TILE + (unsigned long long)wid * 1024 + (unsigned long long)lane * 32;
    WT v[32];
    uint32_t mask = 0;
    if (i0 < nw) {
      src.load32(i0, v);
      WT prev = 0;
      if (stage == 2) prev = i0 > 0 ? (WT)src.word(i0 - 1) : (WT)~v[0];
#pragma unroll
      for (int j = 0; j < 32; j++) {
        const bool in = i0 + j < nw;
        const bool keep = in && (stage == 2 ? (i0 + j == 0 || v[j] != (j ? v[j - 1] : prev)) : v[j] != 0);
        mask |= (uint32_t)keep << (31 - j);  // word i0 at the MSB (np.packbits order)
      }
      *reinterpret_cast<uint32_t*>(bitmap + i0 / 8) = __byte_perm(mask, 0, 0x0123);
    }
    const unsigned c = __popc(mask);
    const unsigned incl = warp_incl_scan<unsigned>(c);
    unsigned long long total;
    unsigned long long wex = block_excl_scan<unsigned long long>(lane == 31 ? incl : 0u, sh, &total);
    wex = __shfl_sync(0xffffffffu, wex, 31);
    if (threadIdx.x < 32) {
      const unsigned long long ex_ = lookback_warp(status, tile, total);
      if (threadIdx.x == 0) base_sh = ex_;
    }
    if (stg) {
      // kept words into shared memory at their tile-local rank
      unsigned d = (unsigned)(wex + incl - c);
      if (mask) {
#pragma unroll
        for (int j = 0; j < 32; j++) {
          if ((mask >> (31 - j)) & 1) {
            if (width == 1)
              stg[d] = (uint8_t)v[j];
            else if (width == 2)
              reinterpret_cast<uint16_t*>(stg)[d] = (uint16_t)v[j];
            else
              reinterpret_cast<uint32_t*>(stg)[d] = (uint32_t)v[j];
            d++;
          }
        }
      }
      __syncthreads();
      const unsigned long long base = base_sh;
      const unsigned tot = (unsigned)total;
      if (width == 4) {
        uint32_t* o = reinterpret_cast<uint32_t*>(payload) + base;
        for (unsigned i = threadIdx.x; i < tot; i += blockDim.x) o[i] = reinterpret_cast<const uint32_t*>(stg)[i];
      } else if (width == 2) {
        uint16_t* o = reinterpret_cast<uint16_t*>(payload) + base;
        for (unsigned i = threadIdx.x; i < tot; i += blockDim.x) o[i] = reinterpret_cast<const uint16_t*>(stg)[i];
      } else {
        uint8_t* o = payload + base;
        for (unsigned i = threadIdx.x; i < tot; i += blockDim.x) o[i] = stg[i];
      }
    } else {
      __syncthreads();
      unsigned long long dst = base_sh + wex + incl - c;
      if (mask) {
#pragma unroll
        for (int j = 0; j < 32; j++) {
          if ((mask >> (31 - j)) & 1) {
            uint8_t* p = payload + dst * width;
            if (width == 1)
              *p = (uint8_t)v[j];
            else if (width == 2)
              *reinterpret_cast<uint16_t*>(p) = (uint16_t)v[j];
            else if (width == 4)
              *reinterpret_cast<uint32_t*>(p) = (uint32_t)v[j];
            else
              *reinterpret_cast<uint64_t*>(p) = (uint64_t)v[j];
            dst++;
          }
        }
      }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      lv->kept = base_sh + total;
      if (done) {
        lv->orig = nw;
        lv->nwords = nw;
        lv->bm_len = cdiv(nw, 8);
        lv->active = 1;
      }
    }
    if (done) __threadfence();
    __syncthreads();
    if (done && threadIdx.x == 0) atomicAdd(done, 1ull);
  }
}

// level 0 of a chain over a typed source
template <class Src, typename WT, int ST = 0, int W = 0>
__global__ void __launch_bounds__(RD_THREADS, sizeof(WT) == 4 ? 4 : 1)
    k_reduce0(Src src, const unsigned long long* len_dev, int stage_rt, int width_rt, BmState* bm, uint8_t* bitmap,
              uint8_t* payload, unsigned long long* lb) {
  extern __shared__ __align__(16) uint8_t rd_stg[];
  const int stage = ST ? ST : stage_rt;
  const int width = W ? W : width_rt;
  Src s2 = src;
  unsigned long long len;
  if constexpr (sizeof(Src) == sizeof(MemSrc) && __is_same(Src, MemSrc)) {
    len = *len_dev;
    s2.len = len;
    if constexpr (W != 0) s2.w = W;
  } else if constexpr (__is_same(Src, TcmsSrc)) {
    s2.n = *len_dev;
    if constexpr (W != 0) s2.tw = 8;  // the CR chain's TCMS8 record
    len = s2.len();
  } else {
    s2.n = *len_dev;
    len = s2.len();
  }
  const unsigned long long nw = cdiv(len, (unsigned long long)width);
  BmLevel* lv = &bm->lv[0];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    lv->orig = len;
    lv->nwords = nw;
    lv->bm_len = cdiv(nw, 8);
    lv->active = 1;
  }
  reduce_tiles<Src, WT, ST, W>(s2, nw, stage, width, bitmap, payload, lb, lv, width <= 4 ? rd_stg : nullptr);
}

// nested RRE1 over the previous level's bitmap (stages.py:178-181)
__global__ void __launch_bounds__(RD_THREADS, 4)
    k_reduce_nested(int level, BmState* bm, const uint8_t* prev_bitmap, uint8_t* bitmap, uint8_t* payload,
                    unsigned long long* lb) {
  __shared__ __align__(16) uint8_t stg[RD_TILE];
  const BmLevel* p = &bm->lv[level - 1];
  if (!p->active || p->bm_len <= 19) return;
  MemSrc src{prev_bitmap, p->bm_len, 1};
  const unsigned long long nw = p->bm_len;
  BmLevel* lv = &bm->lv[level];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    lv->orig = nw;
    lv->nwords = nw;
    lv->bm_len = cdiv(nw, 8);
    lv->active = 1;
  }
  reduce_tiles<MemSrc, uint32_t, 2, 1>(src, nw, 2, 1, bitmap, payload, lb, lv, stg);
}

// dst[0..n) = src[0..n) for a 4-byte aligned src and any dst: aligned 32-bit
// stores built with funnel shifts from two aligned source words; the few
// unaligned head bytes go byte-wise.  Grid-stride over (tid, nth).
__device__ __forceinline__ void copy_to_unaligned(uint8_t* dst, const uint8_t* src, unsigned long long n,
                                                  unsigned long long tid, unsigned long long nth) {
  const unsigned head = (unsigned)((4 - ((uintptr_t)dst & 3)) & 3);
  const unsigned long long h = head < n ? head : n;
  for (unsigned long long i = tid; i < h; i += nth) dst[i] = src[i];
  if (n <= h) return;
  uint32_t* d32 = reinterpret_cast<uint32_t*>(dst + h);
  const unsigned long long nw = (n - h) >> 2;
  const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);  // aligned
  const int sh = (int)(h & 3) * 8;  // source byte offset of d32[0] is h
  for (unsigned long long i = tid; i < nw; i += nth) {
    const unsigned long long b = h + 4 * i;  // source byte index
    const uint32_t lo = s32[b >> 2];
    const uint32_t hi = sh ? s32[(b >> 2) + 1] : 0u;
    d32[i] = sh ? __funnelshift_r(lo, hi, sh) : lo;
  }
  for (unsigned long long i = h + 4 * nw + tid; i < n; i += nth) dst[i] = src[i];
}

struct ChainLayout {
  int last;
  unsigned long long off[4], sec_len[4], pay_off[4], rec_len[4];
  int flag[4];
};

__device__ void chain_layout(const BmState* bm, int width0, ChainLayout* L) {
  int deepest = 0;
  for (int k = 0; k < 4; k++)
    if (bm->lv[k].active) deepest = k;
  for (int k = deepest; k >= 0; k--) {
    const int w = k == 0 ? width0 : 1;
    const BmLevel& v = bm->lv[k];
    bool f = false;
    if (k < deepest) f = L->rec_len[k + 1] < v.bm_len;
    L->flag[k] = f;
    L->sec_len[k] = f ? L->rec_len[k + 1] : v.bm_len;
    L->rec_len[k] = 19 + L->sec_len[k] + v.kept * w;
  }
  L->last = 0;
  L->off[0] = 0;
  for (int k = 0; k <= deepest; k++) {
    L->pay_off[k] = L->off[k] + 19 + L->sec_len[k];
    if (L->flag[k]) {
      L->off[k + 1] = L->off[k] + 19;
    } else {
      L->last = k;
      break;
    }
  }
}

// Write the (nested) record: headers, innermost raw bitmap, payloads.
// dst = out + (dst_off_dev ? *dst_off_dev : 0)
__global__ void k_chain_assemble(int stage, int width0, BmState* bm, uint8_t* const* bitmaps,
                                 uint8_t* const* payloads, uint8_t* out, const unsigned long long* dst_off_dev,
                                 unsigned long long* rec_len_out) {
  __shared__ ChainLayout L;
  if (threadIdx.x == 0) chain_layout(bm, width0, &L);
  __syncthreads();
  uint8_t* dst = out + (dst_off_dev ? *dst_off_dev : 0ull);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k <= L.last; k++) {
      uint8_t* h = dst + L.off[k];
      h[0] = (uint8_t)(k == 0 ? stage : 2);
      h[1] = (uint8_t)(k == 0 ? width0 : 1);
      st_bytes(h + 2, bm->lv[k].orig, 8);
      h[10] = (uint8_t)L.flag[k];
      st_bytes(h + 11, L.sec_len[k], 8);
      bm->lv[k].flag = L.flag[k];
      bm->lv[k].rec_len = L.rec_len[k];
    }
    *rec_len_out = L.rec_len[0];
  }
  // copy ranges: raw bitmap of the last level, then payloads of levels 0..last
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long nth = (unsigned long long)gridDim.x * blockDim.x;
  copy_to_unaligned(dst + L.off[L.last] + 19, bitmaps[L.last], bm->lv[L.last].bm_len, tid, nth);
  for (int k = 0; k <= L.last; k++) {
    const int w = k == 0 ? width0 : 1;
    copy_to_unaligned(dst + L.pay_off[k], payloads[k], bm->lv[k].kept * w, tid, nth);
  }
  // zero pad to the next 8-byte boundary (+8) for word-reading consumers
  const unsigned long long end = L.rec_len[0];
  for (unsigned long long i = end + tid; i < ((end + 7) & ~7ull) + 8; i += nth) dst[i] = 0;
}

// Levels 1..3 of a chain and the record assembly in ONE launch (they were
// four: ~7 us of fixed latency each on small records).  Tiles are handed out
// per level by that level's ticket; a CTA that finds its level's tickets
// exhausted waits until every tile of the level has completed before reading
// the level's sizes.  Tiles are only ever held by running CTAs, so the wait
// cannot deadlock whatever the residency.  Then every CTA lays out the record
// and copies its share (k_chain_assemble's body).
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(RD_THREADS, 4)
    k_reduce_tail(int stage, int width0, BmState* bm, uint8_t* const* bitmaps, uint8_t* const* payloads,
                  unsigned long long* lb_ws, unsigned long long lb_stride, uint8_t* out,
                  const unsigned long long* dst_off_dev, unsigned long long* rec_len_out) {
  __shared__ __align__(16) uint8_t stg[RD_TILE];
  __shared__ ChainLayout L;
  __shared__ BmState sbm;
  for (int level = 1; level <= 3; level++) {
    BmLevel* p = &bm->lv[level - 1];
    // written by k_reduce0 (level 1) or by this kernel before the wait below
    const int active = __ldcg(&p->active);
    const unsigned long long nw = __ldcg(&p->bm_len);
    if (!active || nw <= 19) break;
    BmLevel* lv = &bm->lv[level];
    MemSrc src{bitmaps[level - 1], nw, 1};
    reduce_tiles<MemSrc, uint32_t, 2, 1>(src, nw, 2, 1, bitmaps[level], payloads[level], lb_ws + level * lb_stride, lv,
                                         stg, &lv->tiles_done);
    if (threadIdx.x == 0) {
      const unsigned long long nt = cdiv(nw, RD_TILE);
      while (ld_acquire_u64(&lv->tiles_done) < nt) __nanosleep(64);
    }
    __syncthreads();
  }
  // record layout from an L2-fresh copy of the level table
  if (threadIdx.x < (int)(sizeof(BmState) / 8))
    reinterpret_cast<unsigned long long*>(&sbm)[threadIdx.x] =
        __ldcg(reinterpret_cast<const unsigned long long*>(bm) + threadIdx.x);
  __syncthreads();
  if (threadIdx.x == 0) chain_layout(&sbm, width0, &L);
  __syncthreads();
  uint8_t* dst = out + (dst_off_dev ? *dst_off_dev : 0ull);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k <= L.last; k++) {
      uint8_t* h = dst + L.off[k];
      h[0] = (uint8_t)(k == 0 ? stage : 2);
      h[1] = (uint8_t)(k == 0 ? width0 : 1);
      st_bytes(h + 2, sbm.lv[k].orig, 8);
      h[10] = (uint8_t)L.flag[k];
      st_bytes(h + 11, L.sec_len[k], 8);
      bm->lv[k].flag = L.flag[k];
      bm->lv[k].rec_len = L.rec_len[k];
    }
    *rec_len_out = L.rec_len[0];
  }
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long nth = (unsigned long long)gridDim.x * blockDim.x;
  copy_to_unaligned(dst + L.off[L.last] + 19, bitmaps[L.last], sbm.lv[L.last].bm_len, tid, nth);
  for (int k = 0; k <= L.last; k++) {
    const int w = k == 0 ? width0 : 1;
    copy_to_unaligned(dst + L.pay_off[k], payloads[k], sbm.lv[k].kept * w, tid, nth);
  }
  const unsigned long long end = L.rec_len[0];
  for (unsigned long long i = end + tid; i < ((end + 7) & ~7ull) + 8; i += nth) dst[i] = 0;
}

struct ChainPtrs {
  uint8_t* bitmap[4];
  uint8_t* payload[4];
};

static unsigned persist_grid(unsigned long long tiles_bound) {
  return (unsigned)(tiles_bound < PERSIST_CTAS ? (tiles_bound ? tiles_bound : 1) : PERSIST_CTAS);
}

// Runs level 0 + 3 nested levels + assembly.  lb_ws: 4 zeroed look-back
// regions of (1 + tiles) u64 each, laid out consecutively with stride lb_stride.
void launch_reduce_chain_impl(int stage, int width, int src_kind, const uint8_t* src_ptr,
                              const unsigned long long* len_dev, int tw, unsigned long long max_words,
                              const ReduceBufs& bufs, BmState* bm, uint8_t* rec_out,
                              const unsigned long long* dst_off_dev, unsigned long long* rec_len_dev,
                              unsigned long long* lb_ws, unsigned long long lb_stride, uint8_t* const* dev_ptr_tables,
                              cudaStream_t s, int* launches) {
  const unsigned long long tiles0 = cdiv(max_words, RD_TILE);
  const unsigned g0 = persist_grid(tiles0);
  const size_t stg = width <= 4 ? (size_t)RD_TILE * width : 0;
  switch (src_kind) {
    case SRC_MEM:
      if (stage == 2 && width == 4) {  // CR: RRE4 over the Huffman record
        static const bool attr = [&] {  // once per process, thread-safe (C++11 static init)
          cudaFuncSetAttribute(k_reduce0<MemSrc, uint32_t, 2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               RD_TILE * 4);
          return true;
        }();
        (void)attr;
        k_reduce0<MemSrc, uint32_t, 2, 4><<<g0, RD_THREADS, stg, s>>>(MemSrc{src_ptr, 0, width}, len_dev, stage,
                                                                      width, bm, bufs.bitmap[0], bufs.payload[0],
                                                                      lb_ws);
      } else if (width <= 4) {
        static const bool attr = [&] {
          cudaFuncSetAttribute(k_reduce0<MemSrc, uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               RD_TILE * 4);
          return true;
        }();
        (void)attr;
        k_reduce0<MemSrc, uint32_t><<<g0, RD_THREADS, stg, s>>>(MemSrc{src_ptr, 0, width}, len_dev, stage, width,
                                                                bm, bufs.bitmap[0], bufs.payload[0], lb_ws);
      } else {
        k_reduce0<MemSrc, uint64_t><<<g0, RD_THREADS, 0, s>>>(MemSrc{src_ptr, 0, width}, len_dev, stage, width, bm,
                                                              bufs.bitmap[0], bufs.payload[0], lb_ws);
      }
      break;
    case SRC_TCMS:
      if (stage == 3 && width == 1 && tw == 8)  // CR: RZE1 over TCMS8
        k_reduce0<TcmsSrc, uint32_t, 3, 1><<<g0, RD_THREADS, stg, s>>>(TcmsSrc{src_ptr, 0, tw}, len_dev, stage,
                                                                       width, bm, bufs.bitmap[0], bufs.payload[0],
                                                                       lb_ws);
      else
        k_reduce0<TcmsSrc, uint32_t><<<g0, RD_THREADS, stg, s>>>(TcmsSrc{src_ptr, 0, tw}, len_dev, stage, width,
                                                                 bm, bufs.bitmap[0], bufs.payload[0], lb_ws);
      break;
    default:  // TP: RRE1 over BIT1(TCMS1)
      k_reduce0<TpSrc, uint32_t, 2, 1><<<g0, RD_THREADS, stg, s>>>(TpSrc{src_ptr, 0}, len_dev, stage, width, bm,
                                                                   bufs.bitmap[0], bufs.payload[0], lb_ws);
      break;
  }
  (*launches)++;
  static const bool split_tail = getenv("HB_SPLIT_TAIL") != nullptr;  // the four-launch form (variant tests)
  if (!split_tail) {
    // sized by the level-1 input bound (level-0 bitmap: one bit per word):
    // every CTA of the grid waits out each nested level, so small records
    // must not pay for a full persistent grid
    const unsigned gt = persist_grid(cdiv(cdiv(max_words, 8), RD_TILE));
    k_reduce_tail<<<gt, RD_THREADS, 0, s>>>(stage, width, bm, dev_ptr_tables, dev_ptr_tables + 4, lb_ws,
                                                      lb_stride, rec_out, dst_off_dev, rec_len_dev);
    (*launches)++;
    return;
  }
  unsigned long long words = cdiv(max_words, 8);
  for (int k = 1; k <= 3; k++) {
    const unsigned g = persist_grid(cdiv(words, RD_TILE));
    k_reduce_nested<<<g, RD_THREADS, 0, s>>>(k, bm, bufs.bitmap[k - 1], bufs.bitmap[k], bufs.payload[k],
                                             lb_ws + k * lb_stride);
    (*launches)++;
    words = cdiv(words, 8);
  }
  k_chain_assemble<<<PERSIST_CTAS, 256, 0, s>>>(stage, width, bm, dev_ptr_tables, dev_ptr_tables + 4, rec_out,
                                                dst_off_dev, rec_len_dev);
  (*launches)++;
}

// ------------------------------------------------------------- Huffman
// stages.py:246-329.  Code lengths with the heap's (freq, id) order via the
// equivalent two-queue merge, canonical codes by (len, sym),
// MSB-first packing.

__global__ void k_hist(const uint8_t* __restrict__ in, unsigned long long n, DevState* st) {
  __shared__ unsigned h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    atomicAdd(&h[in[i]], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&st->hist[i], (unsigned long long)h[i]);
}

void launch_hist(const uint8_t* in, unsigned long long n, DevState* st, cudaStream_t s, int* launches) {
  unsigned long long b = cdiv(n ? n : 1, 256 * 16);
  if (b > 148 * 8) b = 148 * 8;
  k_hist<<<(unsigned)b, 256, 0, s>>>(in, n, st);
  (*launches)++;
}

__global__ void __launch_bounds__(512) k_huff_build(DevState* st, unsigned long long n, uint8_t* rec) {
  __shared__ unsigned long long f[256];
  __shared__ int sorted[256];
  __shared__ int parent[512];
  __shared__ unsigned long long ifreq[256];
  __shared__ int anc[512], dep[512];
  __shared__ uint8_t len[256];
  __shared__ int np_sh, cnt[64];
  __shared__ unsigned long long first[64];
  __shared__ unsigned long long red[33];
  const int t = threadIdx.x;
  if (t < 256) {
    f[t] = st->hist[t];
    len[t] = 0;
  }
  if (t < 64) cnt[t] = 0;
  if (t == 0) np_sh = 0;
  __syncthreads();
  if (t < 256 && f[t]) atomicAdd(&np_sh, 1);
  __syncthreads();
  const int np = np_sh;
  if (t < 256 && f[t]) {  // rank by (freq, symbol) = heap pop order of the leaves
    const unsigned long long ft = f[t];
    int r = 0;
    for (int j = 0; j < 256; j++) {
      const unsigned long long fj = f[j];
      r += fj && (fj < ft || (fj == ft && j < t));
    }
    sorted[r] = t;
  }
  __syncthreads();
  // heapq on (freq, id) == two-queue merge: leaves in (freq, sym) order,
  // internal nodes FIFO (ids ascending, freqs non-decreasing), leaf first on
  // ties.  One thread; the heads of both queues live in registers so an
  // iteration waits on at most one shared load (the serial chain is the cost).
  __shared__ unsigned long long sf[256];
  if (t < np) sf[t] = f[sorted[t]];
  __syncthreads();
  if (t == 0 && np > 1) {
    int li = 0, ih = 0;
    unsigned long long fl = sf[0], fi = 0;  // leaf head, internal head (valid while ih < m)
    for (int m = 0; m < np - 1; m++) {
      int pick0, pick1;
      unsigned long long p0, p1;
      if (li < np && (ih >= m || fl <= fi)) {
        pick0 = sorted[li], p0 = fl;
        li++;
        fl = li < np ? sf[li] : 0;
      } else {
        pick0 = 256 + ih, p0 = fi;
        ih++;
        fi = ih < m ? ifreq[ih] : 0;
      }
      if (li < np && (ih >= m || fl <= fi)) {
        pick1 = sorted[li], p1 = fl;
        li++;
        fl = li < np ? sf[li] : 0;
      } else {
        pick1 = 256 + ih, p1 = fi;
        ih++;
        fi = ih < m ? ifreq[ih] : 0;
      }
      parent[pick0] = 256 + m;
      parent[pick1] = 256 + m;
      const unsigned long long nf = p0 + p1;
      ifreq[m] = nf;
      if (ih == m) fi = nf;  // the new node heads an empty internal queue
    }
  }
  __syncthreads();
  // depths by pointer jumping over the parent links (root = 256 + np - 2)
  if (np > 1) {
    const int root = 256 + np - 2;
    const bool node = (t < 256 && f[t]) || (t >= 256 && t <= root);
    anc[t] = node && t != root ? parent[t] : t;
    dep[t] = node && t != root ? 1 : 0;
    __syncthreads();
    for (int k = 0; k < 9; k++) {
      const int a = anc[t];
      const int d = dep[t] + dep[a];
      const int aa = anc[a];
      __syncthreads();
      dep[t] = d;
      anc[t] = aa;
      __syncthreads();
    }
    if (t < 256 && f[t]) len[t] = (uint8_t)dep[t];
  } else if (np == 1 && t == 0) {
    len[sorted[0]] = 1;
  }
  __syncthreads();
  // canonical codes (stages.py:275-287): per length the first code, then rank
  if (t < 256 && len[t]) atomicAdd(&cnt[len[t]], 1);
  __syncthreads();
  if (t == 0) {  // first code per length: start[L+1] = (start[L] + count[L]) << 1
    unsigned long long c = 0;
    for (int L = 1; L < 64; L++) {
      first[L] = c;
      c = (c + cnt[L]) << 1;
    }
  }
  __syncthreads();
  if (t < 256) {
    const int L = len[t];
    unsigned long long c = 0;
    if (L) {
      int r = 0;
      for (int j = 0; j < t; j++) r += len[j] == L;
      c = first[L] + r;
    }
    st->hf_code[t] = c;
    st->hf_len[t] = (uint8_t)L;
  }
  // nbits = sum hist * len
  unsigned long long tot;
  block_excl_scan<unsigned long long>(t < 256 ? f[t] * len[t] : 0ull, red, &tot);
  if (t == 0) {
    const unsigned long long nbits = n ? tot : 0;
    st->hf_nbits = nbits;
    st->hf_rec_len = 274 + cdiv(nbits, 8);
    rec[0] = 1;
    rec[1] = 1;
    st_bytes(rec + 2, n, 8);
    st_bytes(rec + 10, nbits, 8);
    rec[274] = 0;
    rec[275] = 0;
  }
  if (t < 256) rec[18 + t] = len[t];
}

void launch_huffman_build(DevState* st, unsigned long long n, uint8_t* hf_rec, cudaStream_t s, int* launches) {
  k_huff_build<<<1, 512, 0, s>>>(st, n, hf_rec);
  (*launches)++;
}

// zero the payload words [69, end) of the HF record before the OR-packing
__global__ void k_huff_zero(uint32_t* rec_words, DevState* st) {
  const unsigned long long end = cdiv(st->hf_rec_len, 4) + 4;
  for (unsigned long long i = 69 + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < end;
       i += (unsigned long long)gridDim.x * blockDim.x)
    rec_words[i] = 0;
}

constexpr int HE_SYMS = 32;                    // symbols per lane per round
constexpr int HE_ROUNDS = 4;                   // rounds of 32 x 32 symbols per warp tile
constexpr int HE_WTILE = 32 * HE_SYMS * HE_ROUNDS;  // symbols per warp tile (== HE_TILE_SYMS, hb_kernels.h)
constexpr int HE_WARPS = 8;                    // warps per CTA
constexpr int HE_BUF = HE_WTILE / 4 + 2;       // words per warp buffer: <= 8 bits/symbol (+ spill word)
static_assert(HE_WTILE == HE_TILE_SYMS, "look-back workspace sizing");

// MSB-first OR of one code into a big-endian-bit word array (bits [pos, pos+L))
template <bool GLOBAL>
__device__ __forceinline__ void he_put(uint32_t* words, unsigned long long pos, int L, unsigned long long c) {
  const unsigned long long end = pos + L;
  unsigned long long wi = (end - 1) >> 5;
  const int r = (int)(end & 31);
  int left = L, first = r ? r : 32;
  while (left > 0) {
    const int take = left < first ? left : first;
    const uint32_t be = (uint32_t)(c & ((1ull << take) - 1)) << (32 - first);
    if (GLOBAL)
      atomicOr(&words[wi], __byte_perm(be, 0, 0x0123));
    else
      atomicOr(&words[wi], be);
    c >>= take;
    left -= take;
    wi--;
    first = 32;
  }
}

// the 32 symbols of one lane in one round, zero past the end
__device__ __forceinline__ int he_load(const uint8_t* __restrict__ in, unsigned long long n, unsigned long long s0,
                                       uint32_t (&w)[8]) {
  const int cnt = s0 >= n ? 0 : (s0 + HE_SYMS <= n ? HE_SYMS : (int)(n - s0));
  if (cnt == HE_SYMS) {
    const uint4* p = reinterpret_cast<const uint4*>(in + s0);
    const uint4 a = p[0], b = p[1];
    w[0] = a.x, w[1] = a.y, w[2] = a.z, w[3] = a.w, w[4] = b.x, w[5] = b.y, w[6] = b.z, w[7] = b.w;
  } else {
#pragma unroll
    for (int q = 0; q < 8; q++) {
      w[q] = 0;
      for (int k = 0; k < 4; k++)
        if (q * 4 + k < cnt) w[q] |= (uint32_t)in[s0 + q * 4 + k] << (8 * k);
    }
  }
  return cnt;
}

constexpr int HE_PRIV = 8;  // words of a lane's round kept in shared memory (denser lanes re-walk)

// One lane's round: its 32 codes through a 64-bit bit writer into the lane's
// private words (left-aligned, MSB-first), returns the round's bit count and
// whether they all fit the private words.  Codes <= 32 bits.
template <bool FULL>
__device__ __forceinline__ unsigned he_pack_lane(const uint32_t (&w)[8], int cnt, const unsigned long long* stab,
                                                 uint32_t* priv, bool& fits) {
  uint64_t acc = 0;
  unsigned ab = 0, nw = 0;
  auto put32 = [&](uint32_t c, unsigned L) {  // L <= 32, ab < 32 on entry
    acc |= (uint64_t)c << (64 - ab - L);
    ab += L;
    if (ab >= 32) {
      if (nw < HE_PRIV) priv[nw * 32] = (uint32_t)(acc >> 32);
      nw++;
      acc <<= 32;
      ab -= 32;
    }
  };
#pragma unroll
  for (int k = 0; k < HE_SYMS; k++) {
    if (FULL || k < cnt) {
      const unsigned long long e = stab[(w[k >> 2] >> (8 * (k & 3))) & 0xFF];
      const unsigned L = (unsigned)(e >> 56);
      put32((uint32_t)e, L);
    }
  }
  const unsigned nb = nw * 32 + ab;
  if (ab) {
    if (nw < HE_PRIV) priv[nw * 32] = (uint32_t)(acc >> 32);
    nw++;
  }
  fits = nw <= HE_PRIV;
  return nb;
}

// Warp-granular tiles: each warp takes a 4096-symbol tile by ticket (four
// rounds of 32 lanes x 32 symbols).  Per round every lane runs its codes
// through a register bit writer into private shared-memory words, a warp
// scan places the lanes, and each lane ORs its words into the warp's tile
// buffer at the tile-relative bit offset (no CTA barrier anywhere).  Then the
// tile publishes its bit count and resolves its global bit offset by
// decoupled look-back (hb_common.cuh), and streams the buffer out shifted by
// that offset (funnel shift per word, coalesced stores, the buffer re-zeroed
// on the way).  Only the first and last word of a tile can share bits with a
// neighbouring tile (global atomicOr into the pre-zeroed payload).  Rounds
// past the buffer's capacity (> 8 bits/symbol) OR straight into global
// memory after the look-back.
// long_codes: some code exceeds 32 bits -- every lane takes the per-code path
__device__ __forceinline__ void he_tiles(const uint8_t* __restrict__ in, unsigned long long n, uint32_t* rec_words,
                                         unsigned long long* lb, const unsigned long long* stab,
                                         const uint8_t* slen, uint32_t* buf, uint32_t* priv, unsigned* sx,
                                         bool long_codes, int zsym, unsigned zlen) {
  const uint32_t zrep = 0x01010101u * (uint32_t)(zsym & 0xFF);
  const int lane = threadIdx.x & 31;
  unsigned long long* status = lb + 1;
  const unsigned long long ntiles = cdiv(n, HE_WTILE);
  for (;;) {
    unsigned long long tile = 0;
    if (lane == 0) tile = atomicAdd(lb, 1ull);
    tile = __shfl_sync(0xffffffffu, tile, 0);
    if (tile >= ntiles) break;
    const unsigned long long t0 = tile * HE_WTILE + (unsigned long long)lane * HE_SYMS;
    // pass 1: code lengths only -> per-round lane offsets, tile total; the
    // aggregate is published before any packing so successors' look-backs
    // rarely wait
    unsigned total = 0, buf_bits = 0;
    int rd = HE_ROUNDS;  // first round that goes straight to global memory
#pragma unroll 1
    for (int r = 0; r < HE_ROUNDS; r++) {
      uint32_t w[8];
      const int cnt = he_load(in, n, t0 + r * 32 * HE_SYMS, w);
      unsigned nb = 0;
      if (cnt == HE_SYMS) {
#pragma unroll
        for (int k = 0; k < HE_SYMS; k++) nb += slen[(w[k >> 2] >> (8 * (k & 3))) & 0xFF];
      } else {
        for (int k = 0; k < cnt; k++) nb += slen[(w[k >> 2] >> (8 * (k & 3))) & 0xFF];
      }
      const unsigned inc = warp_incl_scan<unsigned>(nb);
      sx[r * 32 + lane] = total + inc - nb;  // the lane's first bit of round r
      total += __shfl_sync(0xffffffffu, inc, 31);
      if (rd == HE_ROUNDS && total > (unsigned)(HE_BUF - 2) * 32) rd = r;  // warp-uniform
      if (r < rd) buf_bits = total;
    }
    if (lane == 0) {
      if (tile == 0) {
        __threadfence();
        atomicExch(&status[0], LB_INC | total);
      } else {
        atomicExch(&status[tile], LB_AGG | total);
      }
    }
    // pass 2: pack the rounds that fit the tile buffer
#pragma unroll 1
    for (int r = 0; r < rd; r++) {
      uint32_t w[8];
      const int cnt = he_load(in, n, t0 + r * 32 * HE_SYMS, w);
      bool fits;
      const unsigned e0 = sx[r * 32 + lane];
      unsigned nb = 0;
      if (zsym >= 0) {
        // sparse: only codes with a set bit are written; the all-zero code
        // (the most frequent symbol of a skewed histogram) only advances the
        // position.  Mask of the lane's other symbols, SWAR per 4 bytes
        uint32_t nz = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const uint32_t b = ~__vcmpeq4(w[q], zrep) & 0x80808080u;  // byte MSB set = not the zero-code symbol
          nz |= ((b * 0x00204081u) >> 28) << (4 * q);                // bits 7/15/23/31 -> bits 0..3
          priv[lane + 32 * q] = w[q];                                  // lane bytes for indexed access
        }
        if (cnt < HE_SYMS) nz &= (1u << cnt) - 1u;
        const uint8_t* pb = reinterpret_cast<const uint8_t*>(priv);
        unsigned pos = e0;
        int prev = -1;
        while (nz) {
          const int k = __ffs(nz) - 1;
          nz &= nz - 1;
          pos += (unsigned)(k - prev - 1) * zlen;
          prev = k;
          const unsigned long long e = stab[pb[4 * (lane + 32 * (k >> 2)) + (k & 3)]];
          const int L = (int)(e >> 56);
          if (L <= 32) {
            const uint64_t v = (e & 0xFFFFFFFFull) << (64 - (int)(pos & 31) - L);
            const unsigned wi = pos >> 5;
            if ((uint32_t)(v >> 32)) atomicOr(&buf[wi], (uint32_t)(v >> 32));
            if ((uint32_t)v) atomicOr(&buf[wi + 1], (uint32_t)v);
          } else {
            he_put<false>(buf, pos, L, e & ((1ull << 56) - 1));
          }
          pos += (unsigned)L;
        }
        __syncwarp();  // private words reused by the next round
        continue;
      }
      if (long_codes)
        fits = false;
      else if (cnt == HE_SYMS)
        nb = he_pack_lane<true>(w, cnt, stab, priv + lane, fits);
      else
        nb = he_pack_lane<false>(w, cnt, stab, priv + lane, fits);
      if (fits) {
        const unsigned b = e0 & 31, wb = e0 >> 5, nwl = (nb + 31) >> 5;
        for (unsigned i = 0; i < nwl; i++) {
          const uint32_t v = priv[lane + 32 * i];
          if (v) {
            atomicOr(&buf[wb + i], v >> b);
            if (b && (v << (32 - b))) atomicOr(&buf[wb + i + 1], v << (32 - b));
          }
        }
      } else {  // a dense lane: re-walk its codes
        unsigned long long pos = e0;
        for (int k = 0; k < HE_SYMS; k++) {
          const unsigned long long e = k < cnt ? stab[(w[k >> 2] >> (8 * (k & 3))) & 0xFF] : 0ull;
          const int L = (int)(e >> 56);
          const unsigned long long c = e & ((1ull << 56) - 1);
          if (c) he_put<false>(buf, pos, L, c);
          pos += L;
        }
      }
      __syncwarp();  // private words reused by the next round
    }
    const unsigned long long base = tile == 0 ? 0ull : lookback_wait(status, tile, total);
    const unsigned long long tstart = 274ull * 8 + base;  // the tile's first bit in the record
    const int s = (int)(tstart & 31);
    const unsigned long long w0 = tstart >> 5;
    const unsigned nout = buf_bits ? (s + buf_bits + 31) >> 5 : 0;
    for (unsigned j = lane; j < nout; j += 32) {
      const uint32_t v = s ? ((j ? buf[j - 1] << (32 - s) : 0u) | (buf[j] >> s)) : buf[j];
      const uint32_t le = __byte_perm(v, 0, 0x0123);
      if (j == 0 || j == nout - 1) {
        if (v) atomicOr(&rec_words[w0 + j], le);
      } else {
        rec_words[w0 + j] = le;
      }
    }
    __syncwarp();
    for (unsigned j = lane; j < nout; j += 32) buf[j] = 0;  // clean for the next tile
    __syncwarp();
#pragma unroll 1
    for (int r = rd; r < HE_ROUNDS; r++) {
      uint32_t w[8];
      const int cnt = he_load(in, n, t0 + r * 32 * HE_SYMS, w);
      unsigned long long pos = tstart + sx[r * 32 + lane];
      for (int k = 0; k < HE_SYMS; k++) {
        const unsigned long long e = k < cnt ? stab[(w[k >> 2] >> (8 * (k & 3))) & 0xFF] : 0ull;
        const int L = (int)(e >> 56);
        const unsigned long long c = e & ((1ull << 56) - 1);
        if (c) he_put<true>(rec_words, pos, L, c);
        pos += L;
      }
    }
  }
}

__global__ void __launch_bounds__(HE_WARPS * 32, 4)
    k_huff_encode(const uint8_t* __restrict__ in, unsigned long long n, uint32_t* rec_words, unsigned long long* lb,
                  DevState* st) {
  __shared__ unsigned long long stab[256];  // code | len << 56
  __shared__ uint8_t slen[256];
  __shared__ uint32_t wbuf[HE_WARPS][HE_BUF];
  __shared__ uint32_t wpriv[HE_WARPS][HE_PRIV * 32];
  __shared__ unsigned wx[HE_WARPS][HE_ROUNDS * 32];
  const unsigned L = st->hf_len[threadIdx.x];
  stab[threadIdx.x] = st->hf_code[threadIdx.x] | ((unsigned long long)L << 56);
  slen[threadIdx.x] = (uint8_t)L;
  for (int i = threadIdx.x; i < HE_WARPS * HE_BUF; i += blockDim.x) (&wbuf[0][0])[i] = 0;
  __shared__ int zsym_sh;
  if (threadIdx.x == 0) zsym_sh = -1;
  __syncthreads();
  // the canonical all-zero code (unique): the sparse pack pays off when that
  // symbol is a large share of the stream (smooth fields), not on flat
  // histograms (rough fields), where the bit-writer pack is kept
  if (L && st->hf_code[threadIdx.x] == 0 && st->hist[threadIdx.x] * 4 >= n) zsym_sh = (int)threadIdx.x;
  const bool any_long = __syncthreads_or(L > 32);
  const int zsym = zsym_sh;
  uint32_t* buf = wbuf[threadIdx.x >> 5];
  uint32_t* priv = wpriv[threadIdx.x >> 5];
  he_tiles(in, n, rec_words, lb, stab, slen, buf, priv, wx[threadIdx.x >> 5], any_long, zsym,
           zsym >= 0 ? slen[zsym] : 0u);
}

void launch_huffman_encode(const uint8_t* seq, unsigned long long n, uint8_t* hf_rec, unsigned long long* lb_ws,
                           DevState* st, cudaStream_t s, int* launches) {
  k_huff_zero<<<PERSIST_CTAS, 256, 0, s>>>(reinterpret_cast<uint32_t*>(hf_rec), st);
  (*launches)++;
  if (n == 0) return;
  const unsigned long long tiles = cdiv(cdiv(n, HE_WTILE), HE_WARPS);
  k_huff_encode<<<persist_grid(tiles), HE_WARPS * 32, 0, s>>>(seq, n, reinterpret_cast<uint32_t*>(hf_rec), lb_ws, st);
  (*launches)++;
}

// ------------------------------------------------------ archive tail
// archive.py:55-74: escape decision, fixed header, counts, stream placement.
// `base` = 46 + 8 + anchors*prec + 8 (host-known); outliers follow, then the
// stream length and stream.  The encoded stream was already assembled at
// stream_off; on escape the raw sequence overwrites it.
__global__ void k_stream_offset(unsigned long long base, int prec, DevState* st) {
  st->scratch[0] = base + st->outlier_count * (8ull + prec) + 8;  // stream_off
}

__global__ void k_archive_tail(uint8_t* arch, unsigned long long base, int prec, const uint8_t* seq,
                               unsigned long long n, const uint8_t* header46, unsigned long long na, DevState* st) {
  const unsigned long long soff = st->scratch[0];
  const unsigned long long enc = st->stream_len;
  const bool esc = enc > n;
  const unsigned long long slen = esc ? n : enc;
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long nth = (unsigned long long)gridDim.x * blockDim.x;
  if (esc) copy_to_unaligned(arch + soff, seq, n, tid, nth);
  if (tid == 0) {
    for (int i = 0; i < 46; i++) arch[i] = header46[i];
    arch[9] = esc ? 1 : 0;
    for (int i = 0; i < 4; i++) arch[10 + i] = st->cfg[i];
    unsigned long long ebits = (unsigned long long)__double_as_longlong(st->eb);
    st_bytes(arch + 38, ebits, 8);
    st_bytes(arch + 46, na, 8);
    st_bytes(arch + base - 8, st->outlier_count, 8);
    st_bytes(arch + soff - 8, slen, 8);
    st->escape = esc;
    st->archive_len = soff + slen;
  }
}

void launch_archive_tail_impl(uint8_t* arch, unsigned long long base, int prec, const uint8_t* seq,
                              unsigned long long n, const uint8_t* header46, unsigned long long na, DevState* st,
                              cudaStream_t s, int* launches) {
  unsigned long long b = cdiv(n, 256 * 8);
  if (b > PERSIST_CTAS) b = PERSIST_CTAS;
  k_archive_tail<<<(unsigned)b, 256, 0, s>>>(arch, base, prec, seq, n, header46, na, st);
  (*launches)++;
}

void launch_stream_offset(unsigned long long base, int prec, DevState* st, cudaStream_t s, int* launches) {
  k_stream_offset<<<1, 1, 0, s>>>(base, prec, st);
  (*launches)++;
}

// ============================================================= decoders

// Parsed nested reducer record (stages.py:187-221), level 0 outermost.
struct BmDec {
  int ok, last;
  int w[4];
  unsigned long long orig[4], nsym[4], bm_off[4], bm_len[4], pay_off[4], pay_len[4];
};

__device__ void bm_parse(int stage, const uint8_t* rec, const unsigned long long* len_dev, BmDec* D,
                         unsigned long long out_cap, unsigned long long* out_len, DevState* st) {
  D->ok = 0;
  if (st->flags & (F_STAGE | F_ARCHIVE)) return;
  unsigned long long off = 0, end = *len_dev;
  for (int k = 0; k < 4; k++) {
    const int expect = k == 0 ? stage : 2;
    if (end - off < 10) return raise_flag(st, F_STAGE, 100);
    const uint8_t* h = rec + off;
    if (h[0] != expect) return raise_flag(st, F_STAGE, 101);
    const int w = h[1];
    if (w != 1 && w != 2 && w != 4 && w != 8) return raise_flag(st, F_STAGE, 102);
    const unsigned long long orig = ld_bytes(h + 2, 8);
    if (end - off < 19) return raise_flag(st, F_STAGE, 103);
    const int flag = h[10];
    const unsigned long long bl = ld_bytes(h + 11, 8);
    if (flag != 0 && flag != 1) return raise_flag(st, F_STAGE, 104);
    if (bl > end - off - 19) return raise_flag(st, F_STAGE, 105);
    D->w[k] = w;
    D->orig[k] = orig;
    D->nsym[k] = orig / w + (orig % w != 0);
    D->bm_off[k] = off + 19;
    D->bm_len[k] = bl;
    D->pay_off[k] = off + 19 + bl;
    D->pay_len[k] = end - (off + 19 + bl);
    if (D->pay_len[k] % w) return raise_flag(st, F_STAGE, 106);
    if (k > 0 && D->orig[k] != cdiv(D->nsym[k - 1], 8)) return raise_flag(st, F_STAGE, 107);
    if (!flag) {
      if (bl != cdiv(D->nsym[k], 8)) return raise_flag(st, F_STAGE, 108);
      D->last = k;
      break;
    }
    if (k == 3) return raise_flag(st, F_STAGE, 109);  // recursion exceeds maximum depth
    off = off + 19;
    end = off + bl;
  }
  if (D->orig[0] > out_cap) return raise_flag(st, F_STAGE, 110);
  for (int k = 1; k <= D->last; k++)
    if (D->orig[k] > out_cap) return raise_flag(st, F_STAGE, 110);
  *out_len = D->orig[0];
  D->ok = 1;
}

__global__ void k_bm_parse(int stage, const uint8_t* rec, const unsigned long long* len_dev, BmDec* D,
                           unsigned long long out_cap, unsigned long long* out_len, DevState* st) {
  bm_parse(stage, rec, len_dev, D, out_cap, out_len, st);
}

// decode one level: bitmap bits + payload -> words (RRE: kept[cumsum-1], RZE: scatter).
// STG / W: compile-time stage / width of the level (0 = runtime), one body
// per combination the archives hold so each runs only its own width's code.
template <int STG, int W>
__device__ __forceinline__ void bm_decode_level(int stg_rt, int w_rt, unsigned long long nsym, const uint8_t* bm,
                                                const uint8_t* pay, unsigned long long npay, uint8_t* out,
                                                unsigned long long* lb, DevState* st,
                                                unsigned long long* done = nullptr) {
  __shared__ unsigned long long sh[33];
  __shared__ unsigned long long tile_sh, base_sh;
  const int stg = STG ? STG : stg_rt;
  const int w = W ? W : w_rt;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned long long ntiles = cdiv(nsym, RD_TILE);
  for (;;) {
    if (threadIdx.x == 0) tile_sh = atomicAdd(lb, 1ull);
    __syncthreads();
    const unsigned long long tile = tile_sh;
    if (tile >= ntiles) break;
    const unsigned long long w0 = tile * RD_TILE + (unsigned long long)wid * 1024;
    // each lane owns 32 consecutive output words (one bitmap word)
    const unsigned long long i0 = w0 + (unsigned long long)lane * 32;
    uint32_t mask = 0;
    if (i0 < nsym) {
      const unsigned long long bb = i0 >> 3, nbm = cdiv(nsym, 8);
      uint32_t be = 0;
      for (int q = 0; q < 4; q++) be |= (bb + q < nbm ? (uint32_t)bm[bb + q] : 0u) << (24 - 8 * q);
      const unsigned long long valid = nsym - i0;
      if (valid < 32) be &= ~(0xFFFFFFFFu >> valid);
      mask = be;  // bit (31 - j) = word i0 + j
    }
    const unsigned c = __popc(mask);
    const unsigned incl = warp_incl_scan<unsigned>(c);
    unsigned long long total;
    unsigned long long wex = block_excl_scan<unsigned long long>(lane == 31 ? incl : 0u, sh, &total);
    wex = __shfl_sync(0xffffffffu, wex, 31);
    if (threadIdx.x < 32) {
      const unsigned long long ex_ = lookback_warp(lb + 1, tile, total);
      if (threadIdx.x == 0) base_sh = ex_;
    }
    __syncthreads();
    if (stg == 2 && tile == 0 && threadIdx.x == 0 && !(mask >> 31)) raise_flag(st, F_STAGE, 121);
    if (i0 < nsym) {
      unsigned long long before = base_sh + wex + incl - c;  // ones before word i0
      uint64_t v[32];
#pragma unroll
      for (int j = 0; j < 32; j++) {
        const int bit = (mask >> (31 - j)) & 1;
        uint64_t x = 0;
        if (stg == 2) {
          const unsigned long long idx = before + bit;  // inclusive count
          if (idx >= 1 && idx <= npay) x = w == 1 ? pay[idx - 1] : ld_bytes(pay + (idx - 1) * w, w);
        } else if (bit && before < npay) {
          x = w == 1 ? pay[before] : ld_bytes(pay + before * w, w);
        }
        before += bit;
        v[j] = x;
      }
      uint8_t* o = out + i0 * w;
      if (w == 1) {
        uint32_t u[8];
#pragma unroll
        for (int k = 0; k < 8; k++)
          u[k] = (uint32_t)v[4 * k] | ((uint32_t)v[4 * k + 1] << 8) | ((uint32_t)v[4 * k + 2] << 16) |
                 ((uint32_t)v[4 * k + 3] << 24);
        uint4* q = reinterpret_cast<uint4*>(o);
        q[0] = make_uint4(u[0], u[1], u[2], u[3]);
        q[1] = make_uint4(u[4], u[5], u[6], u[7]);
      } else if (w == 4) {
        uint4* q = reinterpret_cast<uint4*>(o);
#pragma unroll
        for (int k = 0; k < 8; k++)
          q[k] = make_uint4((uint32_t)v[4 * k], (uint32_t)v[4 * k + 1], (uint32_t)v[4 * k + 2], (uint32_t)v[4 * k + 3]);
      } else if (w == 8) {
#pragma unroll
        for (int k = 0; k < 32; k++) reinterpret_cast<uint64_t*>(o)[k] = v[k];
      } else {
#pragma unroll
        for (int k = 0; k < 32; k++) reinterpret_cast<uint16_t*>(o)[k] = (uint16_t)v[k];
      }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0 && base_sh + total != npay) raise_flag(st, F_STAGE, 122);
    __syncthreads();
    if (done && threadIdx.x == 0) {  // this tile's output is written (k_bm_decode_head waits on the count)
      __threadfence();
      atomicAdd(done, 1ull);
    }
  }
}

__global__ void __launch_bounds__(RD_THREADS)
    k_bm_decode(int stage, int k, const uint8_t* rec, const BmDec* D, const uint8_t* inner_bitmap, uint8_t* out,
                unsigned long long* lb, DevState* st) {
  if (!D->ok || k > D->last) return;
  const int w = D->w[k];
  const int stg = k == 0 ? stage : 2;
  const unsigned long long nsym = D->nsym[k];
  const uint8_t* bm = k == D->last ? rec + D->bm_off[k] : inner_bitmap;
  const uint8_t* pay = rec + D->pay_off[k];
  const unsigned long long npay = D->pay_len[k] / w;
  if (nsym == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && npay != 0) raise_flag(st, F_STAGE, 120);
    return;
  }
  if (stg == 2 && w == 1)  // TP RRE1 and every nested level
    bm_decode_level<2, 1>(stg, w, nsym, bm, pay, npay, out, lb, st);
  else if (stg == 2 && w == 4)  // CR RRE4
    bm_decode_level<2, 4>(stg, w, nsym, bm, pay, npay, out, lb, st);
  else if (stg == 3 && w == 1)  // CR RZE1
    bm_decode_level<3, 1>(stg, w, nsym, bm, pay, npay, out, lb, st);
  else
    bm_decode_level<0, 0>(stg, w, nsym, bm, pay, npay, out, lb, st);
}

struct TmpPtrs {  // level k's decoded bitmap (k >= 1), by value
  uint8_t* p[4];
  __device__ uint8_t* operator[](int k) const { return p[k]; }
};

// The record header walk and the nested bitmap levels (3 -> 1, all small:
// level k has 1/8^k of the level-0 symbols) in ONE launch: every CTA parses
// the headers into shared memory (block 0 also publishes them for the
// level-0 launch), then the CTAs take each level's tiles by ticket and wait
// for the level's completion count before the next level reads its output.
__global__ void __launch_bounds__(RD_THREADS)
    k_bm_decode_head(int stage, const uint8_t* rec, const unsigned long long* len_dev, BmDec* Dg,
                     unsigned long long out_cap, unsigned long long* out_len, TmpPtrs tmp,
                     unsigned long long* lb_ws, unsigned long long lb_stride, DevState* st) {
  __shared__ BmDec D;
  __shared__ int go;
  if (threadIdx.x == 0) {
    unsigned long long dummy;
    bm_parse(stage, rec, len_dev, &D, out_cap, blockIdx.x == 0 ? out_len : &dummy, st);
    if (blockIdx.x == 0) *Dg = D;
    go = D.ok;
  }
  __syncthreads();
  if (!go) return;
  for (int k = 3; k >= 1; k--) {
    if (k > D.last) continue;
    const int w = D.w[k];
    const unsigned long long nsym = D.nsym[k];
    const uint8_t* bm = k == D.last ? rec + D.bm_off[k] : tmp[k + 1];
    const uint8_t* pay = rec + D.pay_off[k];
    const unsigned long long npay = D.pay_len[k] / w;
    if (nsym == 0) {
      if (blockIdx.x == 0 && threadIdx.x == 0 && npay != 0) raise_flag(st, F_STAGE, 120);
      continue;
    }
    unsigned long long* lb = lb_ws + (3 - k) * lb_stride;
    unsigned long long* done = lb + lb_stride - 1;  // spare last entry of the level's zeroed region
    if (w == 1)  // nested levels are RRE1 as written by the encoder
      bm_decode_level<2, 1>(2, w, nsym, bm, pay, npay, tmp[k], lb, st, done);
    else
      bm_decode_level<0, 0>(2, w, nsym, bm, pay, npay, tmp[k], lb, st, done);
    if (threadIdx.x == 0) {
      const unsigned long long nt = cdiv(nsym, RD_TILE);
      while (ld_acquire_u64(done) < nt) __nanosleep(64);
    }
    __syncthreads();
  }
}

void launch_reduce_decode_impl(int stage, const uint8_t* rec, const unsigned long long* rec_len_dev,
                               unsigned long long out_cap, uint8_t* out, unsigned long long* out_len_dev,
                               uint8_t* const tmp[4], void* bmdec, unsigned long long* lb_ws,
                               unsigned long long lb_stride, DevState* st, cudaStream_t s, int* launches) {
  BmDec* D = reinterpret_cast<BmDec*>(bmdec);
  // innermost first: level k writes tmp[k] (k >= 1) or out (k == 0)
  unsigned long long words = out_cap;  // bound on level-0 symbols
  unsigned long long wb[4];
  for (int k = 0; k < 4; k++) {
    wb[k] = words;
    words = cdiv(words, 8);
  }
  static const bool split = getenv("HB_SPLIT_BM_DECODE") != nullptr;  // the five-launch form (variant tests)
  if (!split) {
    const TmpPtrs tp{{tmp[0], tmp[1], tmp[2], tmp[3]}};
    k_bm_decode_head<<<persist_grid(cdiv(wb[1], RD_TILE)), RD_THREADS, 0, s>>>(stage, rec, rec_len_dev, D, out_cap,
                                                                             out_len_dev, tp, lb_ws, lb_stride, st);
    (*launches)++;
    k_bm_decode<<<persist_grid(cdiv(wb[0], RD_TILE)), RD_THREADS, 0, s>>>(stage, 0, rec, D, tmp[1], out,
                                                                        lb_ws + 3 * lb_stride, st);
    (*launches)++;
    return;
  }
  k_bm_parse<<<1, 1, 0, s>>>(stage, rec, rec_len_dev, D, out_cap, out_len_dev, st);
  (*launches)++;
  for (int k = 3; k >= 0; k--) {
    const unsigned g = persist_grid(cdiv(wb[k], RD_TILE));
    k_bm_decode<<<g, RD_THREADS, 0, s>>>(stage, k, rec, D, k < 3 ? tmp[k + 1] : nullptr, k == 0 ? out : tmp[k],
                                         lb_ws + (3 - k) * lb_stride, st);
    (*launches)++;
  }
}

// TCMS decode (stages.py:111-118), any width, record -> bytes
__global__ void k_tcms_decode(const uint8_t* rec, const unsigned long long* len_dev, unsigned long long cap,
                              uint8_t* out, unsigned long long* out_len, DevState* st) {
  if (st->flags & (F_STAGE | F_ARCHIVE)) return;
  const unsigned long long n = *len_dev;
  if (n < 10 || rec[0] != 4) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(st, F_STAGE, 130);
    return;
  }
  const int w = rec[1];
  const unsigned long long orig = ld_bytes(rec + 2, 8), body = n - 10;
  if ((w != 1 && w != 2 && w != 4 && w != 8) || body % w || body < orig || body > cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(st, F_STAGE, 131);
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out_len = orig;
  const unsigned long long nw = body / w;
  if (w == 1 && (reinterpret_cast<uintptr_t>(out) & 7) == 0) {
    // 8 bytes per thread: one aligned 8-byte store, SWAR un-zigzag
    const unsigned long long n8 = nw / 8;
    const uint8_t* q = rec + 10;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
         i += (unsigned long long)gridDim.x * blockDim.x)
      *reinterpret_cast<uint64_t*>(out + 8 * i) = unzz8x1(ld_bytes(q + 8 * i, 8));
    for (unsigned long long i = n8 * 8 + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nw;
         i += (unsigned long long)gridDim.x * blockDim.x)
      out[i] = (uint8_t)unzz(q[i], 1);
    return;
  }
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nw;
       i += (unsigned long long)gridDim.x * blockDim.x)
    st_bytes(out + i * w, unzz(ld_bytes(rec + 10 + i * w, w), w), w);
}

void launch_tcms_decode(const uint8_t* rec, const unsigned long long* rec_len_dev, unsigned long long cap,
                        uint8_t* out, unsigned long long* out_len_dev, DevState* st, cudaStream_t s, int* launches) {
  k_tcms_decode<<<PERSIST_CTAS, 256, 0, s>>>(rec, rec_len_dev, cap, out, out_len_dev, st);
  (*launches)++;
}

// BIT unshuffle (stages.py:144-160), any width: record -> bytes
__global__ void k_bit_decode(const uint8_t* rec, const unsigned long long* len_dev, uint8_t* out,
                             unsigned long long* out_len, unsigned long long cap, DevState* st) {
  if (st->flags & (F_STAGE | F_ARCHIVE)) return;
  const unsigned long long n = *len_dev;
  if (n < 10 || rec[0] != 5) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(st, F_STAGE, 140);
    return;
  }
  const int w = rec[1];
  const unsigned long long orig = ld_bytes(rec + 2, 8), body = n - 10;
  const unsigned long long tile = 8ull * w * w;
  if ((w != 1 && w != 2 && w != 4 && w != 8) || body % tile || body < orig || body > cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(st, F_STAGE, 141);
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out_len = orig;
  const int nb = 8 * w;
  const unsigned long long nwords = body / w;
  const uint8_t* q = rec + 10;
  if (w == 1 && (reinterpret_cast<uintptr_t>(out) & 7) == 0) {
    // one 8-byte tile per thread: its 8 plane bytes in, all 8 words out
    const unsigned long long nt = nwords / 8;
    for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
         t += (unsigned long long)gridDim.x * blockDim.x) {
      const uint64_t g = ld_bytes(q + 8 * t, 8);
      uint64_t u = 0;
#pragma unroll
      for (int j = 0; j < 8; j++) u |= (uint64_t)bit_plane(g, j) << (8 * j);
      *reinterpret_cast<uint64_t*>(out + 8 * t) = u;
    }
    return;
  }
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nwords;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long t = i / nb;
    const int j = (int)(i % nb);
    uint64_t u = 0;
    if (w == 1) {
      uint64_t g = 0;
      for (int k = 0; k < 8; k++) g |= (uint64_t)q[t * 8 + k] << (8 * k);
      u = bit_plane(g, j) ;  // the 8x8 transpose is an involution up to order
      // bit_plane(g, j) gathers bit (7-j) of each plane byte -> word j
    } else {
      for (int k = 0; k < nb; k++)
        if (q[t * tile + k * w + j / 8] & (0x80 >> (j % 8))) u |= 1ull << (nb - 1 - k);
    }
    st_bytes(out + i * w, u, w);
  }
}

void launch_bit_decode(const uint8_t* rec, const unsigned long long* len_dev, uint8_t* out,
                       unsigned long long* out_len_dev, unsigned long long cap, DevState* st, cudaStream_t s,
                       int* launches) {
  k_bit_decode<<<PERSIST_CTAS, 256, 0, s>>>(rec, len_dev, out, out_len_dev, cap, st);
  (*launches)++;
}

// TCMS / BIT encoders for the single-stage API
__global__ void k_tcms_encode(const uint8_t* in, const unsigned long long* n_dev, int w, uint8_t* out,
                              unsigned long long* out_len) {
  const unsigned long long n = *n_dev, nw = cdiv(n, w);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = 4;
    out[1] = (uint8_t)w;
    st_bytes(out + 2, n, 8);
    *out_len = 10 + nw * w;
  }
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nw;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    uint64_t u = 0;
    for (int k = 0; k < w; k++)
      if (i * w + k < n) u |= (uint64_t)in[i * w + k] << (8 * k);
    st_bytes(out + 10 + i * w, zz(u, w), w);
  }
}

void launch_tcms_encode(const uint8_t* in, const unsigned long long* n_dev, int width, uint8_t* out,
                        unsigned long long* out_len_dev, unsigned long long max_n, cudaStream_t s, int* launches) {
  k_tcms_encode<<<PERSIST_CTAS, 256, 0, s>>>(in, n_dev, width, out, out_len_dev);
  (*launches)++;
}

__global__ void k_bit_encode(const uint8_t* in, const unsigned long long* n_dev, int w, uint8_t* out,
                             unsigned long long* out_len) {
  const unsigned long long n = *n_dev;
  const unsigned long long tile = 8ull * w * w, padded = cdiv(n, tile) * tile;
  const int nb = 8 * w;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = 5;
    out[1] = (uint8_t)w;
    st_bytes(out + 2, n, 8);
    *out_len = 10 + padded;
  }
  // one thread per output plane byte
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < padded;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long t = i / tile;
    const unsigned long long r = i % tile;
    const int k = (int)(r / w), jb = (int)(r % w);  // plane k, byte jb of the plane
    uint8_t b = 0;
    for (int m = 0; m < 8; m++) {
      const int j = jb * 8 + m;  // word index within the tile
      const unsigned long long o = t * tile + (unsigned long long)j * w;
      uint64_t u = 0;
      for (int q = 0; q < w; q++)
        if (o + q < n) u |= (uint64_t)in[o + q] << (8 * q);
      if ((u >> (nb - 1 - k)) & 1) b |= (uint8_t)(0x80 >> m);
    }
    out[10 + i] = b;
  }
}

void launch_bit_encode(const uint8_t* in, const unsigned long long* n_dev, int width, uint8_t* out,
                       unsigned long long* out_len_dev, unsigned long long max_n, cudaStream_t s, int* launches) {
  k_bit_encode<<<PERSIST_CTAS, 256, 0, s>>>(in, n_dev, width, out, out_len_dev);
  (*launches)++;
}

// -------------------------------------------------------- Huffman decode
// Self-synchronising parallel decode: the payload is cut into S-bit
// subsequences; each thread decodes from a guessed start until it crosses its
// subsequence end, then passes re-decode only where a predecessor's end
// disagrees with the guess (canonical prefix codes resynchronise within a
// few codewords).  An exclusive scan of per-subsequence symbol counts gives
// the output offsets for the final decode.  Decoding uses a 12-bit LUT in
// shared memory plus a canonical slow path for longer codes; when the most
// frequent symbol has the 1-bit code "0" (smooth fields) runs of zero bits
// are consumed with one clz.  Output goes out in aligned 16-byte stores.

// bits per subsequence: 512 for large payloads (throughput), down to 128 when
// 512-bit subsequences would not fill the GPU (a thread's decode chain is the
// latency of a small stream) -- chosen per stream in k_hd_setup
constexpr int HD_S_MAX = 512, HD_S_MIN = 128;
constexpr unsigned long long HD_FILL = 148ull * 4 * 256;  // subsequences that fill the GPU
constexpr int HD_K = 12;         // LUT bits

struct HDTables {
  int ok;
  unsigned S;  // bits per subsequence
  int maxlen, K;
  int run_sym;  // symbol with the 1-bit code "0", or -1
  unsigned long long nsym, nbits, pay_off, pay_len, nsub;
  unsigned long long first_code[64];
  int first_rank[64], count[64];
  uint8_t syms[256];
  uint16_t lut[1 << HD_K];  // (len << 8) | sym, 0 = none
  // multi-symbol table over the same K-bit window: up to 4 complete codewords
  uint32_t msym[1 << HD_K];  // packed symbols, first in the low byte
  uint8_t mmeta[1 << HD_K];  // count | bits << 3
};

// shared-memory copy of the decode tables used per symbol
struct HDShared {
  uint16_t lut[1 << HD_K];
  uint32_t msym[1 << HD_K];
  uint8_t mmeta[1 << HD_K];
};

__device__ __forceinline__ void hd_load_shared(HDShared* S, const HDTables* T) {
  for (int i = threadIdx.x; i < (1 << HD_K); i += blockDim.x) {
    S->lut[i] = T->lut[i];
    S->msym[i] = T->msym[i];
    S->mmeta[i] = T->mmeta[i];
  }
}

struct HDWork {  // per pass: start, end, count per subsequence
  unsigned long long* s[2];
  unsigned long long* e[2];
  unsigned* c[2];
  unsigned long long* off;
  unsigned long long* bmask;  // codeword starts in [i*S, i*S+64) seen by the first pass
  int* changed;               // per pass
  // streams without a 1-bit code (rough): every codeword start of the first
  // pass, S bits per subsequence (8 words), so a fix-up syncs anywhere
  unsigned long long* bmfull;
  // chain tables (rough streams only): for the subsequences of a window after
  // each chain head, the decode from every possible start offset d < HD_TD
  // (end, count); capacity HD_TCAP rows of HD_TD entries
  unsigned long long* tend;
  unsigned* tcnt;
};
constexpr int HD_TD = 32;                 // start offsets tabulated per subsequence
constexpr unsigned HD_TCAP = 1u << 16;    // table rows (subsequences) per round

// stages.py:332-368: record checks, Kraft, canonical tables, LUT (parallel)
__global__ void __launch_bounds__(256) k_hd_setup(const uint8_t* rec, const unsigned long long* len_dev,
                                                  unsigned long long n_expect, unsigned long long max_out,
                                                  unsigned long long nsub_cap, HDTables* T, DevState* st) {
  __shared__ int ok_sh, cnt[257], maxlen_sh, ns_sh;
  __shared__ uint8_t len[256];
  // shared copies of the canonical tables for the parallel LUT builds below
  __shared__ unsigned long long s_first[64];
  __shared__ int s_rank[64], s_count[64];
  __shared__ uint8_t s_syms[256];
  __shared__ uint16_t s_lut[1 << HD_K];
  const int t = threadIdx.x;
  if (t == 0) {
    T->ok = 0;
    ok_sh = 0;
    maxlen_sh = 0;
    do {
      if (st->flags & (F_STAGE | F_ARCHIVE)) break;
      const unsigned long long n = *len_dev;
      if (n < 10 || rec[0] != 1) { raise_flag(st, F_STAGE, 150); break; }
      const int w = rec[1];
      if (w != 1 && w != 2 && w != 4 && w != 8) { raise_flag(st, F_STAGE, 151); break; }
      if (w != 1) { raise_flag(st, F_STAGE, 152); break; }
      if (n < 10 + 8 + 256) { raise_flag(st, F_STAGE, 153); break; }
      const unsigned long long nsym = ld_bytes(rec + 2, 8), nbits = ld_bytes(rec + 10, 8);
      const unsigned long long plen = n - 274;
      if (n_expect != ~0ull && nsym != n_expect) { raise_flag(st, F_ARCHIVE, 159); break; }
      if (nsym > max_out) { raise_flag(st, F_STAGE, 159); break; }
      T->nsym = nsym;
      T->nbits = nbits;
      T->pay_off = 274;
      T->pay_len = plen;
      st->hd_nsym = nsym;
      if (nsym == 0) {
        if (nbits || plen) { raise_flag(st, F_STAGE, 154); break; }
        T->nsub = 0;
        T->ok = 1;
        break;
      }
      if (nbits / 8 + (nbits % 8 != 0) != plen) { raise_flag(st, F_STAGE, 155); break; }
      if (nbits == 0) { raise_flag(st, F_STAGE, 155); break; }
      ok_sh = 1;
    } while (0);
  }
  __syncthreads();
  if (!ok_sh) return;
  len[t] = rec[18 + t];
  cnt[t] = 0;
  if (t == 0) cnt[256] = 0, ns_sh = 0;
  if (t < 64) s_rank[t] = -1, s_count[t] = 0, s_first[t] = 0;
  __syncthreads();
  if (len[t]) {
    atomicAdd(&cnt[len[t]], 1);
    atomicMax(&maxlen_sh, (int)len[t]);
    atomicAdd(&ns_sh, 1);
  }
  __syncthreads();
  const int maxlen = maxlen_sh;
  if (t == 0) {
    bool good = ns_sh > 0;
    if (!good) raise_flag(st, F_STAGE, 156);
    long long avail = 1;
    for (int L = 1; L <= maxlen && good; L++) {  // Kraft, exact with a cap
      avail = avail * 2 - cnt[L];
      if (avail < 0) {
        raise_flag(st, F_STAGE, 157);
        good = false;
      }
      if (avail > 1024) avail = 1024;
    }
    if (good && maxlen > 56) {
      raise_flag(st, F_UNSUPPORTED, 158);
      good = false;
    }
    if (good) {
      unsigned long long next = 0;
      int prev = 0, r = 0;
      for (int L = 1; L <= maxlen; L++) {
        if (!cnt[L]) continue;
        next <<= (L - prev);
        prev = L;
        s_rank[L] = r;
        s_first[L] = next;
        s_count[L] = cnt[L];
        next += cnt[L];
        r += cnt[L];
      }
      T->maxlen = maxlen;
      T->K = maxlen < HD_K ? maxlen : HD_K;
      unsigned S = HD_S_MAX;
      while (S > HD_S_MIN && T->nbits / S < HD_FILL && cdiv(T->nbits, (unsigned long long)(S / 2)) + 1 <= nsub_cap)
        S >>= 1;
      T->S = S;
      T->nsub = cdiv(T->nbits, (unsigned long long)S);
    }
    ok_sh = good;
  }
  __syncthreads();
  if (!ok_sh) return;
  if (t < 64) T->first_rank[t] = s_rank[t], T->count[t] = s_count[t], T->first_code[t] = s_first[t];
  // sorted symbol list: rank of symbol t among (len, sym)
  if (len[t]) {
    int r = 0;
    for (int L = 1; L < len[t]; L++) r += cnt[L];
    for (int j = 0; j < t; j++) r += len[j] == len[t];
    T->syms[r] = (uint8_t)t;
    s_syms[r] = (uint8_t)t;
  }
  __syncthreads();
  const int K = maxlen < HD_K ? maxlen : HD_K;
  for (int e = t; e < (1 << HD_K); e += 256) {
    uint16_t v = 0;
    if (e < (1 << K)) {
      for (int L = 1; L <= K; L++) {  // codes of <= HD_K bits: 32-bit canonical test
        const unsigned c = (unsigned)e >> (K - L), d = c - (unsigned)s_first[L];
        if (d < (unsigned)s_count[L]) {
          v = (uint16_t)((L << 8) | s_syms[s_rank[L] + (int)d]);
          break;
        }
      }
    }
    T->lut[e] = v;
    s_lut[e] = v;
  }
  __syncthreads();
  // multi-symbol entries: greedy decode of the codewords wholly inside the window
  for (int e = t; e < (1 << HD_K); e += 256) {
    uint32_t packed = 0;
    int n = 0, used = 0;
    if (e < (1 << K)) {
      while (n < 4) {
        const int rem = K - used;
        if (rem <= 0) break;
        const uint16_t v = s_lut[((unsigned)e << used) & ((1u << K) - 1)];
        const int L = v >> 8;
        if (!v || L > rem) break;
        packed |= (uint32_t)(v & 0xFF) << (8 * n);
        n++;
        used += L;
      }
    }
    T->msym[e] = packed;
    T->mmeta[e] = (uint8_t)(n | (used << 3));
  }
  if (t == 0) {
    T->run_sym = (s_count[1] > 0 && s_first[1] == 0) ? s_syms[s_rank[1]] : -1;
    __threadfence();
    T->ok = 1;
  }
}

// MSB-first bit reader over the payload: refills 32 bits at a time from
// aligned big-endian words (one load per 32 bits instead of one per byte).
// Invariant after every operation: nb >= 33 valid bits at the top of buf.
struct BitReader {
  const uint32_t* w;          // aligned word base (at or just before the payload)
  unsigned long long wi, nw;  // next word, words holding payload bytes
  unsigned long long endb;    // payload end in bytes from w
  uint64_t buf;               // MSB-aligned
  int nb;
  __device__ __forceinline__ uint32_t word(unsigned long long i) const {
    if (i + 1 < nw) return __byte_perm(__ldg(w + i), 0, 0x0123);
    // the last (possibly partial) word: byte loads, nothing past the payload
    const uint8_t* b = reinterpret_cast<const uint8_t*>(w);
    uint32_t x = 0;
    for (int k = 0; k < 4; k++) {
      const unsigned long long j = 4 * i + k;
      x = (x << 8) | (j < endb ? b[j] : 0u);
    }
    return x;
  }
  __device__ void init(const uint8_t* pay, unsigned long long plen, unsigned long long pos) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(pay);
    const int sh = (int)(a & 3);
    w = reinterpret_cast<const uint32_t*>(a - sh);
    endb = plen + sh;
    nw = (endb + 3) >> 2;
    const unsigned long long bp = pos + 8ull * sh;
    wi = bp >> 5;
    buf = 0;
    nb = 0;
    refill();
    const int skip = (int)(bp & 31);
    buf <<= skip;
    nb -= skip;
    if (nb <= 32) refill();
  }
  __device__ __forceinline__ void refill() {
    while (nb <= 32) {
      const uint32_t x = wi < nw ? word(wi) : 0u;
      buf |= (uint64_t)x << (32 - nb);
      nb += 32;
      wi++;
    }
  }
  // top L (<= 64) bits, also when L exceeds the buffered bits
  __device__ __forceinline__ uint64_t peek(int L) const {
    if (L <= nb) return buf >> (64 - L);
    const uint64_t x = wi < nw ? word(wi) : 0u;
    return (buf | (x >> (nb - 32))) >> (64 - L);
  }
  __device__ __forceinline__ void consume(int L) {
    if (L < nb) {
      buf <<= L;
      nb -= L;
    } else {  // L >= nb: drop the buffer and skip the rest of L in the next word
      const int skip = L - nb;
      buf = 0;
      nb = 0;
      refill();
      buf <<= skip;
      nb -= skip;
    }
    if (nb <= 32) refill();
  }
};

// 16-byte aligned output writer for one thread's contiguous output range.
// The current window is pre-filled with the run symbol, so a run of that
// symbol only advances the position; other bytes replace their slots.
struct OutWriter {
  uint8_t* out;
  unsigned long long start, p;
  uint64_t lo, hi, rep;
  unsigned zeros;
  __device__ void init(uint8_t* o, unsigned long long s, int fill) {
    out = o;
    start = p = s;
    rep = 0x0101010101010101ull * (uint64_t)(fill & 0xFF);
    lo = hi = rep;
    zeros = 0;
  }
  __device__ __forceinline__ void flush_chunk(unsigned long long base, int upto) {  // bytes [base, base+upto)
    if (base >= start && upto == 16) {
      *reinterpret_cast<uint4*>(out + base) = make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi,
                                                        (uint32_t)(hi >> 32));
    } else {
      for (int k = 0; k < upto; k++) {
        if (base + k < start) continue;
        out[base + k] = (uint8_t)(k < 8 ? (lo >> (8 * k)) : (hi >> (8 * (k - 8))));
      }
    }
    lo = hi = rep;
  }
  // advance over z bytes equal to the fill byte: complete windows go out as
  // they are crossed (the ones wholly inside the run are pure fill)
  __device__ __forceinline__ void skip_fill(unsigned long long z) {
    const unsigned long long q = p + z;
    unsigned long long wb = p & ~15ull;
    while (wb + 16 <= q) {
      flush_chunk(wb, 16);
      wb += 16;
    }
    p = q;
  }
  __device__ __forceinline__ void put(int b) {
    const int k = (int)(p & 15);
    const uint64_t m = 0xFFull << (8 * (k & 7));
    const uint64_t v = (uint64_t)(b & 0xFF) << (8 * (k & 7));
    if (k < 8)
      lo = (lo & ~m) | v;
    else
      hi = (hi & ~m) | v;
    p++;
    if (!(p & 15)) flush_chunk(p - 16, 16);
  }
  // n (<= 4) packed bytes, first in the low byte, replacing window bytes
  __device__ __forceinline__ void put4(uint32_t pk, int n) {
    const uint64_t nm = n >= 4 ? 0xFFFFFFFFull : ((1ull << (8 * n)) - 1);
    const uint64_t v = (uint64_t)pk & nm;
    const int k = (int)(p & 15);
    const int e = k + n;  // window bytes [k, e)
    if (k < 8) {
      lo = (lo & ~(nm << (8 * k))) | (v << (8 * k));
      if (e > 8) hi = (hi & ~(nm >> (64 - 8 * k))) | (v >> (64 - 8 * k));  // k > 4 here, shift < 64
    } else {
      hi = (hi & ~(nm << (8 * (k - 8)))) | (v << (8 * (k - 8)));
    }
    p += n;
    if (e >= 16) {
      // window complete: flush, then carry the bytes that spilled past byte 15
      flush_chunk(p - e, 16);
      if (e > 16) {
        const int sp = 8 * (16 - k);
        lo = (rep & ~(nm >> sp)) | (v >> sp);
      }
    }
  }
  // n copies of byte b
  __device__ __forceinline__ void run(int b, unsigned long long n) {
    const uint64_t r = 0x0101010101010101ull * (uint64_t)b;
    while (n) {
      const int k = (int)(p & 15);
      const int take = n < (unsigned long long)(16 - k) ? (int)n : 16 - k;
      const int a = k, e = k + take;  // bytes [a, e) of the window
      const uint64_t mlo = (a < 8) ? ((e >= 8 ? ~0ull : ((1ull << (8 * e)) - 1)) & (~0ull << (8 * a))) : 0ull;
      const uint64_t mhi = (e > 8) ? ((e >= 16 ? ~0ull : ((1ull << (8 * (e - 8))) - 1)) &
                                      (a <= 8 ? ~0ull : (~0ull << (8 * (a - 8)))))
                                   : 0ull;
      lo = (lo & ~mlo) | (r & mlo);
      hi = (hi & ~mhi) | (r & mhi);
      p += take;
      n -= take;
      if (e == 16) flush_chunk(p - 16, 16);
    }
  }
  __device__ void finish() {
    if (p & 15) flush_chunk(p & ~15ull, (int)(p & 15));
  }
};

// Fast loop for streams whose most frequent symbol has the 1-bit code "0"
// (stages.py:293-302 canonical codes: that code is all zeros): consume the
// leading-zero run with one clz, then decode at the '1' bit through the
// multi-symbol table (slow path for long codes / the stop bound).  Returns
// nonzero on a decode error (pos at the failing codeword).
template <bool EMIT>
__device__ __forceinline__ int hd_fast(const HDTables& T, const HDShared* S, BitReader& br, unsigned long long& pos,
                                       const unsigned long long lim, long long& cnt, OutWriter* ow) {
  const int K = T.K, rs = T.run_sym;
  while (pos < lim) {
    unsigned long long z = br.buf ? (unsigned long long)__clzll(br.buf) : 64ull;
    bool capped = false;
    if (z >= (unsigned long long)br.nb) {
      z = br.nb;
      capped = true;
    }
    if (z >= lim - pos) {
      z = lim - pos;
      capped = true;
    }
    if (z) {
      if (EMIT) {
        ow->skip_fill(z);
        if (rs == 0) ow->zeros += (unsigned)z;
      }
      pos += z;
      cnt += (long long)z;
      br.consume((int)z);
    }
    if (capped) continue;  // at the stop bound, or the run goes on past the buffer
    const unsigned key = (unsigned)(br.buf >> (64 - K));
    const uint8_t mm = S->mmeta[key];
    const int n = mm & 7, b = mm >> 3;
    if (n >= 1 && pos + b <= lim) {
      if (EMIT) {
        const uint32_t pk = S->msym[key];
        ow->put4(pk, n);
        const uint32_t live = n >= 4 ? 0xFFFFFFFFu : ((1u << (8 * n)) - 1);
        ow->zeros += (unsigned)__popc(__vcmpeq4(pk, 0u) & live) >> 3;
      }
      pos += b;
      cnt += n;
      br.consume(b);
      continue;
    }
    const uint16_t e = S->lut[key];
    int L, sym;
    if (e) {
      L = e >> 8;
      sym = e & 0xFF;
    } else {
      sym = -1;
      for (L = K + 1; L <= T.maxlen; L++) {
        if (!T.count[L]) continue;
        const unsigned long long c = br.peek(L);
        if (c >= T.first_code[L] && c - T.first_code[L] < (unsigned long long)T.count[L]) {
          sym = T.syms[T.first_rank[L] + (int)(c - T.first_code[L])];
          break;
        }
      }
      if (sym < 0) return 1;
    }
    if (pos + L > T.nbits) return 1;
    if (EMIT) {
      ow->put(sym);
      ow->zeros += sym == 0;
    }
    pos += L;
    cnt++;
    br.consume(L);
  }
  return 0;
}

// decode from `start` while pos < stop (and < nbits); returns symbols or -1 on error.
// MASK: record codeword starts in [start, start+64) into *mask.
// SYNC: stop early at the first codeword start p with (p - sbase) < 64 and
//       bit (p - sbase) of sync_mask set (*endp = p).
template <bool EMIT, bool MASK = false, bool SYNC = false>
__device__ long long hd_decode(const HDTables& T, const HDShared* S, const uint8_t* pay, unsigned long long start,
                               unsigned long long stop, unsigned long long* endp, OutWriter* ow,
                               unsigned long long* mask = nullptr, unsigned long long sbase = 0,
                               unsigned long long sync_mask = 0) {
  BitReader br;
  br.init(pay, T.pay_len, start);
  unsigned long long pos = start;
  long long cnt = 0;
  unsigned long long m = 0;
  const unsigned long long lim = stop < T.nbits ? stop : T.nbits;
  const int K = T.K, rs = T.run_sym;
  while (pos < lim) {
    if (EMIT && !SYNC && rs >= 0) {
      // emitting a smooth stream: every step = one run of the 1-bit code "0"
      // (possibly empty; a pure position advance for the writer) + one table
      // step at the next '1' bit, the same instruction sequence for every lane
      if (hd_fast<EMIT>(T, S, br, pos, lim, cnt, ow)) {
        *endp = pos;
        if (MASK) *mask = m;
        return -1;
      }
      break;
    }
    if (SYNC) {
      const unsigned long long q = pos - sbase;
      if (q >= 64) break;  // no sync inside the window
      if ((sync_mask >> q) & 1) {
        *endp = pos;
        return cnt;
      }
    }
    if (MASK && pos - start < 64) m |= 1ull << (pos - start);
    // run of the 1-bit code "0": long runs in one step; short ones go through
    // the multi-symbol table below (up to 4 codewords per lookup)
    if (rs >= 0 && !(br.buf >> 63) &&
        (SYNC || (MASK && pos - start < 64) || (br.buf >> 56) == 0)) {
      unsigned long long z = br.buf ? (unsigned long long)__clzll(br.buf) : 64ull;
      if (z > (unsigned long long)br.nb) z = br.nb;
      if (z > lim - pos) z = lim - pos;
      if (SYNC) {  // advance one codeword at a time inside the sync window
        z = 1;
      }
      if (MASK) {
        const unsigned long long q = pos - start;
        if (q < 64) m |= (z >= 64 ? ~0ull : ((1ull << z) - 1)) << q;
      }
      if (EMIT) {
        ow->run(rs, z);
        if (rs == 0) ow->zeros += (unsigned)z;
      }
      pos += z;
      cnt += (long long)z;
      br.consume((int)z);
      continue;
    }
    const unsigned key = (unsigned)(br.buf >> (64 - K));
    if (!SYNC && (!MASK || pos - start >= 64)) {  // several short codewords at once, all starting before lim
      const uint8_t mm = S->mmeta[key];
      const int n = mm & 7, b = mm >> 3;
      if (n >= 2 && pos + b <= lim) {
        if (EMIT) {
          const uint32_t pk = S->msym[key];
          ow->put4(pk, n);
          // zero symbols among the n packed bytes
          const uint32_t live = n >= 4 ? 0xFFFFFFFFu : ((1u << (8 * n)) - 1);
          ow->zeros += (unsigned)__popc(__vcmpeq4(pk, 0u) & live) >> 3;
        }
        pos += b;
        cnt += n;
        br.consume(b);
        continue;
      }
    }
    const uint16_t e = S->lut[key];
    int L, sym;
    if (e) {
      L = e >> 8;
      sym = e & 0xFF;
    } else {
      sym = -1;
      for (L = K + 1; L <= T.maxlen; L++) {
        if (!T.count[L]) continue;
        const unsigned long long c = br.peek(L);
        if (c >= T.first_code[L] && c - T.first_code[L] < (unsigned long long)T.count[L]) {
          sym = T.syms[T.first_rank[L] + (int)(c - T.first_code[L])];
          break;
        }
      }
      if (sym < 0) {
        *endp = pos;
        if (MASK) *mask = m;
        return -1;
      }
    }
    if (pos + L > T.nbits) {
      *endp = pos;
      if (MASK) *mask = m;
      return -1;
    }
    if (EMIT) {
      ow->put(sym);
      ow->zeros += sym == 0;
    }
    pos += L;
    cnt++;
    br.consume(L);
  }
  *endp = pos;
  if (MASK) *mask = m;
  if (SYNC) return -2;  // window exhausted without sync (or hit the end): caller re-decodes fully
  return cnt;
}

// length of the codeword at the reader's position, -1 on an invalid code
__device__ __forceinline__ int hd_step(const HDTables& T, const HDShared* S, const BitReader& br) {
  const unsigned key = (unsigned)(br.buf >> (64 - T.K));
  const uint16_t e = S->lut[key];
  if (e) return e >> 8;
  for (int L = T.K + 1; L <= T.maxlen; L++) {
    if (!T.count[L]) continue;
    const unsigned long long c = br.peek(L);
    if (c >= T.first_code[L] && c - T.first_code[L] < (unsigned long long)T.count[L]) return L;
  }
  return -1;
}

// First pass for streams without a 1-bit code: codeword by codeword,
// recording every codeword start of [s0, stop) (bit q of word q/64).
__device__ long long hd_first_full(const HDTables& T, const HDShared* S, const uint8_t* pay, unsigned long long s0,
                                   unsigned long long stop, unsigned long long* endp, unsigned long long* bm) {
  BitReader br;
  br.init(pay, T.pay_len, s0);
  const unsigned long long lim = stop < T.nbits ? stop : T.nbits;
  unsigned long long pos = s0, word = 0;
  long long cnt = 0;
  int cw = 0;
  bool err = false;
  while (pos < lim) {
    const unsigned q = (unsigned)(pos - s0);
    const int w = (int)(q >> 6);
    while (cw < w) {
      bm[cw++] = word;
      word = 0;
    }
    word |= 1ull << (q & 63);
    const int L = hd_step(T, *&S, br);
    if (L < 0 || pos + L > T.nbits) {
      err = true;
      break;
    }
    pos += L;
    cnt++;
    br.consume(L);
  }
  while (cw < HD_S_MAX / 64) {
    bm[cw++] = word;
    word = 0;
  }
  *endp = pos;
  return err ? -1 : cnt;
}

__global__ void __launch_bounds__(256) k_hd_first(const uint8_t* rec, const HDTables* T, HDWork W, DevState* st) {
  __shared__ HDShared S;
  if (!T->ok) return;
  hd_load_shared(&S, T);
  __syncthreads();
  const unsigned long long nsub = T->nsub;
  const unsigned long long SB = T->S;
  const uint8_t* pay = rec + T->pay_off;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nsub;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long s0 = i * SB;
    unsigned long long e, m = 0;
    long long c;
    if (T->run_sym >= 0) {
      c = hd_decode<false, true>(*T, &S, pay, s0, s0 + SB, &e, nullptr, &m);
    } else {
      c = hd_first_full(*T, &S, pay, s0, s0 + SB, &e, W.bmfull + i * (HD_S_MAX / 64));
      m = W.bmfull[i * (HD_S_MAX / 64)];
    }
    W.bmask[i] = m;
    W.s[0][i] = s0;
    W.e[0][i] = c < 0 ? ~0ull : e;  // error end never matches a successor start
    W.e[1][i] = W.e[0][i];          // first-pass ends, read-only during the fix-up's first round
    W.c[0][i] = c < 0 ? 0u : (unsigned)c;
    W.s[1][i] = 0;          // no fix-up round has listed it
  }
}

// exclusive scan of counts (decoupled look-back over 2048-entry tiles staged
// through shared memory: coalesced loads and stores)
constexpr int HS_TILE = 2048;
__global__ void __launch_bounds__(256) k_hd_scan(const HDTables* T, HDWork W, int fin, unsigned long long* lb,
                                                 DevState* st) {
  __shared__ unsigned long long sh[33];
  __shared__ unsigned long long tile_sh, base_sh;
  __shared__ unsigned sc[HS_TILE];
  __shared__ unsigned long long so[HS_TILE];
  if (!T->ok) return;
  const unsigned long long nsub = T->nsub;
  const unsigned long long ntiles = cdiv(nsub, (unsigned long long)HS_TILE);
  const unsigned* c = (fin ? W.c[1] : W.c[0]);
  for (;;) {
    if (threadIdx.x == 0) tile_sh = atomicAdd(lb, 1ull);
    __syncthreads();
    const unsigned long long tile = tile_sh;
    if (tile >= ntiles) break;
    const unsigned long long b0 = tile * HS_TILE;
    for (int k = threadIdx.x; k < HS_TILE; k += blockDim.x) sc[k] = b0 + k < nsub ? c[b0 + k] : 0u;
    __syncthreads();
    unsigned v[8];
    unsigned long long sum = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      v[k] = sc[threadIdx.x * 8 + k];
      sum += v[k];
    }
    unsigned long long total;
    const unsigned long long ex = block_excl_scan<unsigned long long>(sum, sh, &total);
    if (threadIdx.x < 32) {
      const unsigned long long ex_ = lookback_warp(lb + 1, tile, total);
      if (threadIdx.x == 0) base_sh = ex_;
    }
    __syncthreads();
    unsigned long long r = base_sh + ex;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      so[threadIdx.x * 8 + k] = r;
      r += v[k];
    }
    __syncthreads();
    for (int k = threadIdx.x; k < HS_TILE; k += blockDim.x)
      if (b0 + k < nsub) W.off[b0 + k] = so[k];
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      const unsigned long long tot = base_sh + total;
      if (tot != T->nsym) raise_flag(st, F_STAGE, 160);
      if ((fin ? W.e[1] : W.e[0])[nsub - 1] != T->nbits) raise_flag(st, F_STAGE, 161);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256, 4) k_hd_emit(const uint8_t* rec, const HDTables* T, HDWork W, int fin,
                                                 uint8_t* out, DevState* st) {
  __shared__ HDShared S;
  if (!T->ok) return;
  if (st->flags & F_STAGE) return;
  hd_load_shared(&S, T);
  __syncthreads();
  const unsigned long long nsub = T->nsub;
  const unsigned long long SB = T->S;
  const uint8_t* pay = rec + T->pay_off;
  unsigned zeros = 0;
  bool bad = false;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nsub;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long s0 = (fin ? W.s[1] : W.s[0])[i];
    const unsigned long long want = i == 0 ? 0ull : (fin ? W.e[1] : W.e[0])[i - 1];
    if (want != s0 || (fin ? W.e[1] : W.e[0])[i] == ~0ull) {
      bad = true;
      continue;
    }
    OutWriter ow;
    ow.init(out, W.off[i], T->run_sym >= 0 ? T->run_sym : 0);
    unsigned long long e;
    const long long c = hd_decode<true>(*T, &S, pay, s0, (i + 1) * SB, &e, &ow);
    ow.finish();
    zeros += ow.zeros;
    bad |= c < 0;
  }
  zeros = warp_sum<unsigned>(zeros);
  if ((threadIdx.x & 31) == 0 && zeros) atomicAdd(&st->zero_count, (unsigned long long)zeros);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) raise_flag(st, F_STAGE, 162);
}

// In-place fix-up, iterated to convergence inside one cooperative launch:
// every round re-decodes the subsequences whose start disagrees with their
// predecessor's end (the first round from the first pass's codeword starts
// via the 64-bit sync window), then a grid-wide barrier.  A stale read of a
// predecessor's end only delays a fix by one round; each round fixes at least
// the first inconsistent subsequence, so the loop terminates.  Replaces a
// fixed number of passes + a serial sweep (that sweep cost 0.36 s on a rough
// 512^3 field whose corrections cascade over many subsequences).
constexpr int HD_ROUNDS = 1000;  // then the serial sweep (adversarial streams only)

__device__ __forceinline__ void hd_grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(const_cast<unsigned*>(gen), 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Fix-up round 1 (its own launch: every subsequence independent, full
// occupancy): each subsequence whose first-pass start disagrees with its
// predecessor's first-pass end is decoded from that end until it meets one
// of the first pass's codeword starts (64-bit window), else re-decoded fully.
__global__ void __launch_bounds__(256, 4) k_hd_fix1(const uint8_t* rec, const HDTables* T, HDWork W) {
  __shared__ HDShared S;
  if (!T->ok) return;
  hd_load_shared(&S, T);
  __syncthreads();
  const unsigned long long nsub = T->nsub;
  const unsigned long long SB = T->S;
  const uint8_t* pay = rec + T->pay_off;
  volatile unsigned long long* E = W.e[0];
  auto redecode = [&](unsigned long long i, unsigned long long want) {
    unsigned long long e = want;
    long long c = 0;
    if (want < (i + 1) * SB) c = hd_decode<false>(*T, &S, pay, want, (i + 1) * SB, &e, nullptr);
    W.c[0][i] = c < 0 ? 0u : (unsigned)c;
    W.s[0][i] = want;
    E[i] = c < 0 ? ~0ull : e;
  };
  // round 1: every subsequence against the first pass; from the true start
  // until it meets one of the first pass's codeword starts (64-bit window)
  // (predecessor ends are read from the first pass's copy: no thread sees a
  // half-updated neighbour, so every subsequence whose predecessor
  // resynchronised comes out exact)
  const unsigned long long* E1 = W.e[1];
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nsub;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long want = i == 0 ? 0ull : E1[i - 1];
    const unsigned long long s0 = W.s[0][i];
    if (want == s0 || want == ~0ull) continue;
    bool done = false;
    if (T->run_sym < 0 && E1[i] != ~0ull && want >= i * SB) {
      // decode from the true start until a first-pass codeword start anywhere
      // in the subsequence; reaching the end without one IS the full re-decode
      const unsigned long long* bw = W.bmfull + i * (HD_S_MAX / 64);
      const unsigned long long lim = (i + 1) * SB < T->nbits ? (i + 1) * SB : T->nbits;
      BitReader br;
      br.init(pay, T->pay_len, want);
      unsigned long long pos = want, cur = 0;
      int cw = -1;
      unsigned k = 0, before = 0;
      bool synced = false, err = false;
      while (pos < lim) {
        const unsigned q = (unsigned)(pos - i * SB);
        if ((int)(q >> 6) != cw) {  // entering word q/64: count the first pass's starts of the words before it
          for (int x = cw < 0 ? 0 : cw; x < (int)(q >> 6); x++) before += __popcll(bw[x]);
          cw = (int)(q >> 6);
          cur = bw[cw];
        }
        if ((cur >> (q & 63)) & 1) {
          before += __popcll(cur & ((1ull << (q & 63)) - 1));
          synced = true;
          break;
        }
        const int L = hd_step(*T, &S, br);
        if (L < 0 || pos + L > T->nbits) {
          err = true;
          break;
        }
        pos += L;
        k++;
        br.consume(L);
      }
      if (synced) {
        W.c[0][i] = W.c[0][i] - before + k;
        W.s[0][i] = want;
      } else {
        W.c[0][i] = err ? 0u : k;
        W.s[0][i] = want;
        E[i] = err ? ~0ull : pos;
      }
      done = true;
    }
    if (!done && E1[i] != ~0ull && want >= i * SB) {
      unsigned long long ps;
      const unsigned long long bm = W.bmask[i];
      const long long k = hd_decode<false, false, true>(*T, &S, pay, want, (i + 1) * SB, &ps, nullptr, nullptr,
                                                        i * SB, bm);
      if (k >= 0) {
        const unsigned long long q = ps - i * SB;
        const unsigned before = __popcll(bm & ((1ull << q) - 1));
        W.c[0][i] = W.c[0][i] - before + (unsigned)k;
        W.s[0][i] = want;
        done = true;
      }
    }
    if (!done) redecode(i, want);
  }
}

__global__ void __launch_bounds__(256) k_hd_fix(const uint8_t* rec, const HDTables* T, HDWork W) {
  __shared__ HDShared S;
  __shared__ int s_n;
  if (!T->ok) return;  // uniform: every block returns
  hd_load_shared(&S, T);
  __syncthreads();
  const unsigned long long nsub = T->nsub;
  const unsigned long long SB = T->S;
  const uint8_t* pay = rec + T->pay_off;
  unsigned* bar = reinterpret_cast<unsigned*>(W.changed + HD_ROUNDS + 2);
  volatile unsigned long long* E = W.e[0];
  const unsigned long long* E1 = W.e[1];
  // rounds >= 2: runs of still inconsistent subsequences are chains (the
  // first pass did not resynchronise before their end, e.g. inside periodic
  // stretches); one thread per chain head walks it sequentially until the
  // stored state agrees again or it reaches the next head (its own walker)
  unsigned long long* wl = W.off;     // work list (the scan's offsets are written later)
  unsigned long long* mark = W.s[1];  // round that listed the subsequence
  const int lane = threadIdx.x & 31;
  const unsigned long long gwarp = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
  for (int r = 2; r <= HD_ROUNDS; r++) {
    hd_grid_barrier(bar, bar + 1, gridDim.x);
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nsub;
         i += (unsigned long long)gridDim.x * blockDim.x) {
      // list chain heads only: inconsistent, with a consistent predecessor
      const unsigned long long want = i == 0 ? 0ull : E[i - 1];
      const bool bad_i = want != ~0ull && want != W.s[0][i];
      bool bad_prev = false;
      if (i > 0) {
        const unsigned long long wp = i == 1 ? 0ull : E[i - 2];
        bad_prev = wp != ~0ull && wp != W.s[0][i - 1];
      }
      if (bad_i && !bad_prev) {
        const int k = atomicAdd(&W.changed[r], 1);
        wl[k] = i;
        mark[i] = (unsigned long long)r;
      }
    }
    hd_grid_barrier(bar, bar + 1, gridDim.x);
    if (threadIdx.x == 0) s_n = *(volatile int*)&W.changed[r];
    __syncthreads();
    const int n = s_n;
    if (n == 0) return;
    // Chains: the first pass never resynchronised inside them (periodic
    // stretches of rough streams), so fixing them is sequential.  Every
    // subsequence of a window of `win` after each head is first decoded from
    // EVERY start offset d < HD_TD in parallel (the true start of a
    // subsequence is its predecessor's end, within maxlen bits of its
    // nominal start); one warp per chain then walks the window with table
    // lookups -- 8 subsequences per memory round trip -- instead of one
    // re-decode per subsequence.  A chain longer than the window is picked up
    // again by the next round's listing.
    const unsigned win = (unsigned)max(8, min(256, (int)(HD_TCAP / (unsigned)n)) & ~7);  // whole batches of 8
    const unsigned long long tabn = (unsigned long long)min((unsigned)n, HD_TCAP / win) * win * HD_TD;
    for (unsigned long long x = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; x < tabn;
         x += (unsigned long long)gridDim.x * blockDim.x) {
      const int d = (int)(x % HD_TD);
      const unsigned long long row = x / HD_TD, k = row / win, jj = wl[k] + row % win;
      unsigned long long e = ~0ull;
      unsigned c = 0;
      if (jj < nsub && d < T->maxlen) {
        const unsigned long long st0 = jj * SB + d;
        e = st0;
        long long cc = 0;
        if (st0 < (jj + 1) * SB) cc = hd_decode<false>(*T, &S, pay, st0, (jj + 1) * SB, &e, nullptr);
        if (cc < 0) e = ~0ull;
        c = cc < 0 ? 0u : (unsigned)cc;
      }
      W.tend[x] = e;
      W.tcnt[x] = c;
    }
    hd_grid_barrier(bar, bar + 1, gridDim.x);
    for (unsigned long long k = gwarp; k < (unsigned long long)n; k += nwarps) {
      const unsigned long long head = wl[k];
      const bool tab = k * win * HD_TD < tabn;
      unsigned long long t = head == 0 ? 0ull : E[head - 1];  // true start of the current subsequence
      bool stop = t == ~0ull;
      for (unsigned b0 = 0; !stop && b0 < win; b0 += 8) {
        // lane l: table entry d = l of the batch's 8 subsequences, and their stored starts / marks
        unsigned long long te[8], sst = ~0ull, est = ~0ull, mk = 0;
        unsigned tc[8];
#pragma unroll
        for (int b = 0; b < 8; b++) {
          const unsigned long long row = k * win + b0 + b;
          te[b] = tab ? W.tend[row * HD_TD + lane] : ~0ull;
          tc[b] = tab ? W.tcnt[row * HD_TD + lane] : 0u;
        }
        // lanes 0..8: stored starts of the batch and its successor; 0..7: stored ends, marks
        if (lane < 9 && head + b0 + lane < nsub) {
          sst = W.s[0][head + b0 + lane];
          if (lane < 8) {
            est = E[head + b0 + lane];
            mk = mark[head + b0 + lane];
          }
        }
#pragma unroll
        for (int b = 0; b < 8; b++) {
          const unsigned long long jj = head + b0 + b;
          const unsigned long long S_ = __shfl_sync(0xffffffffu, sst, b), S1 = __shfl_sync(0xffffffffu, sst, b + 1),
                                   E_ = __shfl_sync(0xffffffffu, est, b), M_ = __shfl_sync(0xffffffffu, mk, b);
          if (stop) continue;
          if (jj >= nsub || b0 + b >= win || (jj != head && M_ == (unsigned long long)r) || t == ~0ull) {
            stop = true;  // end of the stream / window, or the next head (its own walker)
            continue;
          }
          unsigned long long e;
          if (t == S_) {
            e = E_;  // decoded from its true start already: its end stands
            if (e == S1) {  // and the successor agrees too: chain resolved
              stop = true;
              continue;
            }
          } else {
            const unsigned long long d = t - jj * SB;
            const int src = d < (unsigned long long)HD_TD ? (int)d : 0;
            e = __shfl_sync(0xffffffffu, te[b], src);
            unsigned c = __shfl_sync(0xffffffffu, tc[b], src);
            if (lane == 0) {
              if (!tab || t < jj * SB || d >= (unsigned long long)HD_TD || e == ~0ull) {  // not tabulated: decode
                long long cc = 0;
                e = t;
                if (t < (jj + 1) * SB) cc = hd_decode<false>(*T, &S, pay, t, (jj + 1) * SB, &e, nullptr);
                if (cc < 0) e = ~0ull;
                c = cc < 0 ? 0u : (unsigned)cc;
              }
              // (no fence: only this walker touches the chain; the next
              // round reads it after a grid barrier)
              W.c[0][jj] = c;
              W.s[0][jj] = t;
              E[jj] = e;
            }
            e = __shfl_sync(0xffffffffu, e, 0);
          }
          if (jj + 1 >= nsub || e == ~0ull) {
            stop = true;
            continue;
          }
          t = e;
        }
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) W.changed[HD_ROUNDS + 1] = 1;  // not converged: serial sweep
}

// serial fallback when the fix-up rounds did not converge (adversarial streams)
__global__ void k_hd_serial(const uint8_t* rec, const HDTables* T, HDWork W, int fin) {
  if (!T->ok || !W.changed[HD_ROUNDS + 1]) return;
  const unsigned long long nsub = T->nsub;
  const unsigned long long SB = T->S;
  const uint8_t* pay = rec + T->pay_off;
  for (unsigned long long i = 1; i < nsub; i++) {
    const unsigned long long want = (fin ? W.e[1] : W.e[0])[i - 1];
    if (want == ~0ull) {
      (fin ? W.e[1] : W.e[0])[i] = ~0ull;
      continue;
    }
    if (want == (fin ? W.s[1] : W.s[0])[i]) continue;
    unsigned long long e = want;
    long long c = 0;
    if (want < (i + 1) * SB)
      c = hd_decode<false>(*T, reinterpret_cast<const HDShared*>(T->lut), pay, want, (i + 1) * SB, &e, nullptr);
    (fin ? W.s[1] : W.s[0])[i] = want;
    (fin ? W.e[1] : W.e[0])[i] = c < 0 ? ~0ull : e;
    (fin ? W.c[1] : W.c[0])[i] = c < 0 ? 0u : (unsigned)c;
  }
}

// subsequence slots: every stream fits at 512 bits; short ones may use
// smaller subsequences up to the GPU-filling count
static unsigned long long hd_nsub_cap(unsigned long long max_payload_bytes) {
  const unsigned long long at_max = cdiv(max_payload_bytes * 8, (unsigned long long)HD_S_MAX) + 1;
  return at_max > 4 * HD_FILL ? at_max : 4 * HD_FILL;
}

size_t huffman_decode_ws_bytes(unsigned long long max_payload_bytes) {
  const unsigned long long nsub = hd_nsub_cap(max_payload_bytes);
  return sizeof(HDTables) + 256 + ((HD_ROUNDS + 8) * 4 + 256) + nsub * (8 * 2 + 8 * 2 + 4 * 2 + 8 + 8) + 64 +
         (size_t)HD_TCAP * HD_TD * 12 + 64 + nsub * (HD_S_MAX / 8);
}

void launch_huffman_decode_impl(const uint8_t* hf_rec, const unsigned long long* len_dev, unsigned long long n,
                                unsigned long long max_out, unsigned long long max_payload, uint8_t* seq, void* ws,
                                unsigned long long* lb_ws, DevState* st, cudaStream_t s, int* launches) {
  const unsigned long long nsub_max = hd_nsub_cap(max_payload);
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  HDTables* T = reinterpret_cast<HDTables*>(p);
  p += (sizeof(HDTables) + 255) & ~255ull;
  HDWork W;
  W.changed = reinterpret_cast<int*>(p);  // HD_ROUNDS + 4 ints (flags, barrier): zeroed here, the rest of the
  cudaMemsetAsync(W.changed, 0, (HD_ROUNDS + 8) * 4, s);  // workspace is written before it is read
  p += ((HD_ROUNDS + 8) * 4 + 255) & ~255ull;
  for (int b = 0; b < 2; b++) {
    W.s[b] = reinterpret_cast<unsigned long long*>(p);
    p += nsub_max * 8;
    W.e[b] = reinterpret_cast<unsigned long long*>(p);
    p += nsub_max * 8;
  }
  W.off = reinterpret_cast<unsigned long long*>(p);
  p += nsub_max * 8;
  W.bmask = reinterpret_cast<unsigned long long*>(p);
  p += nsub_max * 8;
  for (int b = 0; b < 2; b++) {
    W.c[b] = reinterpret_cast<unsigned*>(p);
    p += nsub_max * 4;
  }
  p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  W.bmfull = reinterpret_cast<unsigned long long*>(p);
  p += nsub_max * HD_S_MAX / 8;
  W.tend = reinterpret_cast<unsigned long long*>(p);
  p += (size_t)HD_TCAP * HD_TD * 8;
  W.tcnt = reinterpret_cast<unsigned*>(p);
  p += (size_t)HD_TCAP * HD_TD * 4;
  k_hd_setup<<<1, 256, 0, s>>>(hf_rec, len_dev, n, max_out, nsub_max, T, st);
  (*launches)++;
  const unsigned g = persist_grid(cdiv(nsub_max, 256));
  k_hd_first<<<g, 256, 0, s>>>(hf_rec, T, W, st);
  (*launches)++;
  k_hd_fix1<<<g, 256, 0, s>>>(hf_rec, T, W);
  (*launches)++;
  {  // every block resident (cooperative launch): the fix-up rounds use a grid barrier
    static const int per_sm = [] {
      int v = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_hd_fix, 256, 0);
      return v < 1 ? 1 : v;
    }();
    const unsigned gf = (unsigned)std::min<unsigned long long>(cdiv(nsub_max, 256), (unsigned long long)kSMs * per_sm);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gf);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_hd_fix, hf_rec, (const HDTables*)T, W);
    (*launches)++;
    if (getenv("HB_DEBUG_HD")) {
      std::vector<int> ch(HD_ROUNDS + 8);
      cudaStreamSynchronize(s);
      cudaMemcpy(ch.data(), W.changed, ch.size() * 4, cudaMemcpyDeviceToHost);
      int rounds = 1;
      for (int i = 2; i <= HD_ROUNDS; i++) rounds += ch[i] != 0;
      unsigned long long nsub = 0;
      cudaMemcpy(&nsub, &T->nsub, 8, cudaMemcpyDeviceToHost);
      fprintf(stderr, "hd_fix: grid %u nsub %llu rounds-with-changes %d serial %d; per round:", gf, nsub, rounds,
              ch[HD_ROUNDS + 1]);
      for (int i = 2; i <= rounds + 1 && i <= 40; i++) fprintf(stderr, " %d", ch[i]);
      fprintf(stderr, "\n");
    }
  }
  const int fin = 0;
  k_hd_serial<<<1, 1, 0, s>>>(hf_rec, T, W, fin);
  (*launches)++;
  k_hd_scan<<<persist_grid(cdiv(nsub_max, (unsigned long long)HS_TILE)), 256, 0, s>>>(T, W, fin, lb_ws, st);
  (*launches)++;
  k_hd_emit<<<g, 256, 0, s>>>(hf_rec, T, W, fin, seq, st);
  (*launches)++;
}

// zero count over a sequence (escape / TP paths)
__global__ void k_count_zeros(const uint8_t* seq, unsigned long long n, DevState* st) {
  unsigned c = 0;
  // aligned 16-byte body, per-byte compare in SIMD-within-a-register
  const unsigned long long head = min(n, (unsigned long long)((16 - (reinterpret_cast<uintptr_t>(seq) & 15)) & 15));
  const unsigned long long n16 = (n - head) / 16;
  const uint4* v = reinterpret_cast<const uint4*>(seq + head);
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint4 x = __ldcs(v + i);
    c += (__popc(__vcmpeq4(x.x, 0u)) + __popc(__vcmpeq4(x.y, 0u)) + __popc(__vcmpeq4(x.z, 0u)) +
          __popc(__vcmpeq4(x.w, 0u))) >> 3;
  }
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    if (i < head || i >= head + 16 * n16) c += seq[i] == 0;
  c = warp_sum<unsigned>(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&st->zero_count, (unsigned long long)c);
}

void launch_count_zeros(const uint8_t* seq, unsigned long long n, DevState* st, cudaStream_t s, int* launches) {
  unsigned long long b = cdiv(n ? n : 1, 256 * 16);
  if (b > PERSIST_CTAS * 2) b = PERSIST_CTAS * 2;
  k_count_zeros<<<(unsigned)b, 256, 0, s>>>(seq, n, st);
  (*launches)++;
}

}  // namespace hb
