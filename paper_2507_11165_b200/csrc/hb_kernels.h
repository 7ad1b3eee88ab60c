// hb_kernels.h -- host-side launch interface of the device kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "hb_common.cuh"

namespace hb {

// ---------------------------------------------------------------- geometry
// One interpolation level (predictor.py:264-304) seen in its own lattice:
// level L with stride s = 2^(L-1) acts on the grid of D = ceil(d/s) points per
// axis, predicting positions with at least one odd coordinate from the
// all-even ones (the 2s-lattice), exactly like level 1 on a sub-sampled grid.
struct LevelGeom {
  long long d[3];   // global dims
  long long D[3];   // lattice dims ceil(d/s)
  long long Ed[3];  // even-lattice (recon store) dims ceil(d/2)
  long long s;
  int level;         // predictor level (1..top)
  int T[3];          // tile extent in lattice units (even, or 1 on size-1 axes)
  int ntile[3];
  int seq_order[3];  // seq1d axis order from the GLOBAL dims (predictor.py:177)
  // smem class arrays: extents per class mask (bit a = axis a odd)
  int ext[8][3];
  int off[8];        // offsets in doubles; -1 = not stored
  int smem_doubles;
  // LevelMap closed form (ordering.py:68-84) at ordering level L-1
  long long prefix;  // points at coarser ordering levels
  // affine address steps per unit of half-index (kernel-parameter constants)
  long long kl[3];   // field element index
  long long ke[3];   // even-lattice E index
  long long ks0, ks1_odd0, ks1_even0, eyez, ez;  // Eq. 3 slot
};

void make_level_geom(const uint64_t dims[3], int level, LevelGeom* g);

// k_quality.cu: sum of squared differences (numpy pairwise order), max |o - r|,
// min / max of o -> out_dev[4] (field.py:145-187)
size_t quality_scratch_bytes(unsigned long long n);
void launch_quality(const void* orig, const void* recon, int prec, unsigned long long n, void* scratch,
                    double* out_dev, cudaStream_t s, int* launches);

// field dtype tag
enum { P32 = 4, P64 = 8 };

// --- k_predict.cu
void launch_minmax(const void* field, int prec, unsigned long long n, DevState* st, int eb_mode, double mag,
                   cudaStream_t s, int* launches);
void launch_set_eb(DevState* st, double eb, cudaStream_t s, int* launches);
void launch_anchor_init(const void* field, int prec, const uint64_t dims[3], int A, double* E, uint8_t* seq,
                        uint8_t* anchors_out /*byte-addressed, may be unaligned*/, DevState* st, bool count_hist,
                        cudaStream_t s, int* launches);
void launch_level_compress(const LevelGeom& g, const void* field, int prec, double* E, uint8_t* seq,
                           uint32_t* obitmap, DevState* st, cudaStream_t s, int* launches, int cfg = -1,
                           double* scr = nullptr);
void launch_outlier_compact(const uint32_t* obitmap, unsigned long long n, const void* field, int prec,
                            uint8_t* rec_out /*byte addressed*/, uint64_t* oidx_out, void* oval_out,
                            unsigned long long* lb_status, DevState* st, cudaStream_t s, int* launches);
void launch_anchor_load(const uint8_t* anchors /*byte addressed*/, int prec, const uint64_t dims[3], int A,
                        double* E, cudaStream_t s, int* launches);
void launch_level_decompress(const LevelGeom& g, const uint8_t* seq, const uint64_t* oidx, const double* oval,
                             const unsigned long long* ocount_dev, double* E, void* out, int prec, DevState* st,
                             cudaStream_t s, int* launches, int cfg = -1, double* scr = nullptr);
// k_pass.cu: 3D levels as dependency passes (no halo recompute); scr = level-1
// class arrays of level_scratch_bytes(dims).  Returns launches, 0 = not handled.
size_t level_scratch_bytes(const uint64_t dims[3]);
int launch_level_pass_compress(const LevelGeom& g, const void* field, int prec, double* E, uint8_t* seq, uint32_t* obm,
                               double* scr, DevState* st, cudaStream_t s, int cfg);
int launch_level_pass_decompress(const LevelGeom& g, const uint8_t* seq, const uint64_t* oidx, const double* oval,
                                 const unsigned long long* ocount_dev, double* E, void* out, int prec, double* scr,
                                 DevState* st, cudaStream_t s, int cfg);
// k_march.cu: a multidim 3D level in one launch (axis-0 march, rolling plane
// window in shared memory).  Returns launches, 0 = not handled.
int launch_level_march_compress(const LevelGeom& g, const void* field, int prec, double* E, uint8_t* seq,
                                uint32_t* obm, DevState* st, cudaStream_t s, int cfg);
int launch_level_march_decompress(const LevelGeom& g, const uint8_t* seq, const uint64_t* oidx, const double* oval,
                                  const unsigned long long* ocount_dev, double* E, void* out, int prec, DevState* st,
                                  cudaStream_t s, int cfg);
void launch_copy_anchors_out(const uint8_t* anchors, int prec, unsigned long long n, void* out, DevState* st,
                             cudaStream_t s, int* launches);
void launch_outliers_parse(const uint8_t* rec, int prec, unsigned long long count_max,
                           const unsigned long long* count_dev, unsigned long long n, uint64_t* oidx, double* oval,
                           DevState* st, cudaStream_t s, int* launches);
void launch_reorder(const uint8_t* in, const uint64_t dims[3], int stride, uint8_t* out, bool inverse,
                    cudaStream_t s, int* launches);
void level_kernel_smem_init();
// k_level_{c,d}.cu: column kernels (3D) / 64x64x1 tiles (2D); returns the
// number of kernels launched, 0 = shape not handled (use the generic kernel)
int launch_level_tiled_compress(const LevelGeom& g, const void* field, int prec, double* E, uint8_t* seq,
                                 uint32_t* obm, DevState* st, cudaStream_t s, int cfg);
int launch_level_tiled_decompress(const LevelGeom& g, const uint8_t* seq, const uint64_t* oidx, const double* oval,
                                   const unsigned long long* ocount_dev, double* E, void* out, int prec, DevState* st,
                                   cudaStream_t s, int cfg);

// --- k_tune.cu
struct TunePlan {
  int nb;
  int shape[3];
  int top;
  unsigned long long bn;
};
bool tune_supported(const TunePlan& p);
// one launch per level; the CTA that finishes last runs the select (tuning.py:135-140)
// and publishes the level's config byte (also to host_cfg, mapped pinned memory)
size_t tune_ws_bytes(const TunePlan& p);
void launch_tune_level(const TunePlan& p, const void* field, int prec, const uint64_t dims[3],
                       const unsigned long long* origins, int level, double* trials, double* berr, DevState* st,
                       cudaStream_t s, int* launches, uint8_t* host_cfg = nullptr,
                       cudaGraphConditionalHandle cond = 0);
// whole-field blocks too large for shared memory
size_t tune_global_bytes(unsigned long long bn);
int launch_tune_global(const void* field, int prec, const uint64_t dims[3], int top, uint8_t* scratch,
                       DevState* st, cudaStream_t s, int* launches,
                       int (*upload)(void* ctx, void* dev, const void* src, size_t n), void* up_ctx);

// --- k_stages.cu
struct ReduceBufs {
  uint8_t* bitmap[4];
  uint8_t* payload[4];
};
// source kinds for the level-0 reducer of a chain
enum SrcKind { SRC_MEM = 0, SRC_TCMS = 1, SRC_TP = 2 };

void launch_reduce_chain_impl(int stage, int width, int src_kind, const uint8_t* src_ptr,
                              const unsigned long long* len_dev, int tw, unsigned long long max_words,
                              const ReduceBufs& bufs, BmState* bm, uint8_t* rec_out,
                              const unsigned long long* dst_off_dev, unsigned long long* rec_len_dev,
                              unsigned long long* lb_ws, unsigned long long lb_stride, uint8_t* const* dev_ptr_tables,
                              cudaStream_t s, int* launches);
void launch_hist(const uint8_t* in, unsigned long long n, DevState* st, cudaStream_t s, int* launches);
void launch_huffman_build(DevState* st, unsigned long long n, uint8_t* hf_rec, cudaStream_t s, int* launches);
// symbols per Huffman-encode tile (one look-back entry each)
constexpr unsigned long long HE_TILE_SYMS = 4096;
void launch_huffman_encode(const uint8_t* seq, unsigned long long n, uint8_t* hf_rec, unsigned long long* lb_ws,
                           DevState* st, cudaStream_t s, int* launches);
void launch_stream_offset(unsigned long long base, int prec, DevState* st, cudaStream_t s, int* launches);
void launch_archive_tail_impl(uint8_t* arch, unsigned long long base, int prec, const uint8_t* seq,
                              unsigned long long n, const uint8_t* header46, unsigned long long na, DevState* st,
                              cudaStream_t s, int* launches);
// decoders
void launch_reduce_decode_impl(int stage, const uint8_t* rec, const unsigned long long* rec_len_dev,
                               unsigned long long out_cap, uint8_t* out, unsigned long long* out_len_dev,
                               uint8_t* const tmp[4], void* bmdec, unsigned long long* lb_ws,
                               unsigned long long lb_stride, DevState* st, cudaStream_t s, int* launches);
void launch_tcms_decode(const uint8_t* rec, const unsigned long long* rec_len_dev, unsigned long long cap,
                        uint8_t* out, unsigned long long* out_len_dev, DevState* st, cudaStream_t s, int* launches);
void launch_bit_decode(const uint8_t* rec, const unsigned long long* len_dev, uint8_t* out,
                       unsigned long long* out_len_dev, unsigned long long cap, DevState* st, cudaStream_t s,
                       int* launches);
size_t huffman_decode_ws_bytes(unsigned long long max_payload_bytes);
void launch_huffman_decode_impl(const uint8_t* hf_rec, const unsigned long long* len_dev, unsigned long long n_expect,
                                unsigned long long max_out, unsigned long long max_payload, uint8_t* seq, void* ws,
                                unsigned long long* lb_ws, DevState* st, cudaStream_t s, int* launches);
void launch_count_zeros(const uint8_t* seq, unsigned long long n, DevState* st, cudaStream_t s, int* launches);
// single-stage encoders (hb_stage_encode)
void launch_tcms_encode(const uint8_t* in, const unsigned long long* n_dev, int width, uint8_t* out,
                        unsigned long long* out_len_dev, unsigned long long max_n, cudaStream_t s, int* launches);
void launch_bit_encode(const uint8_t* in, const unsigned long long* n_dev, int width, uint8_t* out,
                       unsigned long long* out_len_dev, unsigned long long max_n, cudaStream_t s, int* launches);

}  // namespace hb
