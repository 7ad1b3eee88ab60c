/* hibound_b200.h -- C ABI of libhibound_b200.so, the B200 (sm_100a) drop-in for
 * the reference `hibound` compress/decompress hot path.
 *
 * Every entry point replaces one reference interface; the Python package
 * paper_2507_11165_b200 binds them with ctypes exactly as a maintainer of the
 * reference would.  Plain pointers and sizes only.
 *
 * Conventions
 *  - `field`, `out`, `archive` may be device pointers (cudaMalloc / torch
 *    CUDA tensors) or host pointers (pageable or pinned); the library detects
 *    which with cudaPointerGetAttributes and stages host data itself.
 *  - dims are slowest-first (C order, last dim fastest); 2D fields are passed
 *    as (d0, d1, 1) with ndim = 2 (reference field.py:23-29).
 *  - precision is the element size: 4 (f32) or 8 (f64).
 *  - Return codes mirror the reference exception classes (errors.py:4-21):
 *    HB_EFIELD -> FieldError, HB_EBOUND -> DegenerateBoundError,
 *    HB_EARCHIVE -> ArchiveError, HB_ESTAGE -> StageError (a subclass of
 *    ArchiveError).  hb_last_error() gives the message.
 *  - A context is bound to one device and one CUDA stream and is not
 *    thread-safe; distinct contexts are independent (reference calls are
 *    reentrant).  Calls are asynchronous on the stream except for
 *    the single size/status read-back at the end of compress / decompress.
 */
#ifndef HIBOUND_B200_H
#define HIBOUND_B200_H
#include <stddef.h>
#include <stdint.h>
#if defined(__GNUC__)
#define HB_API __attribute__((visibility("default")))
#else
#define HB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HB_OK = 0,
  HB_EARG = 2,        /* ValueError / TypeError in the reference */
  HB_EFIELD = 3,      /* FieldError */
  HB_EBOUND = 4,      /* DegenerateBoundError */
  HB_EARCHIVE = 5,    /* ArchiveError */
  HB_ESTAGE = 7,      /* StageError */
  HB_ECUDA = 8,       /* CUDA error / out of device memory */
  HB_EUNSUPPORTED = 9 /* shape this build does not handle yet */
};

enum { HB_MODE_CR = 0, HB_MODE_TP = 1 };
enum { HB_EB_ABS = 0, HB_EB_REL = 1 };
enum {
  HB_STAGE_HUFFMAN = 1, HB_STAGE_RRE = 2, HB_STAGE_RZE = 3, HB_STAGE_TCMS = 4, HB_STAGE_BIT = 5,
  HB_PIPE_CR = 10, HB_PIPE_TP = 11
};

typedef struct hb_ctx hb_ctx;

/* Archive header summary (archive.py:93-118 + section walk of :174-200). */
typedef struct {
  int mode, precision, ndim, stride, escape;
  uint8_t cfg[4];
  uint64_t dims[3];
  double eb;
  uint64_t anchor_count, outlier_count, stream_len;
  uint64_t anchor_off, outlier_off, stream_off;
} hb_info;

/* context: one device + one stream (0 = a private non-blocking stream) */
HB_API int hb_ctx_create(int device, void* cuda_stream, hb_ctx** out);
HB_API void hb_ctx_destroy(hb_ctx* ctx);
HB_API const char* hb_last_error(const hb_ctx* ctx);
/* kernels launched by the last call (for the bench's gpu_launches claim) */
HB_API uint64_t hb_last_launch_count(const hb_ctx* ctx);

/* Optional per-phase device timing (CUDA events on the context streams) of
 * the last compress / decompress; names are static strings.  enable: 0 off,
 * 1 every phase, 2 only the level passes (level1..4 / rlevel1..4). */
HB_API void hb_profile(hb_ctx* ctx, int enable);
HB_API int hb_last_phases(const hb_ctx* ctx, const char** names, float* ms, int cap);

/* Upper bound of an archive for these dims (header + anchors + every point an
 * outlier + raw-escaped stream). */
HB_API int hb_compress_bound(const uint64_t dims[3], int precision, size_t* max_bytes);

/* hibound.compress(field, ErrorBoundSpec(eb_mode, eb), mode) -> bytes
 * reference: archive.py:41-74 (resolve_error_bound field.py:135, tune
 * tuning.py:168, decompose predictor.py:372, reorder ordering.py:142,
 * pipeline_{cr,tp}_encode stages.py:422/430).  Writes *out_len bytes to out
 * (capacity cap).  abs_eb_out / cfg_out may be NULL. */
HB_API int hb_compress(hb_ctx* ctx, const void* field, int precision, const uint64_t dims[3], int ndim, int eb_mode,
                double eb, int mode, void* out, size_t cap, size_t* out_len, double* abs_eb_out,
                uint8_t cfg_out[4]);

/* field.py:129-132 value_range on the device: min and max of n values (the
 * reference subtracts them in the field dtype); FieldError on NaN/Inf. */
HB_API int hb_value_range(hb_ctx* ctx, const void* field, int precision, uint64_t n, double* vmin, double* vmax);

/* field.py:145-187 quality metrics in one device pass over n values of the
 * original and the reconstruction (device or host pointers):
 *   out[0] = sum((o - r)^2) in numpy's pairwise order (mse = out[0] / n, bit-
 *            identical to np.mean(d * d)),  out[1] = max |o - r|,
 *   out[2] = min(o), out[3] = max(o)  (value_range subtracts them in dtype). */
HB_API int hb_quality(hb_ctx* ctx, const void* orig, const void* recon, int precision, uint64_t n, double out[4]);

/* archive.py:93-118 on host bytes (no device work). */
HB_API int hb_archive_info(const void* host_blob, size_t len, hb_info* info);

/* hibound.decompress(blob) -> Field; reference archive.py:121-171.  Writes
 * prod(dims)*precision bytes to field_out (capacity cap). info may be NULL. */
HB_API int hb_decompress(hb_ctx* ctx, const void* archive, size_t len, void* field_out, size_t cap, hb_info* info);

/* ---- parity hooks: one per reference stage (device or host buffers) ---- */

/* tuning.py:105-150: chosen config bytes + error table errs[(level-1)*4 + i]
 * for CONFIG_CHOICES order (cubic-multidim, cubic-seq1d, linear-multidim,
 * linear-seq1d); NaN for untuned levels. */
HB_API int hb_tune(hb_ctx* ctx, const void* field, int precision, const uint64_t dims[3], double eb, uint8_t cfg_out[4],
            double errs_out[16]);

/* predictor.py:332-375 + ordering.py:142-159 fused: writes the level-grouped
 * code sequence (N bytes), outliers ascending (idx u64, value in field dtype;
 * capacities N) and the anchor grid.  *ocount receives the outlier count. */
HB_API int hb_decompose(hb_ctx* ctx, const void* field, int precision, const uint64_t dims[3], double eb,
                 const uint8_t cfg[4], uint8_t* seq_out, uint64_t* oidx_out, void* oval_out, uint64_t* ocount,
                 void* anchors_out);

/* predictor.py:378-416 + ordering.py:162-179 fused: from the level-grouped
 * sequence (N bytes), outliers and anchors to the field. */
HB_API int hb_reconstruct(hb_ctx* ctx, const uint8_t* seq, const uint64_t* oidx, const void* oval, uint64_t ocount,
                   const void* anchors, int precision, const uint64_t dims[3], int stride, double eb,
                   const uint8_t cfg[4], void* field_out);

/* ordering.py:142-179 on a code grid / sequence of prod(dims) bytes */
HB_API int hb_reorder(hb_ctx* ctx, const uint8_t* codes, const uint64_t dims[3], int stride, uint8_t* seq_out);
HB_API int hb_inverse_reorder(hb_ctx* ctx, const uint8_t* seq, const uint64_t dims[3], int stride, uint8_t* codes_out);

/* stages.py: one stage (HB_STAGE_*, width 1/2/4/8) or a whole pipeline
 * (HB_PIPE_CR / HB_PIPE_TP).  Output capacity cap; *out_len receives the
 * record length. */
HB_API int hb_stage_encode(hb_ctx* ctx, int stage, int width, const void* in, size_t n, void* out, size_t cap,
                    size_t* out_len);
HB_API int hb_stage_decode(hb_ctx* ctx, int stage, const void* in, size_t n, void* out, size_t cap, size_t* out_len);

#ifdef __cplusplus
}
#endif
#endif
