/* hb_oracle.c -- CPU restatement of the reference `hibound` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path and the CPU-baseline leg of bench.py; it is never linked into
 * or called by paper_2507_11165_b200.  It restates the behaviour of
 * /root/reference/pkg/src/hibound (cited as file:line below) in plain C and is
 * pinned to that package's own outputs by tests/golden/ (see
 * tests/test_oracle_golden.py).
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off -fopenmp).  FP
 * contraction must stay off: the reference evaluates every stencil as
 * separately rounded products and sums (predictor.py:221-226).
 */
#include "hb_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ errors */

static __thread char g_err[512];

const char* hbo_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

void hbo_free(void* p) { free(p); }

void hbo_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* --------------------------------------------------------------- utilities */

typedef struct {
  uint8_t* p;
  size_t n, cap;
} buf_t;

static int buf_reserve(buf_t* b, size_t extra) {
  if (b->n + extra <= b->cap) return 0;
  size_t cap = b->cap ? b->cap : 64;
  while (cap < b->n + extra) cap *= 2;
  uint8_t* q = (uint8_t*)realloc(b->p, cap);
  if (!q) return -1;
  b->p = q;
  b->cap = cap;
  return 0;
}
static int buf_put(buf_t* b, const void* src, size_t n) {
  if (buf_reserve(b, n)) return -1;
  if (n) memcpy(b->p + b->n, src, n);
  b->n += n;
  return 0;
}
static int buf_u8(buf_t* b, uint8_t v) { return buf_put(b, &v, 1); }
static int buf_u64(buf_t* b, uint64_t v) {
  uint8_t t[8];
  for (int i = 0; i < 8; i++) t[i] = (uint8_t)(v >> (8 * i));
  return buf_put(b, t, 8);
}
static uint64_t rd_u64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; i++) v |= (uint64_t)p[i] << (8 * i);
  return v;
}
static uint64_t rd_word(const uint8_t* p, int w) {
  uint64_t v = 0;
  for (int i = 0; i < w; i++) v |= (uint64_t)p[i] << (8 * i);
  return v;
}
static void wr_word(uint8_t* p, uint64_t v, int w) {
  for (int i = 0; i < w; i++) p[i] = (uint8_t)(v >> (8 * i));
}

static inline double load_val(const void* v, int prec, uint64_t i) {
  return prec == 4 ? (double)((const float*)v)[i] : ((const double*)v)[i];
}
static inline void store_val(void* v, int prec, uint64_t i, double x) {
  if (prec == 4)
    ((float*)v)[i] = (float)x;
  else
    ((double*)v)[i] = x;
}

/* ------------------------------------------------------- field.py:129-142 */

int hbo_resolve_eb(const void* vals, int prec, uint64_t n, int eb_mode, double mag, double* eb) {
  if (!(isfinite(mag) && mag > 0)) return fail(HBO_EBOUND, "error-bound magnitude must be positive, got %g", mag);
  if (eb_mode == 0) {
    *eb = mag;
    return 0;
  }
  if (n == 0) return fail(HBO_EFIELD, "empty field");
  double rng;
  if (prec == 4) {
    const float* v = (const float*)vals;
    float lo = v[0], hi = v[0];
    for (uint64_t i = 1; i < n; i++) {
      if (v[i] < lo) lo = v[i];
      if (v[i] > hi) hi = v[i];
    }
    volatile float d = hi - lo; /* subtraction in the field dtype (field.py:132) */
    rng = (double)d;
  } else {
    const double* v = (const double*)vals;
    double lo = v[0], hi = v[0];
    for (uint64_t i = 1; i < n; i++) {
      if (v[i] < lo) lo = v[i];
      if (v[i] > hi) hi = v[i];
    }
    rng = hi - lo;
  }
  if (rng == 0.0) return fail(HBO_EBOUND, "relative error bound on a constant field (value range 0)");
  *eb = mag * rng;
  return 0;
}

/* --------------------------------------------------- predictor.py:114-124 */

int hbo_anchor_stride(const uint64_t dims[3]) {
  uint64_t limit = 0;
  for (int a = 0; a < 3; a++)
    if (dims[a] > 1 && (limit == 0 || dims[a] < limit)) limit = dims[a];
  if (limit == 0) limit = 1;
  uint64_t cap = limit < 16 ? limit : 16;
  int s = 1;
  while ((uint64_t)(s * 2) <= cap) s *= 2;
  return s;
}

static int ilog2i(int a) {
  int t = 0;
  while ((1 << (t + 1)) <= a) t++;
  return t;
}

/* ------------------------------------------ stencils, predictor.py:47-52,181-206 */

typedef struct {
  int n;
  int off[4];
  double w[4];
  int order;
} stencil_t;

static const stencil_t ST_CUBIC = {4, {-3, -1, 1, 3}, {-0.0625, 0.5625, 0.5625, -0.0625}, 4};
static const stencil_t ST_QLO = {3, {-1, 1, 3, 0}, {0.375, 0.75, -0.125, 0}, 3};
static const stencil_t ST_QHI = {3, {-3, -1, 1, 0}, {-0.125, 0.75, 0.375, 0}, 3};
static const stencil_t ST_MID = {2, {-1, 1, 0, 0}, {0.5, 0.5, 0, 0}, 2};
static const stencil_t ST_TRAIL = {2, {-3, -1, 0, 0}, {-0.5, 1.5, 0, 0}, 2};
static const stencil_t ST_COPY = {1, {-1, 0, 0, 0}, {1.0, 0, 0, 0}, 1};

static inline const stencil_t* classify(int64_t pos, int64_t d, int64_t s, int linear) {
  int p1 = pos + s < d, m3 = pos >= 3 * s;
  if (linear) return p1 ? &ST_MID : (m3 ? &ST_TRAIL : &ST_COPY);
  int p3 = pos + 3 * s < d;
  if (m3 && p3) return &ST_CUBIC;
  if (!m3 && p3) return &ST_QLO;
  if (m3 && p1) return &ST_QHI;
  if (p1) return &ST_MID;
  if (m3) return &ST_TRAIL;
  return &ST_COPY;
}

typedef struct {
  int64_t d[3];  /* dims of the grid being walked */
  int64_t st[3]; /* element strides */
  int64_t s;     /* level stride 2^(l-1) */
  int linear;
} walk_t;

/* predictor.py:209-231 (one target, one axis) */
static inline double interp_axis(const double* g, const walk_t* w, const int64_t c[3], int a, int* order) {
  const stencil_t* S = classify(c[a], w->d[a], w->s, w->linear);
  int64_t base = c[0] * w->st[0] + c[1] * w->st[1] + c[2] * w->st[2];
  int64_t step = w->s * w->st[a];
  double acc = g[base + S->off[0] * step] * S->w[0];
  for (int i = 1; i < S->n; i++) acc = acc + g[base + S->off[i] * step] * S->w[i];
  *order = S->order;
  return acc;
}

/* predictor.py:234-256 */
static inline double predict(const double* g, const walk_t* w, const int64_t c[3], const int* axes, int k) {
  int o[3];
  double p[3];
  if (k == 1) return interp_axis(g, w, c, axes[0], &o[0]);
  int best = 0;
  for (int i = 0; i < k; i++) {
    p[i] = interp_axis(g, w, c, axes[i], &o[i]);
    if (o[i] > best) best = o[i];
  }
  double num = 0.0;
  int den = 0;
  for (int i = 0; i < k; i++)
    if (o[i] == best) {
      num = num + p[i];
      den++;
    }
  return num / (double)den;
}

/* predictor.py:313-329 (one element) */
static inline int quantize1(double o, double p, double eb, double two_eb, int cast32, double* recon) {
  double err = o - p;
  double q = copysign(floor(fabs(err) / two_eb + 0.5), err);
  int small = fabs(q) <= 127.0;
  double r = p + two_eb * q;
  double stored = cast32 ? (double)(float)r : r;
  int ok = small && (fabs(o - stored) <= eb);
  if (ok) {
    *recon = r;
    return (int)(q + 128.0);
  }
  *recon = o;
  return 0;
}

/* ----------------------------------------------- predictor.py:264-296 */

typedef struct {
  int64_t start[3], step[3], count[3];
  int axes[3];
  int k;
} substep_t;

static int level_steps(const int64_t d[3], int level, int seq1d, substep_t out[7]) {
  int64_t s = (int64_t)1 << (level - 1);
  int n = 0;
  if (seq1d) {
    int order[3] = {0, 1, 2};
    for (int i = 0; i < 3; i++) /* sort by (-d, a) */
      for (int j = i + 1; j < 3; j++)
        if (d[order[j]] > d[order[i]] || (d[order[j]] == d[order[i]] && order[j] < order[i])) {
          int t = order[i];
          order[i] = order[j];
          order[j] = t;
        }
    for (int k = 0; k < 3; k++) {
      int a = order[k];
      substep_t ss;
      for (int j = 0; j < 3; j++) {
        int earlier = 0;
        for (int m = 0; m < k; m++) earlier |= order[m] == j;
        if (j == a) {
          ss.start[j] = s;
          ss.step[j] = 2 * s;
        } else if (earlier) {
          ss.start[j] = 0;
          ss.step[j] = s;
        } else {
          ss.start[j] = 0;
          ss.step[j] = 2 * s;
        }
        ss.count[j] = d[j] > ss.start[j] ? (d[j] - ss.start[j] + ss.step[j] - 1) / ss.step[j] : 0;
      }
      ss.axes[0] = a;
      ss.k = 1;
      if (ss.count[a] > 0) out[n++] = ss;
    }
  } else {
    static const int sets[7][3] = {{0}, {1}, {2}, {0, 1}, {0, 2}, {1, 2}, {0, 1, 2}};
    static const int ks[7] = {1, 1, 1, 2, 2, 2, 3};
    for (int t = 0; t < 7; t++) {
      substep_t ss;
      int empty = 0;
      for (int j = 0; j < 3; j++) {
        int odd = 0;
        for (int m = 0; m < ks[t]; m++) odd |= sets[t][m] == j;
        ss.start[j] = odd ? s : 0;
        ss.step[j] = 2 * s;
        ss.count[j] = d[j] > ss.start[j] ? (d[j] - ss.start[j] + ss.step[j] - 1) / ss.step[j] : 0;
        if (odd && ss.count[j] == 0) empty = 1;
      }
      if (empty) continue;
      ss.k = ks[t];
      for (int m = 0; m < ks[t]; m++) ss.axes[m] = sets[t][m];
      out[n++] = ss;
    }
  }
  return n;
}

/* -------------------------------------------------- predictor.py:332-375 */

int hbo_decompose(const void* vals, int prec, const uint64_t dims[3], double eb, const uint8_t cfg[4],
                  uint8_t* codes, uint64_t* oidx, void* oval, uint64_t* ocount, void* anchors) {
  if (!(isfinite(eb) && eb > 0)) return fail(HBO_EBOUND, "error bound must be positive and finite, got %g", eb);
  int64_t d[3] = {(int64_t)dims[0], (int64_t)dims[1], (int64_t)dims[2]};
  int64_t N = d[0] * d[1] * d[2];
  int A = hbo_anchor_stride(dims), top = ilog2i(A);
  int cast32 = prec == 4;
  double two_eb = 2.0 * eb;
  double* grid = (double*)malloc((size_t)N * sizeof(double));
  if (!grid) return fail(HBO_ENOMEM, "out of memory");
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; i++) grid[i] = load_val(vals, prec, (uint64_t)i);
  memset(codes, 128, (size_t)N);
  walk_t w = {{d[0], d[1], d[2]}, {d[1] * d[2], d[2], 1}, 0, 0};
  for (int level = top; level >= 1; level--) {
    uint8_t b = cfg[level - 1];
    w.s = (int64_t)1 << (level - 1);
    w.linear = b & 1;
    substep_t ss[7];
    int nss = level_steps(d, level, (b >> 1) & 1, ss);
    for (int t = 0; t < nss; t++) {
      substep_t* S = &ss[t];
#pragma omp parallel for schedule(static)
      for (int64_t i0 = 0; i0 < S->count[0]; i0++) {
        int64_t c[3];
        c[0] = S->start[0] + i0 * S->step[0];
        for (int64_t i1 = 0; i1 < S->count[1]; i1++) {
          c[1] = S->start[1] + i1 * S->step[1];
          for (int64_t i2 = 0; i2 < S->count[2]; i2++) {
            c[2] = S->start[2] + i2 * S->step[2];
            int64_t lin = c[0] * w.st[0] + c[1] * w.st[1] + c[2];
            double p = predict(grid, &w, c, S->axes, S->k);
            double o = load_val(vals, prec, (uint64_t)lin), r;
            codes[lin] = (uint8_t)quantize1(o, p, eb, two_eb, cast32, &r);
            grid[lin] = r;
          }
        }
      }
    }
  }
  free(grid);
  /* outliers, ascending linear index (predictor.py:361-365): code 0 never
   * marks an anchor slot, so a linear scan yields the stable-sorted list. */
  uint64_t k = 0;
  for (int64_t i = 0; i < N; i++)
    if (codes[i] == 0) {
      oidx[k] = (uint64_t)i;
      if (prec == 4)
        ((float*)oval)[k] = ((const float*)vals)[i];
      else
        ((double*)oval)[k] = ((const double*)vals)[i];
      k++;
    }
  *ocount = k;
  /* anchors (predictor.py:360) */
  uint64_t j = 0;
  for (int64_t x = 0; x < d[0]; x += A)
    for (int64_t y = 0; y < d[1]; y += A)
      for (int64_t z = 0; z < d[2]; z += A) {
        int64_t lin = (x * d[1] + y) * d[2] + z;
        if (prec == 4)
          ((float*)anchors)[j++] = ((const float*)vals)[lin];
        else
          ((double*)anchors)[j++] = ((const double*)vals)[lin];
      }
  return 0;
}

/* -------------------------------------------------- predictor.py:378-416 */

static int reconstruct_impl(const uint8_t* codes, const uint64_t* oidx, const void* oval, uint64_t ocount,
                            const void* anchors, int prec, const uint64_t dims[3], double eb, const uint8_t cfg[4],
                            void* out, int A) {
  if (!(isfinite(eb) && eb > 0)) return fail(HBO_EBOUND, "error bound must be positive and finite, got %g", eb);
  int64_t d[3] = {(int64_t)dims[0], (int64_t)dims[1], (int64_t)dims[2]};
  int64_t N = d[0] * d[1] * d[2];
  int top = ilog2i(A);
  double two_eb = 2.0 * eb;
  double* grid = (double*)calloc((size_t)N, sizeof(double));
  if (!grid) return fail(HBO_ENOMEM, "out of memory");
  uint64_t j = 0;
  for (int64_t x = 0; x < d[0]; x += A)
    for (int64_t y = 0; y < d[1]; y += A)
      for (int64_t z = 0; z < d[2]; z += A) grid[(x * d[1] + y) * d[2] + z] = load_val(anchors, prec, j++);
  walk_t w = {{d[0], d[1], d[2]}, {d[1] * d[2], d[2], 1}, 0, 0};
  int orphan = 0;
  for (int level = top; level >= 1; level--) {
    uint8_t b = cfg[level - 1];
    w.s = (int64_t)1 << (level - 1);
    w.linear = b & 1;
    substep_t ss[7];
    int nss = level_steps(d, level, (b >> 1) & 1, ss);
    for (int t = 0; t < nss; t++) {
      substep_t* S = &ss[t];
#pragma omp parallel for schedule(static) reduction(| : orphan)
      for (int64_t i0 = 0; i0 < S->count[0]; i0++) {
        int64_t c[3];
        c[0] = S->start[0] + i0 * S->step[0];
        for (int64_t i1 = 0; i1 < S->count[1]; i1++) {
          c[1] = S->start[1] + i1 * S->step[1];
          for (int64_t i2 = 0; i2 < S->count[2]; i2++) {
            c[2] = S->start[2] + i2 * S->step[2];
            int64_t lin = c[0] * w.st[0] + c[1] * w.st[1] + c[2];
            double p = predict(grid, &w, c, S->axes, S->k);
            uint8_t cb = codes[lin];
            double r = p + two_eb * ((double)cb - 128.0);
            if (cb == 0) {
              /* searchsorted (predictor.py:402-406) */
              uint64_t lo = 0, hi = ocount;
              while (lo < hi) {
                uint64_t mid = (lo + hi) / 2;
                if (oidx[mid] < (uint64_t)lin)
                  lo = mid + 1;
                else
                  hi = mid;
              }
              if (lo < ocount && oidx[lo] == (uint64_t)lin)
                r = load_val(oval, prec, lo);
              else
                orphan = 1;
            }
            grid[lin] = r;
          }
        }
      }
      if (orphan) {
        free(grid);
        return fail(HBO_EARCHIVE, "outlier marker without a matching outlier entry");
      }
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; i++) store_val(out, prec, (uint64_t)i, grid[i]);
  free(grid);
  return 0;
}

int hbo_reconstruct(const uint8_t* codes, const uint64_t* oidx, const void* oval, uint64_t ocount,
                    const void* anchors, int prec, const uint64_t dims[3], double eb, const uint8_t cfg[4],
                    void* out) {
  return reconstruct_impl(codes, oidx, oval, ocount, anchors, prec, dims, eb, cfg, out, hbo_anchor_stride(dims));
}

/* -------------------------------------------------------- tuning.py:66-170 */

int hbo_plan_blocks(const uint64_t dims[3], uint64_t* origins, int max, uint64_t shape[3]) {
  uint64_t mn = 0;
  int any = 0;
  for (int a = 0; a < 3; a++)
    if (dims[a] > 1) {
      if (!any || dims[a] < mn) mn = dims[a];
      any = 1;
    }
  if (!any || mn < 17) {
    for (int a = 0; a < 3; a++) shape[a] = dims[a];
    if (max < 1) return -1;
    origins[0] = origins[1] = origins[2] = 0;
    return 1;
  }
  uint64_t cnt[3];
  for (int a = 0; a < 3; a++) {
    shape[a] = dims[a] > 1 ? 17 : 1;
    cnt[a] = dims[a] == 1 ? 1 : (dims[a] - shape[a]) / 16 + 1;
  }
  uint64_t m = cnt[0] * cnt[1] * cnt[2];
  uint64_t total = dims[0] * dims[1] * dims[2];
  uint64_t bp = shape[0] * shape[1] * shape[2];
  uint64_t want = (total * 2 + bp * 1000 - 1) / (bp * 1000);
  if (want < 1) want = 1;
  if (want > m) want = m;
  int n = 0;
  uint64_t prev = (uint64_t)-1;
  for (uint64_t i = 0; i < want; i++) {
    uint64_t ci = want == 1 ? m / 2 : (i * (m - 1)) / (want - 1);
    if (ci == prev) continue; /* sorted set: indices are non-decreasing */
    prev = ci;
    uint64_t o[3];
    o[2] = (ci % cnt[2]) * 16;
    o[1] = ((ci / cnt[2]) % cnt[1]) * 16;
    o[0] = (ci / (cnt[2] * cnt[1])) * 16;
    int ok = 1;
    for (int p = 0; p < n && ok; p++) {
      int sep = 0;
      for (int a = 0; a < 3; a++) {
        uint64_t diff = o[a] > origins[3 * p + a] ? o[a] - origins[3 * p + a] : origins[3 * p + a] - o[a];
        if (diff >= shape[a]) sep = 1;
      }
      if (!sep) ok = 0;
    }
    if (!ok) continue;
    if (n >= max) return -1;
    for (int a = 0; a < 3; a++) origins[3 * n + a] = o[a];
    n++;
  }
  return n;
}

/* numpy pairwise summation of a contiguous f64 array (umath loops, PW_BLOCKSIZE 128) */
static double pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; i++) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise(a, n2) + pairwise(a + n2, n - n2);
}

/* CPython >= 3.12 builtin sum() over floats starting from int 0 (Neumaier) */
static double py_sum(const double* x, int n) {
  if (n == 0) return 0.0;
  double f = 0.0 + x[0], c = 0.0;
  for (int i = 1; i < n; i++) {
    double t = f + x[i];
    if (fabs(f) >= fabs(x[i]))
      c += (f - t) + x[i];
    else
      c += (x[i] - t) + f;
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f += c;
  return f;
}

/* tuning.py:153-165 */
static double trial_level(double* g, const double* orig, const int64_t sh[3], int level, int linear, int seq1d,
                          double eb, int cast32, double* scratch) {
  double total = 0.0, two_eb = 2.0 * eb;
  walk_t w = {{sh[0], sh[1], sh[2]}, {sh[1] * sh[2], sh[2], 1}, (int64_t)1 << (level - 1), linear};
  substep_t ss[7];
  int nss = level_steps(sh, level, seq1d, ss);
  for (int t = 0; t < nss; t++) {
    substep_t* S = &ss[t];
    int64_t n = 0, c[3];
    for (int64_t i0 = 0; i0 < S->count[0]; i0++) {
      c[0] = S->start[0] + i0 * S->step[0];
      for (int64_t i1 = 0; i1 < S->count[1]; i1++) {
        c[1] = S->start[1] + i1 * S->step[1];
        for (int64_t i2 = 0; i2 < S->count[2]; i2++) {
          c[2] = S->start[2] + i2 * S->step[2];
          int64_t lin = c[0] * w.st[0] + c[1] * w.st[1] + c[2];
          double p = predict(g, &w, c, S->axes, S->k), r;
          double o = orig[lin];
          scratch[n++] = fabs(o - p);
          quantize1(o, p, eb, two_eb, cast32, &r);
          g[lin] = r;
        }
      }
    }
    total += pairwise(scratch, n);
  }
  return total;
}

static const uint8_t CONFIG_CHOICES[4] = {0x0, 0x2, 0x1, 0x3}; /* cm, cs, lm, ls (tuning.py:29) */

int hbo_tune(const void* vals, int prec, const uint64_t dims[3], double eb, uint8_t cfg[4], double errs[16]) {
  int maxb = 1 << 20;
  uint64_t* org = (uint64_t*)malloc(sizeof(uint64_t) * 3 * (size_t)maxb);
  if (!org) return fail(HBO_ENOMEM, "out of memory");
  uint64_t shp[3];
  int nb = hbo_plan_blocks(dims, org, maxb, shp);
  if (nb < 1) {
    free(org);
    return fail(HBO_EARG, "block plan failed");
  }
  int64_t sh[3] = {(int64_t)shp[0], (int64_t)shp[1], (int64_t)shp[2]};
  int64_t bn = sh[0] * sh[1] * sh[2];
  int A = hbo_anchor_stride(shp), top = ilog2i(A);
  double* origs = (double*)malloc(sizeof(double) * (size_t)(bn * nb));
  double* states = (double*)malloc(sizeof(double) * (size_t)(bn * nb));
  double* trials = (double*)malloc(sizeof(double) * (size_t)(bn * nb) * 4);
  double* berr = (double*)malloc(sizeof(double) * (size_t)nb * 4);
  if (!origs || !states || !trials || !berr) {
    free(org), free(origs), free(states), free(trials), free(berr);
    return fail(HBO_ENOMEM, "out of memory");
  }
  for (int b = 0; b < nb; b++)
    for (int64_t x = 0; x < sh[0]; x++)
      for (int64_t y = 0; y < sh[1]; y++)
        for (int64_t z = 0; z < sh[2]; z++) {
          uint64_t gl = ((org[3 * b] + x) * dims[1] + org[3 * b + 1] + y) * dims[2] + org[3 * b + 2] + z;
          origs[b * bn + (x * sh[1] + y) * sh[2] + z] = load_val(vals, prec, gl);
        }
  memcpy(states, origs, sizeof(double) * (size_t)(bn * nb));
  for (int i = 0; i < 16; i++) errs[i] = NAN;
  for (int i = 0; i < 4; i++) cfg[i] = 0;
  int cast32 = prec == 4;
  for (int level = top; level >= 1; level--) {
    double e[4];
#pragma omp parallel for schedule(dynamic) collapse(2)
    for (int ci = 0; ci < 4; ci++)
      for (int b = 0; b < nb; b++) {
        double* scratch = (double*)malloc(sizeof(double) * (size_t)bn);
        double* g = trials + ((size_t)ci * nb + b) * bn;
        memcpy(g, states + (size_t)b * bn, sizeof(double) * (size_t)bn);
        uint8_t cb = CONFIG_CHOICES[ci];
        berr[ci * nb + b] = trial_level(g, origs + (size_t)b * bn, sh, level, cb & 1, (cb >> 1) & 1, eb, cast32, scratch);
        free(scratch);
      }
    for (int ci = 0; ci < 4; ci++) e[ci] = py_sum(berr + ci * nb, nb);
    int best = 0;
    for (int ci = 1; ci < 4; ci++)
      if (e[ci] < e[best]) best = ci;
    for (int ci = 0; ci < 4; ci++) errs[(level - 1) * 4 + ci] = e[ci];
    cfg[level - 1] = CONFIG_CHOICES[best];
    memcpy(states, trials + (size_t)best * nb * bn, sizeof(double) * (size_t)(bn * nb));
  }
  free(org), free(origs), free(states), free(trials), free(berr);
  return 0;
}

/* ----------------------------------------------------- ordering.py:24-179 */

typedef struct {
  int64_t d[3];
  int top;
  int64_t sub[5][3];
  int64_t prefix[5];
} lmap_t;

static void lmap_init(lmap_t* m, const uint64_t dims[3], int stride) {
  for (int a = 0; a < 3; a++) m->d[a] = (int64_t)dims[a];
  m->top = ilog2i(stride);
  for (int l = 0; l <= m->top; l++)
    for (int a = 0; a < 3; a++) m->sub[l][a] = (m->d[a] + ((int64_t)1 << l) - 1) >> l;
  for (int l = 0; l <= m->top; l++)
    m->prefix[l] = l == m->top ? 0 : m->sub[l + 1][0] * m->sub[l + 1][1] * m->sub[l + 1][2];
}

static inline int64_t lmap_index(const lmap_t* m, int64_t x, int64_t y, int64_t z) {
  int l = m->top;
  while (l > 0) {
    int64_t msk = ((int64_t)1 << l) - 1;
    if (!(x & msk) && !(y & msk) && !(z & msk)) break;
    l--;
  }
  int64_t gy = m->sub[l][1], gz = m->sub[l][2];
  int64_t X = x >> l, Y = y >> l, Z = z >> l;
  int64_t rank = X * gy * gz + Y * gz + Z;
  if (l < m->top) {
    int64_t ey = (gy + 1) / 2, ez = (gz + 1) / 2;
    rank -= ((X + 1) / 2) * ey * ez;
    if (!(X & 1)) {
      rank -= ((Y + 1) / 2) * ez;
      if (!(Y & 1)) rank -= (Z + 1) / 2;
    }
  }
  return m->prefix[l] + rank;
}

uint64_t hbo_index_of(const uint64_t dims[3], int stride, uint64_t x, uint64_t y, uint64_t z) {
  lmap_t m;
  lmap_init(&m, dims, stride);
  return (uint64_t)lmap_index(&m, (int64_t)x, (int64_t)y, (int64_t)z);
}

int hbo_reorder(const uint8_t* codes, const uint64_t dims[3], int stride, uint8_t* seq) {
  lmap_t m;
  lmap_init(&m, dims, stride);
#pragma omp parallel for schedule(static)
  for (int64_t x = 0; x < m.d[0]; x++)
    for (int64_t y = 0; y < m.d[1]; y++)
      for (int64_t z = 0; z < m.d[2]; z++) seq[lmap_index(&m, x, y, z)] = codes[(x * m.d[1] + y) * m.d[2] + z];
  return 0;
}

int hbo_inverse_reorder(const uint8_t* seq, const uint64_t dims[3], int stride, uint8_t* codes) {
  lmap_t m;
  lmap_init(&m, dims, stride);
#pragma omp parallel for schedule(static)
  for (int64_t x = 0; x < m.d[0]; x++)
    for (int64_t y = 0; y < m.d[1]; y++)
      for (int64_t z = 0; z < m.d[2]; z++) codes[(x * m.d[1] + y) * m.d[2] + z] = seq[lmap_index(&m, x, y, z)];
  return 0;
}

/* ------------------------------------------------------------ stages.py */

#define COMMON 10
#define BM_EXTRA 9
#define MAX_DEPTH 3

static int put_common(buf_t* b, int stage, int width, uint64_t orig) {
  if (buf_u8(b, (uint8_t)stage) || buf_u8(b, (uint8_t)width) || buf_u64(b, orig)) return -1;
  return 0;
}
static int width_ok(int w) { return w == 1 || w == 2 || w == 4 || w == 8; }

static int parse_common(const uint8_t* p, size_t n, int expect, int* width, uint64_t* orig) {
  if (n < COMMON) return fail(HBO_ESTAGE, "truncated stage header");
  if (p[0] != expect) return fail(HBO_ESTAGE, "expected stage %d record, found stage id %d", expect, p[0]);
  if (!width_ok(p[1])) return fail(HBO_ESTAGE, "symbol width must be one of (1, 2, 4, 8), got %d", p[1]);
  *width = p[1];
  *orig = rd_u64(p + 2);
  return 0;
}

/* stages.py:103-118 */
static int tcms_encode(const uint8_t* in, size_t n, int w, buf_t* out) {
  if (!width_ok(w)) return fail(HBO_ESTAGE, "bad width %d", w);
  size_t nw = (n + w - 1) / w;
  if (put_common(out, 4, w, n) || buf_reserve(out, nw * w)) return fail(HBO_ENOMEM, "oom");
  uint64_t top = (uint64_t)(8 * w - 1), mask = w == 8 ? ~0ULL : ((1ULL << (8 * w)) - 1);
  uint8_t tmp[8];
  for (size_t i = 0; i < nw; i++) {
    memset(tmp, 0, 8);
    size_t m = (i + 1) * w <= n ? (size_t)w : n - i * w;
    memcpy(tmp, in + i * w, m);
    uint64_t u = rd_word(tmp, w);
    uint64_t e = ((u << 1) ^ (0 - (u >> top))) & mask;
    wr_word(out->p + out->n, e, w);
    out->n += w;
  }
  return 0;
}

static int tcms_decode(const uint8_t* p, size_t n, buf_t* out) {
  int w;
  uint64_t orig;
  int rc = parse_common(p, n, 4, &w, &orig);
  if (rc) return rc;
  size_t body = n - COMMON;
  if (body % w || body < orig) return fail(HBO_ESTAGE, "tcms record length mismatch");
  if (buf_reserve(out, body)) return fail(HBO_ENOMEM, "oom");
  uint64_t mask = w == 8 ? ~0ULL : ((1ULL << (8 * w)) - 1);
  for (size_t i = 0; i < body / w; i++) {
    uint64_t u = rd_word(p + COMMON + i * w, w);
    uint64_t d = ((u >> 1) ^ (0 - (u & 1))) & mask;
    wr_word(out->p + out->n + i * w, d, w);
  }
  out->n += orig;
  return 0;
}

/* stages.py:126-160 */
static int bit_shuffle(const uint8_t* in, size_t n, int w, buf_t* out) {
  if (!width_ok(w)) return fail(HBO_ESTAGE, "bad width %d", w);
  size_t tile = 8 * (size_t)w * w, nb = 8 * (size_t)w;
  size_t padded = (n + tile - 1) / tile * tile;
  if (put_common(out, 5, w, n) || buf_reserve(out, padded)) return fail(HBO_ENOMEM, "oom");
  uint8_t* o = out->p + out->n;
  memset(o, 0, padded);
  uint8_t tmp[8];
  for (size_t t = 0; t < padded / tile; t++)
    for (size_t j = 0; j < nb; j++) { /* word j of tile t */
      size_t off = t * tile + j * w;
      memset(tmp, 0, 8);
      if (off < n) memcpy(tmp, in + off, off + w <= n ? (size_t)w : n - off);
      uint64_t u = rd_word(tmp, w);
      for (size_t k = 0; k < nb; k++) /* plane k holds bit nb-1-k */
        if ((u >> (nb - 1 - k)) & 1) o[t * tile + k * w + j / 8] |= (uint8_t)(0x80 >> (j % 8));
    }
  out->n += padded;
  return 0;
}

static int bit_unshuffle(const uint8_t* p, size_t n, buf_t* out) {
  int w;
  uint64_t orig;
  int rc = parse_common(p, n, 5, &w, &orig);
  if (rc) return rc;
  size_t body = n - COMMON, tile = 8 * (size_t)w * w, nb = 8 * (size_t)w;
  if (body % tile || body < orig) return fail(HBO_ESTAGE, "bit-shuffle record length mismatch");
  if (buf_reserve(out, body)) return fail(HBO_ENOMEM, "oom");
  const uint8_t* q = p + COMMON;
  for (size_t t = 0; t < body / tile; t++)
    for (size_t j = 0; j < nb; j++) {
      uint64_t u = 0;
      for (size_t k = 0; k < nb; k++)
        if (q[t * tile + k * w + j / 8] & (0x80 >> (j % 8))) u |= 1ULL << (nb - 1 - k);
      wr_word(out->p + out->n + t * tile + j * w, u, w);
    }
  out->n += orig;
  return 0;
}

/* stages.py:165-184 */
static int bitmap_encode(int stage, const uint8_t* in, size_t n, int w, int depth_left, buf_t* out) {
  size_t nw = (n + w - 1) / w;
  uint8_t* words = (uint8_t*)calloc(nw * w + 8, 1);
  uint8_t* bm = (uint8_t*)calloc((nw + 7) / 8 + 1, 1);
  if (!words || !bm) {
    free(words), free(bm);
    return fail(HBO_ENOMEM, "oom");
  }
  if (n) memcpy(words, in, n);
  size_t kept = 0;
  for (size_t i = 0; i < nw; i++) {
    int keep;
    if (stage == 2)
      keep = i == 0 || memcmp(words + i * w, words + (i - 1) * w, w) != 0;
    else {
      keep = 0;
      for (int b = 0; b < w; b++) keep |= words[i * w + b] != 0;
    }
    if (keep) {
      bm[i / 8] |= (uint8_t)(0x80 >> (i % 8));
      kept++;
    }
  }
  size_t bm_len = (nw + 7) / 8;
  buf_t nested = {0};
  int flag = 0;
  if (depth_left > 0 && bm_len > COMMON + BM_EXTRA) {
    int rc = bitmap_encode(2, bm, bm_len, 1, depth_left - 1, &nested);
    if (rc) {
      free(words), free(bm), free(nested.p);
      return rc;
    }
    if (nested.n < bm_len) flag = 1;
  }
  int err = put_common(out, stage, w, n) || buf_u8(out, (uint8_t)flag);
  err = err || buf_u64(out, flag ? nested.n : bm_len);
  err = err || (flag ? buf_put(out, nested.p, nested.n) : buf_put(out, bm, bm_len));
  err = err || buf_reserve(out, kept * w);
  if (!err)
    for (size_t i = 0; i < nw; i++)
      if (bm[i / 8] & (0x80 >> (i % 8))) {
        memcpy(out->p + out->n, words + i * w, w);
        out->n += w;
      }
  free(words), free(bm), free(nested.p);
  return err ? fail(HBO_ENOMEM, "oom") : 0;
}

/* stages.py:187-221 */
static int bitmap_decode(int stage, const uint8_t* p, size_t n, int depth_left, buf_t* out) {
  int w;
  uint64_t orig;
  int rc = parse_common(p, n, stage, &w, &orig);
  if (rc) return rc;
  size_t off = COMMON;
  if (n < off + BM_EXTRA) return fail(HBO_ESTAGE, "truncated bitmap record");
  int flag = p[off];
  uint64_t bm_len = rd_u64(p + off + 1);
  off += BM_EXTRA;
  if (flag != 0 && flag != 1) return fail(HBO_ESTAGE, "invalid bitmap flag %d", flag);
  if (bm_len > n - off) return fail(HBO_ESTAGE, "bitmap section overruns record");
  const uint8_t* bm = p + off;
  size_t bml = (size_t)bm_len;
  off += bml;
  buf_t inner = {0};
  if (flag) {
    if (depth_left <= 0) return fail(HBO_ESTAGE, "bitmap recursion exceeds maximum depth");
    rc = bitmap_decode(2, bm, bml, depth_left - 1, &inner);
    if (rc) {
      free(inner.p);
      return rc;
    }
    bm = inner.p;
    bml = inner.n;
  }
  uint64_t nsym = (orig + (w - orig % w) % w) / w;
  if (bml != (nsym + 7) / 8) {
    free(inner.p);
    return fail(HBO_ESTAGE, "bitmap length does not match symbol count");
  }
  size_t plen = n - off;
  if (plen % w) {
    free(inner.p);
    return fail(HBO_ESTAGE, "payload is not a whole number of symbols");
  }
  uint64_t ones = 0;
  for (uint64_t i = 0; i < nsym; i++) ones += (bm[i / 8] >> (7 - i % 8)) & 1;
  if (ones != plen / w) {
    free(inner.p);
    return fail(HBO_ESTAGE, "payload symbol count does not match bitmap");
  }
  if (stage == 2 && nsym && !(bm[0] & 0x80)) {
    free(inner.p);
    return fail(HBO_ESTAGE, "first-symbol bit must be set");
  }
  if (buf_reserve(out, nsym * w + 8)) {
    free(inner.p);
    return fail(HBO_ENOMEM, "oom");
  }
  const uint8_t* pay = p + off;
  uint8_t* o = out->p + out->n;
  int64_t r = -1;
  for (uint64_t i = 0; i < nsym; i++) {
    int bit = (bm[i / 8] >> (7 - i % 8)) & 1;
    if (stage == 2) {
      r += bit;
      memcpy(o + i * w, pay + r * w, w);
    } else if (bit) {
      r++;
      memcpy(o + i * w, pay + r * w, w);
    } else
      memset(o + i * w, 0, w);
  }
  out->n += orig;
  free(inner.p);
  return 0;
}

/* stages.py:246-287 */
static void huffman_lengths(const uint64_t hist[256], uint8_t len[256]) {
  memset(len, 0, 256);
  /* heap of (freq, id); ids unique so the pop order is fully determined */
  uint64_t hf[512];
  int hid[512], hn = 0;
  int parent[512];
  int nalive = 0, last = -1;
  for (int s = 0; s < 256; s++)
    if (hist[s]) nalive++, last = s;
  if (nalive == 0) return;
  if (nalive == 1) {
    len[last] = 1;
    return;
  }
#define LESS(i, j) (hf[i] < hf[j] || (hf[i] == hf[j] && hid[i] < hid[j]))
#define SWAP(i, j)        \
  do {                    \
    uint64_t tf = hf[i];  \
    int ti = hid[i];      \
    hf[i] = hf[j];        \
    hid[i] = hid[j];      \
    hf[j] = tf;           \
    hid[j] = ti;          \
  } while (0)
  for (int s = 0; s < 256; s++)
    if (hist[s]) {
      int i = hn++;
      hf[i] = hist[s];
      hid[i] = s;
      while (i > 0 && LESS(i, (i - 1) / 2)) {
        SWAP(i, (i - 1) / 2);
        i = (i - 1) / 2;
      }
    }
  int nxt = 256;
  uint64_t popf[2];
  int popi[2];
  while (hn > 1) {
    for (int k = 0; k < 2; k++) {
      popf[k] = hf[0];
      popi[k] = hid[0];
      hn--;
      hf[0] = hf[hn];
      hid[0] = hid[hn];
      int i = 0;
      for (;;) {
        int l = 2 * i + 1, r = l + 1, m = i;
        if (l < hn && LESS(l, m)) m = l;
        if (r < hn && LESS(r, m)) m = r;
        if (m == i) break;
        SWAP(i, m);
        i = m;
      }
    }
    parent[popi[0]] = nxt;
    parent[popi[1]] = nxt;
    int i = hn++;
    hf[i] = popf[0] + popf[1];
    hid[i] = nxt;
    while (i > 0 && LESS(i, (i - 1) / 2)) {
      SWAP(i, (i - 1) / 2);
      i = (i - 1) / 2;
    }
    nxt++;
  }
#undef LESS
#undef SWAP
  int root = hid[0];
  int depth[512];
  depth[root] = 0;
  for (int node = root - 1; node >= 256; node--) depth[node] = depth[parent[node]] + 1;
  for (int s = 0; s < 256; s++)
    if (hist[s]) len[s] = (uint8_t)(depth[parent[s]] + 1);
}

/* canonical codes: symbols sorted by (length, symbol) */
static int canonical(const uint8_t len[256], uint64_t code[256], int syms[256]) {
  int n = 0;
  for (int L = 1; L <= 255; L++)
    for (int s = 0; s < 256; s++)
      if (len[s] == L) syms[n++] = s;
  uint64_t next = 0;
  int prev = 0;
  for (int i = 0; i < n; i++) {
    int L = len[syms[i]];
    int sh = L - prev;
    next = sh >= 64 ? 0 : next << sh;
    code[syms[i]] = next++;
    prev = L;
  }
  return n;
}

static int huffman_encode(const uint8_t* in, size_t n, buf_t* out) {
  uint64_t hist[256] = {0};
  for (size_t i = 0; i < n; i++) hist[in[i]]++;
  uint8_t len[256];
  huffman_lengths(hist, len);
  uint64_t code[256] = {0};
  int syms[256];
  canonical(len, code, syms);
  uint64_t total = 0;
  for (int s = 0; s < 256; s++) total += hist[s] * len[s];
  if (put_common(out, 1, 1, n) || buf_u64(out, n ? total : 0) || buf_put(out, len, 256))
    return fail(HBO_ENOMEM, "oom");
  if (n == 0) return 0;
  size_t nbytes = (size_t)((total + 7) / 8);
  if (buf_reserve(out, nbytes)) return fail(HBO_ENOMEM, "oom");
  uint8_t* o = out->p + out->n;
  memset(o, 0, nbytes);
  uint64_t pos = 0;
  for (size_t i = 0; i < n; i++) {
    int L = len[in[i]];
    uint64_t c = code[in[i]];
    for (int b = L - 1; b >= 0; b--, pos++)
      if (b < 64 && ((c >> b) & 1)) o[pos >> 3] |= (uint8_t)(0x80 >> (pos & 7));
  }
  out->n += nbytes;
  return 0;
}

/* stages.py:332-417 */
static int huffman_decode(const uint8_t* p, size_t n, buf_t* out) {
  int w;
  uint64_t nsym;
  int rc = parse_common(p, n, 1, &w, &nsym);
  if (rc) return rc;
  if (w != 1) return fail(HBO_ESTAGE, "huffman records use width 1");
  if (n < COMMON + 8 + 256) return fail(HBO_ESTAGE, "truncated huffman header");
  uint64_t nbits = rd_u64(p + COMMON);
  const uint8_t* len = p + COMMON + 8;
  const uint8_t* pay = p + COMMON + 8 + 256;
  size_t plen = n - (COMMON + 8 + 256);
  if (nsym == 0) {
    if (nbits || plen) return fail(HBO_ESTAGE, "nonempty payload for an empty huffman record");
    return 0;
  }
  if (nbits / 8 + (nbits % 8 != 0) != plen) return fail(HBO_ESTAGE, "huffman payload length mismatch");
  uint64_t code[256] = {0};
  int syms[256];
  int ns = canonical(len, code, syms);
  if (ns == 0) return fail(HBO_ESTAGE, "huffman record with an empty code table");
  int maxlen = len[syms[ns - 1]];
  /* Kraft: available slots never negative (exact, capped) */
  {
    int64_t avail = 1, remaining = ns;
    int cnt[256] = {0};
    for (int i = 0; i < ns; i++) cnt[len[syms[i]]]++;
    for (int L = 1; L <= maxlen; L++) {
      avail = avail * 2 - cnt[L];
      remaining -= cnt[L];
      if (avail < 0) return fail(HBO_ESTAGE, "code-length table violates the prefix bound");
      if (avail > 1024) avail = 1024; /* can no longer go negative */
      (void)remaining;
    }
  }
  uint64_t first_code[256];
  int first_rank[256], count[256];
  for (int L = 0; L < 256; L++) first_rank[L] = -1, count[L] = 0;
  for (int i = 0; i < ns; i++) {
    int L = len[syms[i]];
    if (first_rank[L] < 0) first_code[L] = code[syms[i]], first_rank[L] = i;
    count[L]++;
  }
  if (buf_reserve(out, (size_t)nsym)) return fail(HBO_ENOMEM, "oom");
  uint8_t* o = out->p + out->n;
  /* bit-serial canonical decode; equivalent to the reference's LUT+slow path */
  uint64_t pos = 0;
  for (uint64_t i = 0; i < nsym; i++) {
    uint64_t c = 0;
    int L = 0, sym = -1;
    while (L < maxlen) {
      int bit = pos + L < (uint64_t)plen * 8 ? (pay[(pos + L) >> 3] >> (7 - ((pos + L) & 7))) & 1 : 0;
      c = (c << 1) | (uint64_t)bit;
      L++;
      if (first_rank[L] >= 0 && c >= first_code[L] && c - first_code[L] < (uint64_t)count[L]) {
        sym = syms[first_rank[L] + (int)(c - first_code[L])];
        break;
      }
    }
    if (sym < 0) return fail(HBO_ESTAGE, "invalid huffman code in bitstream");
    if (pos + L > nbits) return fail(HBO_ESTAGE, "huffman bitstream overrun");
    pos += L;
    o[i] = (uint8_t)sym;
  }
  if (pos != nbits) return fail(HBO_ESTAGE, "huffman bit count mismatch");
  out->n += nsym;
  return 0;
}

static int pipe_apply(int enc, int stage, int width, const uint8_t* in, size_t n, buf_t* out) {
  if (enc) {
    switch (stage) {
      case 1: return huffman_encode(in, n, out);
      case 2: return width_ok(width) ? bitmap_encode(2, in, n, width, MAX_DEPTH, out) : fail(HBO_ESTAGE, "bad width");
      case 3: return width_ok(width) ? bitmap_encode(3, in, n, width, MAX_DEPTH, out) : fail(HBO_ESTAGE, "bad width");
      case 4: return tcms_encode(in, n, width, out);
      case 5: return bit_shuffle(in, n, width, out);
    }
  } else {
    switch (stage) {
      case 1: return huffman_decode(in, n, out);
      case 2: return bitmap_decode(2, in, n, MAX_DEPTH, out);
      case 3: return bitmap_decode(3, in, n, MAX_DEPTH, out);
      case 4: return tcms_decode(in, n, out);
      case 5: return bit_unshuffle(in, n, out);
    }
  }
  return fail(HBO_EARG, "unknown stage %d", stage);
}

/* stages.py:422-435 */
static int run_chain(int enc, const int* st, const int* wd, int k, const uint8_t* in, size_t n, buf_t* res) {
  buf_t cur = {0}, nxt = {0};
  const uint8_t* src = in;
  size_t sn = n;
  for (int i = 0; i < k; i++) {
    nxt.n = 0;
    int rc = pipe_apply(enc, st[i], wd[i], src, sn, &nxt);
    if (rc) {
      free(cur.p), free(nxt.p);
      return rc;
    }
    buf_t t = cur;
    cur = nxt;
    nxt = t;
    src = cur.p;
    sn = cur.n;
  }
  free(nxt.p);
  *res = cur;
  return 0;
}

int hbo_stage_encode(int stage, int width, const uint8_t* in, size_t n, uint8_t** out, size_t* outlen) {
  buf_t b = {0};
  int rc;
  if (stage == HBO_PIPE_CR) {
    int st[4] = {1, 2, 4, 3}, wd[4] = {1, 4, 8, 1};
    rc = run_chain(1, st, wd, 4, in, n, &b);
  } else if (stage == HBO_PIPE_TP) {
    int st[3] = {4, 5, 2}, wd[3] = {1, 1, 1};
    rc = run_chain(1, st, wd, 3, in, n, &b);
  } else
    rc = pipe_apply(1, stage, width, in, n, &b);
  if (rc) {
    free(b.p);
    return rc;
  }
  if (!b.p) b.p = (uint8_t*)malloc(1);
  *out = b.p;
  *outlen = b.n;
  return 0;
}

int hbo_stage_decode(int stage, const uint8_t* in, size_t n, uint8_t** out, size_t* outlen) {
  buf_t b = {0};
  int rc;
  if (stage == HBO_PIPE_CR) {
    int st[4] = {3, 4, 2, 1}, wd[4] = {0};
    rc = run_chain(0, st, wd, 4, in, n, &b);
  } else if (stage == HBO_PIPE_TP) {
    int st[3] = {2, 5, 4}, wd[3] = {0};
    rc = run_chain(0, st, wd, 3, in, n, &b);
  } else
    rc = pipe_apply(0, stage, 0, in, n, &b);
  if (rc) {
    free(b.p);
    return rc;
  }
  if (!b.p) b.p = (uint8_t*)malloc(1);
  *out = b.p;
  *outlen = b.n;
  return 0;
}

/* ------------------------------------------------------- archive.py:41-171 */

#define FIXED 46

int hbo_compress(const void* vals, int prec, const uint64_t dims[3], int ndim, int eb_mode, double mag, int mode,
                 uint8_t** out, size_t* outlen) {
  if (mode != 0 && mode != 1) return fail(HBO_EARG, "mode must be 'cr' or 'tp'");
  if (prec != 4 && prec != 8) return fail(HBO_EFIELD, "unsupported precision");
  uint64_t N = dims[0] * dims[1] * dims[2];
  for (uint64_t i = 0; i < N; i++)
    if (!isfinite(load_val(vals, prec, i))) return fail(HBO_EFIELD, "field contains NaN or Inf values");
  double eb;
  int rc = hbo_resolve_eb(vals, prec, N, eb_mode, mag, &eb);
  if (rc) return rc;
  if (!(isfinite(eb) && eb > 0)) return fail(HBO_EBOUND, "error bound must be positive and finite, got %g", eb);
  uint8_t cfg[4];
  double errs[16];
  rc = hbo_tune(vals, prec, dims, eb, cfg, errs);
  if (rc) return rc;
  int A = hbo_anchor_stride(dims);
  uint64_t na = ((dims[0] + A - 1) / A) * ((dims[1] + A - 1) / A) * ((dims[2] + A - 1) / A);
  uint8_t* codes = (uint8_t*)malloc(N);
  uint8_t* seq = (uint8_t*)malloc(N);
  uint64_t* oidx = (uint64_t*)malloc(N * 8);
  void* oval = malloc(N * prec);
  void* anc = malloc(na * prec);
  if (!codes || !seq || !oidx || !oval || !anc) {
    free(codes), free(seq), free(oidx), free(oval), free(anc);
    return fail(HBO_ENOMEM, "oom");
  }
  uint64_t oc;
  rc = hbo_decompose(vals, prec, dims, eb, cfg, codes, oidx, oval, &oc, anc);
  if (!rc) rc = hbo_reorder(codes, dims, A, seq);
  uint8_t* enc = NULL;
  size_t elen = 0;
  if (!rc) rc = hbo_stage_encode(mode == 0 ? HBO_PIPE_CR : HBO_PIPE_TP, 0, seq, N, &enc, &elen);
  if (rc) {
    free(codes), free(seq), free(oidx), free(oval), free(anc), free(enc);
    return rc;
  }
  int escape = elen > N;
  buf_t b = {0};
  uint8_t hdr[FIXED];
  memcpy(hdr, "CSZH", 4);
  hdr[4] = 1;
  hdr[5] = (uint8_t)mode;
  hdr[6] = (uint8_t)prec;
  hdr[7] = (uint8_t)ndim;
  hdr[8] = (uint8_t)A;
  hdr[9] = (uint8_t)escape;
  memcpy(hdr + 10, cfg, 4);
  for (int a = 0; a < 3; a++)
    for (int i = 0; i < 8; i++) hdr[14 + 8 * a + i] = (uint8_t)(dims[a] >> (8 * i));
  uint64_t ebits;
  memcpy(&ebits, &eb, 8);
  for (int i = 0; i < 8; i++) hdr[38 + i] = (uint8_t)(ebits >> (8 * i));
  int err = buf_put(&b, hdr, FIXED) || buf_u64(&b, na) || buf_put(&b, anc, na * prec) || buf_u64(&b, oc);
  for (uint64_t i = 0; i < oc && !err; i++)
    err = buf_u64(&b, oidx[i]) || buf_put(&b, (uint8_t*)oval + i * prec, prec);
  if (!err) err = buf_u64(&b, escape ? N : elen) || buf_put(&b, escape ? seq : enc, escape ? N : elen);
  free(codes), free(seq), free(oidx), free(oval), free(anc), free(enc);
  if (err) {
    free(b.p);
    return fail(HBO_ENOMEM, "oom");
  }
  *out = b.p;
  *outlen = b.n;
  return 0;
}

int hbo_archive_info(const uint8_t* blob, size_t len, hbo_info* I) {
  memset(I, 0, sizeof *I);
  if (len < FIXED) return fail(HBO_EARCHIVE, "archive truncated in header");
  if (memcmp(blob, "CSZH", 4)) return fail(HBO_EARCHIVE, "bad magic");
  if (blob[4] != 1) return fail(HBO_EARCHIVE, "unsupported archive version %d", blob[4]);
  if (blob[5] > 1) return fail(HBO_EARCHIVE, "unknown mode byte %d", blob[5]);
  if (blob[6] != 4 && blob[6] != 8) return fail(HBO_EARCHIVE, "unsupported precision %d", blob[6]);
  if (blob[7] != 2 && blob[7] != 3) return fail(HBO_EARCHIVE, "unsupported ndim %d", blob[7]);
  int st = blob[8];
  if (st < 1 || st > 16 || (st & (st - 1))) return fail(HBO_EARCHIVE, "invalid anchor stride %d", st);
  if (blob[9] > 1) return fail(HBO_EARCHIVE, "invalid escape flag %d", blob[9]);
  I->mode = blob[5];
  I->precision = blob[6];
  I->ndim = blob[7];
  I->stride = st;
  I->escape = blob[9];
  memcpy(I->cfg, blob + 10, 4);
  for (int a = 0; a < 3; a++) I->dims[a] = rd_u64(blob + 14 + 8 * a);
  uint64_t ebits = rd_u64(blob + 38);
  memcpy(&I->eb, &ebits, 8);
  for (int a = 0; a < 3; a++)
    if (I->dims[a] < 1) return fail(HBO_EARCHIVE, "invalid dims");
  if (I->ndim == 2 && I->dims[2] != 1) return fail(HBO_EARCHIVE, "2D archive must carry a trailing dimension of 1");
  if (!(isfinite(I->eb) && I->eb > 0)) return fail(HBO_EARCHIVE, "invalid error bound");
  for (int i = 0; i < 4; i++)
    if (I->cfg[i] & ~3) return fail(HBO_EARCHIVE, "invalid interpolation config byte 0x%02x", I->cfg[i]);
  size_t off = FIXED;
  unsigned __int128 need;
  if (len - off < 8) return fail(HBO_EARCHIVE, "archive truncated in anchor count");
  I->anchor_count = rd_u64(blob + off);
  off += 8;
  uint64_t ea = 1;
  for (int a = 0; a < 3; a++) ea *= (I->dims[a] + st - 1) / st;
  if (I->anchor_count != ea) return fail(HBO_EARCHIVE, "anchor count does not match dims");
  need = (unsigned __int128)I->anchor_count * I->precision;
  if (need > len - off) return fail(HBO_EARCHIVE, "archive truncated in anchor values");
  I->anchor_off = off;
  off += (size_t)need;
  if (len - off < 8) return fail(HBO_EARCHIVE, "archive truncated in outlier count");
  I->outlier_count = rd_u64(blob + off);
  off += 8;
  unsigned __int128 n = (unsigned __int128)I->dims[0] * I->dims[1] * I->dims[2];
  if (I->outlier_count > n) return fail(HBO_EARCHIVE, "outlier count exceeds point count");
  need = (unsigned __int128)I->outlier_count * (8 + I->precision);
  if (need > len - off) return fail(HBO_EARCHIVE, "archive truncated in outlier section");
  I->outlier_off = off;
  off += (size_t)need;
  if (len - off < 8) return fail(HBO_EARCHIVE, "archive truncated in stream length");
  I->stream_len = rd_u64(blob + off);
  off += 8;
  if (I->stream_len > len - off) return fail(HBO_EARCHIVE, "archive truncated in code stream");
  I->stream_off = off;
  off += (size_t)I->stream_len;
  if (off != len) return fail(HBO_EARCHIVE, "trailing bytes after code stream");
  return 0;
}

int hbo_decompress(const uint8_t* blob, size_t len, void* out, size_t cap, hbo_info* info) {
  hbo_info I;
  int rc = hbo_archive_info(blob, len, &I);
  if (info) *info = I;
  if (rc) return rc;
  uint64_t N = I.dims[0] * I.dims[1] * I.dims[2];
  if (cap < N * I.precision) return fail(HBO_EARG, "output buffer too small");
  const uint8_t* op = blob + I.outlier_off;
  uint64_t k = I.outlier_count;
  uint64_t* oidx = (uint64_t*)malloc(k * 8 + 8);
  void* oval = malloc(k * I.precision + 8);
  if (!oidx || !oval) {
    free(oidx), free(oval);
    return fail(HBO_ENOMEM, "oom");
  }
  for (uint64_t i = 0; i < k; i++) {
    oidx[i] = rd_u64(op + i * (8 + I.precision));
    memcpy((uint8_t*)oval + i * I.precision, op + i * (8 + I.precision) + 8, I.precision);
  }
  for (uint64_t i = 0; i < k; i++)
    if (oidx[i] >= N) {
      free(oidx), free(oval);
      return fail(HBO_EARCHIVE, "outlier index out of range");
    }
  for (uint64_t i = 1; i < k; i++)
    if (oidx[i] <= oidx[i - 1]) {
      free(oidx), free(oval);
      return fail(HBO_EARCHIVE, "outlier indices not strictly ascending");
    }
  uint8_t* raw = NULL;
  size_t rlen = 0;
  if (I.escape) {
    raw = (uint8_t*)malloc(I.stream_len + 1);
    if (raw) memcpy(raw, blob + I.stream_off, I.stream_len);
    rlen = I.stream_len;
  } else {
    rc = hbo_stage_decode(I.mode == 0 ? HBO_PIPE_CR : HBO_PIPE_TP, blob + I.stream_off, I.stream_len, &raw, &rlen);
    if (rc) {
      free(oidx), free(oval);
      return rc;
    }
  }
  if (rlen != N) {
    free(oidx), free(oval), free(raw);
    return fail(HBO_EARCHIVE, "decoded code sequence has %zu bytes, expected %llu", rlen, (unsigned long long)N);
  }
  uint8_t* codes = (uint8_t*)malloc(N);
  if (!codes) {
    free(oidx), free(oval), free(raw);
    return fail(HBO_ENOMEM, "oom");
  }
  hbo_inverse_reorder(raw, I.dims, I.stride, codes);
  uint64_t zeros = 0;
  for (uint64_t i = 0; i < N; i++) zeros += codes[i] == 0;
  if (zeros != k) {
    free(oidx), free(oval), free(raw), free(codes);
    return fail(HBO_EARCHIVE, "outlier markers do not match the outlier section");
  }
  /* the archive's own stride drives the walk (archive.py:166-171) */
  rc = reconstruct_impl(codes, oidx, oval, k, blob + I.anchor_off, I.precision, I.dims, I.eb, I.cfg, out, I.stride);
  free(oidx), free(oval), free(raw), free(codes);
  return rc;
}
