/*
 * btnn_oracle.c — TEST INFRASTRUCTURE ONLY. CPU restatement of the reference btnn
 * hot path (arXiv 2006.16578 CPU reference, /root/reference/proj/include/btnn), in
 * plain C, scalar, single-threaded. It is the checker the parity tests, smoke() and
 * bench.py's cpu_baseline leg compare the CUDA path against; the product never links,
 * loads or calls it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every function here against the
 * reference's own known-answer tests (test_bitcore.cpp, test_oracle.cpp, test_bconv.cpp,
 * test_nn.cpp hand cases) and against outputs of the reference itself, compiled from
 * its unmodified headers into oracle/_ref/libbtnn_ref.so (oracle/ref_shim.cpp) and
 * frozen as fixtures under tests/golden/ (tests/golden/make_golden.py).
 *
 * All bit storage follows the reference: uint64 words, bit b in word b/64 at position
 * b%64 (bit_buffer.hpp:14-16), pad bits zero. Arithmetic mirrors the reference
 * statement by statement, including f64 evaluation order (the reference builds with
 * -ffp-contract=off, CMakeLists.txt:16-18; this file is compiled the same way).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/btnn_cuda.h"

#define BO_OK 0
#define BO_INVALID 1
#define BO_UNSUPPORTED 2

static size_t ru(size_t v, size_t m) { return (v + m - 1) / m * m; }  /* common.hpp:34 */
static size_t cdiv(size_t a, size_t b) { return (a + b - 1) / b; }    /* common.hpp:38 */
static int bget(const uint64_t* w, size_t b) { return (int)((w[b >> 6] >> (b & 63)) & 1u); }
static void bset(uint64_t* w, size_t b) { w[b >> 6] |= (uint64_t)1 << (b & 63); }
static int popc64(uint64_t x) { return __builtin_popcountll(x); }

/* ---------------- bit_buffer.hpp ---------------- */

/* pack_signs (bit_buffer.hpp:77-91): bit i = values[i] >= 0; non-finite rejected. */
int bo_pack_signs_f32(const float* v, size_t n, uint64_t* out) {
  memset(out, 0, cdiv(n, 64) * 8);
  for (size_t i = 0; i < n; ++i) {
    if (!isfinite(v[i])) return BO_INVALID;
    if (v[i] >= 0.0f) bset(out, i);
  }
  return BO_OK;
}

/* xor_popcount / dot_pm1 (bit_buffer.hpp:94-113). */
int64_t bo_dot_pm1(const uint64_t* a, const uint64_t* b, size_t n) {
  const size_t full = n >> 6;
  int64_t acc = 0;
  for (size_t i = 0; i < full; ++i) acc += popc64(a[i] ^ b[i]);
  const size_t rem = n & 63;
  if (rem) acc += popc64((a[full] ^ b[full]) & (((uint64_t)1 << rem) - 1));
  return (int64_t)n - 2 * acc;
}

/* ---------------- bit_matrix.hpp ---------------- */

/* BitMatrix::padded_rows/padded_cols (bit_matrix.hpp:83-102). */
size_t bo_padded_rows(size_t rows, int layout, size_t bh, size_t bw) {
  switch (layout) {
    case BTNN_ROW_PACKED: return rows;
    case BTNN_COL_PACKED: return ru(rows, 128);
    case BTNN_FSB_ROW: return ru(rows, bh);
    default: return ru(rows, bw);
  }
}
size_t bo_padded_cols(size_t cols, int layout, size_t bh, size_t bw) {
  switch (layout) {
    case BTNN_ROW_PACKED: return ru(cols, 128);
    case BTNN_COL_PACKED: return cols;
    case BTNN_FSB_ROW: return ru(cols, bw);
    default: return ru(cols, bh);
  }
}
size_t bo_matrix_words(size_t rows, size_t cols, int layout, size_t bh, size_t bw) {
  return bo_padded_rows(rows, layout, bh, bw) * bo_padded_cols(cols, layout, bh, bw) / 64;
}

/* BitMatrix::bit_index (bit_matrix.hpp:106-114) with FsbGeometry::row/col_tiled_index (:44-56). */
size_t bo_bit_index(size_t rows, size_t cols, int layout, size_t bh, size_t bw, size_t r, size_t c) {
  const size_t pr = bo_padded_rows(rows, layout, bh, bw), pc = bo_padded_cols(cols, layout, bh, bw);
  switch (layout) {
    case BTNN_ROW_PACKED: return r * pc + c;
    case BTNN_COL_PACKED: return c * pr + r;
    case BTNN_FSB_ROW: return ((r / bh) * (pc / bw) + c / bw) * (bh * bw) + (r % bh) * bw + (c % bw);
    default: return ((c / bh) * (pr / bw) + r / bw) * (bh * bw) + (c % bh) * bw + (r % bw);
  }
}

/* pack_matrix (bit_matrix.hpp:135-155). */
int bo_pack_matrix(const float* v, size_t rows, size_t cols, int layout, size_t bh, size_t bw,
                   uint64_t* out) {
  memset(out, 0, bo_matrix_words(rows, cols, layout, bh, bw) * 8);
  for (size_t r = 0; r < rows; ++r)
    for (size_t c = 0; c < cols; ++c) {
      const float x = v[r * cols + c];
      if (!isfinite(x)) return BO_INVALID;
      if (x >= 0.0f) bset(out, bo_bit_index(rows, cols, layout, bh, bw, r, c));
    }
  return BO_OK;
}

/* Generic layout copy (bit_matrix.hpp:163-168, to_fsb :224-237, from_fsb :240-253). */
void bo_convert_matrix(size_t rows, size_t cols, int src_layout, size_t sbh, size_t sbw,
                       const uint64_t* src, int dst_layout, size_t dbh, size_t dbw, uint64_t* dst) {
  memset(dst, 0, bo_matrix_words(rows, cols, dst_layout, dbh, dbw) * 8);
  for (size_t r = 0; r < rows; ++r)
    for (size_t c = 0; c < cols; ++c)
      if (bget(src, bo_bit_index(rows, cols, src_layout, sbh, sbw, r, c)))
        bset(dst, bo_bit_index(rows, cols, dst_layout, dbh, dbw, r, c));
}

/* ---------------- tensors.hpp ---------------- */

/* BitTensorHWNC geometry (tensors.hpp:79-99). */
static size_t act_npad(size_t n, int tiled, size_t bh) { return ru(n, tiled ? bh : 8); }
static size_t act_cpad(size_t c, int tiled, size_t bw) { return ru(c, tiled ? bw : 128); }
size_t bo_act_words(size_t h, size_t w, size_t n, size_t c, int tiled, size_t bh, size_t bw) {
  return h * w * act_npad(n, tiled, bh) * act_cpad(c, tiled, bw) / 64;
}
size_t bo_act_bit_index(size_t h, size_t w, size_t n, size_t c, int tiled, size_t bh, size_t bw,
                        size_t hh, size_t ww, size_t nn, size_t cc) {
  const size_t np = act_npad(n, tiled, bh), cp = act_cpad(c, tiled, bw);
  const size_t base = (hh * w + ww) * np * cp;
  (void)h;
  if (!tiled) return base + nn * cp + cc;
  return base + ((nn / bh) * (cp / bw) + cc / bw) * (bh * bw) + (nn % bh) * bw + (cc % bw);
}
/* BitFilterKKOC geometry (tensors.hpp:127-147). */
size_t bo_filter_words(size_t kh, size_t kw, size_t o, size_t c, int tiled, size_t bh, size_t bw) {
  return kh * kw * ru(o, tiled ? bh : 8) * ru(c, tiled ? bw : 128) / 64;
}
size_t bo_filter_bit_index(size_t kh, size_t kw, size_t o, size_t c, int tiled, size_t bh, size_t bw,
                           size_t r, size_t s, size_t oo, size_t cc) {
  const size_t op = ru(o, tiled ? bh : 8), cp = ru(c, tiled ? bw : 128);
  const size_t base = (r * kw + s) * op * cp;
  (void)kh;
  if (!tiled) return base + oo * cp + cc;
  /* geo.col_tiled_index(c, o, c_pad) (tensors.hpp:146) */
  return base + ((oo / bh) * (cp / bw) + cc / bw) * (bh * bw) + (oo % bh) * bw + (cc % bw);
}

/* pack_nhwc (tensors.hpp:162-174). */
int bo_pack_nhwc(const float* x, size_t n, size_t h, size_t w, size_t c, int tiled, size_t bh,
                 size_t bw, uint64_t* out) {
  memset(out, 0, bo_act_words(h, w, n, c, tiled, bh, bw) * 8);
  for (size_t nn = 0; nn < n; ++nn)
    for (size_t hh = 0; hh < h; ++hh)
      for (size_t ww = 0; ww < w; ++ww)
        for (size_t cc = 0; cc < c; ++cc) {
          const float v = x[((nn * h + hh) * w + ww) * c + cc];
          if (!isfinite(v)) return BO_INVALID;
          if (v >= 0.0f) bset(out, bo_act_bit_index(h, w, n, c, tiled, bh, bw, hh, ww, nn, cc));
        }
  return BO_OK;
}

/* pack_filter (tensors.hpp:177-193): flat (r, s, o, c) floats. */
int bo_pack_filter(const float* wt, size_t kh, size_t kw, size_t o, size_t c, int tiled, size_t bh,
                   size_t bw, uint64_t* out) {
  memset(out, 0, bo_filter_words(kh, kw, o, c, tiled, bh, bw) * 8);
  size_t i = 0;
  for (size_t r = 0; r < kh; ++r)
    for (size_t s = 0; s < kw; ++s)
      for (size_t oo = 0; oo < o; ++oo)
        for (size_t cc = 0; cc < c; ++cc, ++i) {
          if (!isfinite(wt[i])) return BO_INVALID;
          if (wt[i] >= 0.0f) bset(out, bo_filter_bit_index(kh, kw, o, c, tiled, bh, bw, r, s, oo, cc));
        }
  return BO_OK;
}

/* flatten_to_matrix (tensors.hpp:226-237): row n, feature (h*W + w)*C + c. */
void bo_flatten(size_t h, size_t w, size_t n, size_t c, int tiled, size_t bh, size_t bw,
                const uint64_t* act, int layout, size_t mbh, size_t mbw, uint64_t* out) {
  const size_t features = h * w * c;
  memset(out, 0, bo_matrix_words(n, features, layout, mbh, mbw) * 8);
  for (size_t nn = 0; nn < n; ++nn)
    for (size_t hh = 0; hh < h; ++hh)
      for (size_t ww = 0; ww < w; ++ww)
        for (size_t cc = 0; cc < c; ++cc)
          if (bget(act, bo_act_bit_index(h, w, n, c, tiled, bh, bw, hh, ww, nn, cc)))
            bset(out, bo_bit_index(n, features, layout, mbh, mbw, nn, (hh * w + ww) * c + cc));
}

/* ---------------- layer_math.hpp ---------------- */

/* BnParams::apply (layer_math.hpp:32-34). */
static double bn_apply(const btnn_bn* bn, size_t ch, double x) {
  return (x - bn->mean[ch]) / sqrt(bn->var[ch] + bn->eps) * bn->gamma[ch] + bn->beta[ch];
}
double bo_bn_apply(const btnn_bn* bn, size_t ch, double x) { return bn_apply(bn, ch, x); }

/* Threshold::fire (layer_math.hpp:44-52). */
static int fire(double tau, uint8_t kind, double x) {
  switch (kind) {
    case BTNN_GEQ: return x >= tau;
    case BTNN_LEQ: return x <= tau;
    case BTNN_CONST_PLUS: return 1;
    default: return 0;
  }
}
int bo_fire(double tau, uint8_t kind, double x) { return fire(tau, kind, x); }

/* fold_bn_sign (layer_math.hpp:61-67). */
void bo_fold_bn_sign(double gamma, double beta, double mean, double var, double eps, double* tau,
                     uint8_t* kind) {
  const double s = sqrt(var + eps);
  if (gamma > 0.0) { *tau = mean - beta * s / gamma; *kind = BTNN_GEQ; return; }
  if (gamma < 0.0) { *tau = mean - beta * s / gamma; *kind = BTNN_LEQ; return; }
  *tau = 0.0;
  *kind = beta >= 0.0 ? BTNN_CONST_PLUS : BTNN_CONST_MINUS;
}

/* ---------------- bmm.hpp ---------------- */

/* bmm_naive accumulator (bmm.hpp:81-99): xor popcount over padded inner words. Packed
 * layouts index by row/col words; fsb layouts are read through the bit index. */
static int32_t bmm_acc(const btnn_matrix_desc* a, const uint64_t* aw, const btnn_matrix_desc* b,
                       const uint64_t* bw, size_t i, size_t j) {
  if (a->layout == BTNN_ROW_PACKED) {
    const size_t kw = bo_padded_cols(a->cols, a->layout, 0, 0) / 64;
    int32_t acc = 0;
    for (size_t w = 0; w < kw; ++w) acc += popc64(aw[i * kw + w] ^ bw[j * kw + w]);
    return acc;
  }
  /* bmm_fsb (bmm.hpp:143-186) visits padded inner bits kb*bw..; pad bits are zero. */
  const size_t kp = bo_padded_cols(a->cols, a->layout, a->bh, a->bw);
  int32_t acc = 0;
  for (size_t k = 0; k < kp; ++k) {
    const int x = k < a->cols ? bget(aw, bo_bit_index(a->rows, a->cols, a->layout, a->bh, a->bw, i, k)) : 0;
    const int y = k < b->rows ? bget(bw, bo_bit_index(b->rows, b->cols, b->layout, b->bh, b->bw, k, j)) : 0;
    acc += x ^ y;
  }
  return acc;
}

/* check_bmm_operands (bmm.hpp:57-76). */
int bo_check_bmm(const btnn_matrix_desc* a, const btnn_matrix_desc* b, int variant) {
  if (a->cols != b->rows) return BO_INVALID;
  if (variant == BTNN_BMM_FSB) {
    if (a->layout != BTNN_FSB_ROW || b->layout != BTNN_FSB_COL) return BO_INVALID;
    if (a->bh != b->bh || a->bw != b->bw) return BO_UNSUPPORTED;
    if (a->bw % 64 != 0) return BO_UNSUPPORTED;
  } else {
    if (a->layout != BTNN_ROW_PACKED || b->layout != BTNN_COL_PACKED) return BO_INVALID;
  }
  if (bo_padded_cols(a->cols, a->layout, a->bh, a->bw) != bo_padded_rows(b->rows, b->layout, b->bh, b->bw))
    return BO_UNSUPPORTED;
  return BO_OK;
}

/* bmm_raw (bmm.hpp:204-214). */
int bo_bmm_raw(const btnn_matrix_desc* a, const uint64_t* aw, const btnn_matrix_desc* b,
               const uint64_t* bw, int variant, int32_t* out) {
  if (a->cols % 128 != 0) return BO_UNSUPPORTED;
  int st = bo_check_bmm(a, b, variant);
  if (st) return st;
  for (size_t i = 0; i < a->rows; ++i)
    for (size_t j = 0; j < b->cols; ++j) out[i * b->cols + j] = bmm_acc(a, aw, b, bw, i, j);
  return BO_OK;
}

/* bmm_pm1 (bmm.hpp:219-228): v = n - 2*acc with n the logical inner dim. */
int bo_bmm_pm1(const btnn_matrix_desc* a, const uint64_t* aw, const btnn_matrix_desc* b,
               const uint64_t* bw, int variant, int32_t* out) {
  int st = bo_check_bmm(a, b, variant);
  if (st) return st;
  const int32_t n = (int32_t)a->cols;
  for (size_t i = 0; i < a->rows; ++i)
    for (size_t j = 0; j < b->cols; ++j) out[i * b->cols + j] = n - 2 * bmm_acc(a, aw, b, bw, i, j);
  return BO_OK;
}

/* bmm_pm1_bin (bmm.hpp:256-274): output in A's family (RowPacked or FsbRow, A's geometry). */
int bo_bmm_pm1_bin(const btnn_matrix_desc* a, const uint64_t* aw, const btnn_matrix_desc* b,
                   const uint64_t* bw, int variant, const double* tau, const uint8_t* kind,
                   size_t n_thr, uint64_t* out) {
  if (n_thr != 0 && n_thr != b->cols) return BO_INVALID;
  int st = bo_check_bmm(a, b, variant);
  if (st) return st;
  const int lay = a->layout == BTNN_FSB_ROW ? BTNN_FSB_ROW : BTNN_ROW_PACKED;
  memset(out, 0, bo_matrix_words(a->rows, b->cols, lay, a->bh, a->bw) * 8);
  const int32_t n = (int32_t)a->cols;
  for (size_t i = 0; i < a->rows; ++i)
    for (size_t j = 0; j < b->cols; ++j) {
      const int32_t v = n - 2 * bmm_acc(a, aw, b, bw, i, j);
      const int bit = n_thr == 0 ? v >= 0 : fire(tau[j], kind[j], (double)v);
      if (bit) bset(out, bo_bit_index(a->rows, b->cols, lay, a->bh, a->bw, i, j));
    }
  return BO_OK;
}

/* ---------------- bconv.hpp ---------------- */

static size_t out_dim(size_t x, size_t k, size_t s, size_t p) { return (x + 2 * p - k) / s + 1; }

/* bconv_sites (bconv.hpp:76-133): value = C*KH*KW - exclude*C - 2*acc per (p,q,n,o). */
static int conv_value(const btnn_act_desc* in, const uint64_t* iw, const btnn_filter_desc* f,
                      const uint64_t* fw, const btnn_conv_geom* g, size_t p, size_t q, size_t n,
                      size_t o, int32_t* v) {
  const int32_t c = (int32_t)in->channels;
  const int32_t full = c * (int32_t)(g->kh * g->kw);
  int32_t exclude = 0, acc = 0;
  for (size_t r = 0; r < g->kh; ++r)
    for (size_t s = 0; s < g->kw; ++s) {
      const int64_t hh = (int64_t)(p * g->stride + r) - (int64_t)g->pad;
      const int64_t ww = (int64_t)(q * g->stride + s) - (int64_t)g->pad;
      if (hh < 0 || ww < 0 || hh >= (int64_t)in->height || ww >= (int64_t)in->width) {
        ++exclude;
        continue;
      }
      for (size_t cc = 0; cc < in->channels; ++cc) {
        const int x = bget(iw, bo_act_bit_index(in->height, in->width, in->batch, in->channels, in->tiled,
                                                in->bh, in->bw, (size_t)hh, (size_t)ww, n, cc));
        const int y = bget(fw, bo_filter_bit_index(f->kh, f->kw, f->out_channels, f->in_channels, f->tiled,
                                                   f->bh, f->bw, r, s, o, cc));
        acc += x ^ y;
      }
    }
  *v = full - exclude * c - 2 * acc;
  return 0;
}

/* Operand checks of bconv_sites (bconv.hpp:79-91). */
int bo_check_conv(const btnn_act_desc* in, const btnn_filter_desc* f, const btnn_conv_geom* g) {
  if (g->kh == 0 || g->kw == 0 || g->stride == 0) return BO_INVALID;
  if (g->kh != f->kh || g->kw != f->kw) return BO_INVALID;
  if (in->channels != f->in_channels) return BO_INVALID;
  if (in->tiled != f->tiled) return BO_INVALID;
  if (in->tiled) {
    if (in->bh != f->bh || in->bw != f->bw) return BO_UNSUPPORTED;
    if (in->bw % 64 != 0) return BO_UNSUPPORTED;
  }
  if (in->height + 2 * g->pad < g->kh || in->width + 2 * g->pad < g->kw) return BO_UNSUPPORTED;
  return BO_OK;
}

/* bconv_pm1 (bconv.hpp:138-146): IntTensorPQNO ((p*Q + q)*N + n)*O + o. */
int bo_bconv_pm1(const btnn_act_desc* in, const uint64_t* iw, const btnn_filter_desc* f,
                 const uint64_t* fw, const btnn_conv_geom* g, int32_t* out) {
  int st = bo_check_conv(in, f, g);
  if (st) return st;
  const size_t P = out_dim(in->height, g->kh, g->stride, g->pad), Q = out_dim(in->width, g->kw, g->stride, g->pad);
  const size_t N = in->batch, O = f->out_channels;
  for (size_t p = 0; p < P; ++p)
    for (size_t q = 0; q < Q; ++q)
      for (size_t n = 0; n < N; ++n)
        for (size_t o = 0; o < O; ++o) conv_value(in, iw, f, fw, g, p, q, n, o, &out[((p * Q + q) * N + n) * O + o]);
  return BO_OK;
}

/* bconv_fused (bconv.hpp:160-194). Output HWNC in the input's layout. */
int bo_bconv_fused(const btnn_act_desc* in, const uint64_t* iw, const btnn_filter_desc* f,
                   const uint64_t* fw, const btnn_conv_geom* g, const btnn_conv_fused* fu, uint64_t* out) {
  const size_t O = f->out_channels;
  const int thresholded = fu->n_thresholds != 0;
  if (thresholded == (fu->bn != NULL)) return BO_INVALID;
  if (thresholded && fu->n_thresholds != O) return BO_INVALID;
  if (fu->bn && fu->bn->channels != O) return BO_INVALID;
  if ((fu->residual_in || fu->residual_out) && !fu->bn) return BO_INVALID;
  int st = bo_check_conv(in, f, g);
  if (st) return st;
  const size_t P = out_dim(in->height, g->kh, g->stride, g->pad), Q = out_dim(in->width, g->kw, g->stride, g->pad);
  const size_t N = in->batch;
  memset(out, 0, bo_act_words(P, Q, N, O, in->tiled, in->bh, in->bw) * 8);
  for (size_t p = 0; p < P; ++p)
    for (size_t q = 0; q < Q; ++q)
      for (size_t n = 0; n < N; ++n)
        for (size_t o = 0; o < O; ++o) {
          int32_t v;
          conv_value(in, iw, f, fw, g, p, q, n, o, &v);
          int bit;
          if (thresholded) {
            bit = fire(fu->tau[o], fu->kind[o], (double)v);
          } else {
            const size_t idx = ((p * Q + q) * N + n) * O + o;
            double y = bn_apply(fu->bn, o, (double)v);
            if (fu->residual_in) y += fu->residual_in[idx];
            if (fu->residual_out) fu->residual_out[idx] = y;
            bit = y >= 0.0;
          }
          if (bit) bset(out, bo_act_bit_index(P, Q, N, O, in->tiled, in->bh, in->bw, p, q, n, o));
        }
  return BO_OK;
}

/* first_conv_bwn (bconv.hpp:198-243): (r, s, c)-ordered f64 sum per output. */
int bo_first_conv_bwn(const float* x, size_t N, size_t H, size_t W, size_t C, const float* wpm1,
                      size_t kh, size_t kw, size_t O, const btnn_conv_geom* g, double* out) {
  if (g->kh == 0 || g->kw == 0 || g->stride == 0) return BO_INVALID;
  if (g->kh != kh || g->kw != kw) return BO_INVALID;
  if (H + 2 * g->pad < kh || W + 2 * g->pad < kw) return BO_UNSUPPORTED;
  const size_t P = out_dim(H, kh, g->stride, g->pad), Q = out_dim(W, kw, g->stride, g->pad);
  for (size_t p = 0; p < P; ++p)
    for (size_t q = 0; q < Q; ++q)
      for (size_t n = 0; n < N; ++n)
        for (size_t o = 0; o < O; ++o) {
          const float* wb = wpm1 + o * kh * kw * C;
          double acc = 0.0;
          for (size_t r = 0; r < kh; ++r)
            for (size_t s = 0; s < kw; ++s) {
              const int64_t hh = (int64_t)(p * g->stride + r) - (int64_t)g->pad;
              const int64_t ww = (int64_t)(q * g->stride + s) - (int64_t)g->pad;
              if (hh < 0 || ww < 0 || hh >= (int64_t)H || ww >= (int64_t)W) continue;
              const float* xr = x + ((n * H + (size_t)hh) * W + (size_t)ww) * C;
              const float* wr = wb + (r * kw + s) * C;
              for (size_t c = 0; c < C; ++c) acc += (double)xr[c] * (double)wr[c];
            }
          out[((p * Q + q) * N + n) * O + o] = acc;
        }
  return BO_OK;
}

/* or_pool (bconv.hpp:247-272): OR of whole site planes. */
int bo_or_pool(const btnn_act_desc* in, const uint64_t* iw, size_t window, size_t stride, uint64_t* out) {
  if (window == 0 || stride == 0) return BO_INVALID;
  if (in->height < window || in->width < window) return BO_UNSUPPORTED;
  if ((in->height - window) % stride || (in->width - window) % stride) return BO_UNSUPPORTED;
  const size_t oh = (in->height - window) / stride + 1, ow = (in->width - window) / stride + 1;
  const size_t pw = act_npad(in->batch, in->tiled, in->bh) * act_cpad(in->channels, in->tiled, in->bw) / 64;
  memset(out, 0, oh * ow * pw * 8);
  for (size_t p = 0; p < oh; ++p)
    for (size_t q = 0; q < ow; ++q)
      for (size_t r = 0; r < window; ++r)
        for (size_t s = 0; s < window; ++s) {
          const uint64_t* src = iw + ((p * stride + r) * in->width + (q * stride + s)) * pw;
          uint64_t* dst = out + (p * ow + q) * pw;
          for (size_t w = 0; w < pw; ++w) dst[w] |= src[w];
        }
  return BO_OK;
}

/* ---------------- inference.hpp ---------------- */

/* adapt_shortcut (inference.hpp:43-63): 2x2 mean in the order ((a+b)+c)+d, times 0.25;
 * channels >= src.C are 0. */
static double adapt_value(const double* src, size_t sp, size_t sq, size_t sn, size_t sc,
                          size_t out_p, size_t p, size_t q, size_t n, size_t c) {
  (void)sp;
  if (c >= sc) return 0.0;
  if (sp == out_p) return src[((p * sq + q) * sn + n) * sc + c];
  double v = ((src[((2 * p * sq + 2 * q) * sn + n) * sc + c] + src[((2 * p * sq + 2 * q + 1) * sn + n) * sc + c]) +
              src[(((2 * p + 1) * sq + 2 * q) * sn + n) * sc + c]) +
             src[(((2 * p + 1) * sq + 2 * q + 1) * sn + n) * sc + c];
  v *= 0.25;
  return v;
}

typedef struct {
  size_t p, q, ch;
  double* v;
} tap_t;

/* run_inference (inference.hpp:67-186) on a resolved model and a plain- or fsb-layout
 * store, restated over the functions above. logits batch*classes, labels batch. */
int bo_run_inference(const btnn_model_spec* m, const btnn_weight_store* ws, const float* x, size_t batch,
                     double* logits, int32_t* labels) {
  if (ws->n_layers != m->n_layers) return BO_INVALID;
  if (batch == 0) return BO_INVALID;
  for (size_t i = 0; i < batch * m->in_h * m->in_w * m->in_c; ++i)
    if (!isfinite(x[i])) return BO_INVALID;
  const int tiled = ws->tiled;
  const size_t bh = ws->bh, bw = ws->bw;
  tap_t* taps = (tap_t*)calloc(m->n_layers, sizeof(tap_t));
  uint64_t* act = NULL;
  btnn_act_desc ad = {0};
  uint64_t* fc = NULL;
  btnn_matrix_desc fd = {0};
  int in_fc = 0, st = BO_OK;
  for (size_t i = 0; i < m->n_layers && st == BO_OK; ++i) {
    const btnn_layer_spec* l = &m->layers[i];
    const btnn_layer_weights* lw = &ws->layers[i];
    btnn_conv_geom g = {l->kh, l->kw, l->stride, l->pad};
    if (l->kind == BTNN_FIRST_CONV_BWN) {
      const size_t P = l->out_h, Q = l->out_w, O = l->out_channels;
      double* acc = (double*)malloc(P * Q * batch * O * sizeof(double));
      st = bo_first_conv_bwn(x, batch, l->in_h, l->in_w, l->in_channels, lw->conv_pm1, l->kh, l->kw, O, &g, acc);
      btnn_act_desc nd = {P, Q, batch, O, tiled, bh, bw};
      uint64_t* out = (uint64_t*)calloc(bo_act_words(P, Q, batch, O, tiled, bh, bw), 8);
      if (l->residual_out) {
        taps[i].p = P; taps[i].q = Q; taps[i].ch = O;
        taps[i].v = (double*)malloc(P * Q * batch * O * sizeof(double));
      }
      for (size_t p = 0; p < P; ++p)
        for (size_t q = 0; q < Q; ++q)
          for (size_t n = 0; n < batch; ++n)
            for (size_t o = 0; o < O; ++o) {
              const size_t idx = ((p * Q + q) * batch + n) * O + o;
              const double y = bn_apply(&lw->bn, o, acc[idx]);
              if (l->residual_out) taps[i].v[idx] = y;
              if (y >= 0.0) bset(out, bo_act_bit_index(P, Q, batch, O, tiled, bh, bw, p, q, n, o));
            }
      free(acc);
      free(act);
      act = out;
      ad = nd;
    } else if (l->kind == BTNN_BIT_CONV) {
      btnn_filter_desc f = {l->kh, l->kw, l->out_channels, l->in_channels, tiled, bh, bw};
      btnn_conv_fused fu;
      memset(&fu, 0, sizeof fu);
      if (lw->n_thresholds) {
        fu.tau = lw->tau; fu.kind = lw->tkind; fu.n_thresholds = lw->n_thresholds;
      } else {
        fu.bn = &lw->bn;
      }
      const size_t P = l->out_h, Q = l->out_w, O = l->out_channels;
      double* adapted = NULL;
      if (l->residual_in) {
        const tap_t* t = &taps[l->shortcut_from];
        adapted = (double*)malloc(P * Q * batch * O * sizeof(double));
        for (size_t p = 0; p < P; ++p)
          for (size_t q = 0; q < Q; ++q)
            for (size_t n = 0; n < batch; ++n)
              for (size_t o = 0; o < O; ++o)
                adapted[((p * Q + q) * batch + n) * O + o] = adapt_value(t->v, t->p, t->q, batch, t->ch, P, p, q, n, o);
        fu.residual_in = adapted;
      }
      if (l->residual_out) {
        taps[i].p = P; taps[i].q = Q; taps[i].ch = O;
        taps[i].v = (double*)malloc(P * Q * batch * O * sizeof(double));
        fu.residual_out = taps[i].v;
      }
      btnn_act_desc nd = {P, Q, batch, O, tiled, bh, bw};
      uint64_t* out = (uint64_t*)calloc(bo_act_words(P, Q, batch, O, tiled, bh, bw), 8);
      st = bo_bconv_fused(&ad, act, &f, lw->filter_words, &g, &fu, out);
      free(adapted);
      free(act);
      act = out;
      ad = nd;
    } else if (l->kind == BTNN_OR_POOL) {
      const size_t oh = l->out_h, ow = l->out_w;
      btnn_act_desc nd = {oh, ow, batch, ad.channels, tiled, bh, bw};
      uint64_t* out = (uint64_t*)calloc(bo_act_words(oh, ow, batch, ad.channels, tiled, bh, bw), 8);
      st = bo_or_pool(&ad, act, l->window, l->pool_stride, out);
      free(act);
      act = out;
      ad = nd;
    } else {
      const int alay = tiled ? BTNN_FSB_ROW : BTNN_ROW_PACKED;
      if (!in_fc) {
        if (i == 0) {
          fd.rows = batch; fd.cols = l->in_channels; fd.layout = alay; fd.bh = bh; fd.bw = bw;
          fc = (uint64_t*)calloc(bo_matrix_words(batch, l->in_channels, alay, bh, bw), 8);
          st = bo_pack_matrix(x, batch, l->in_channels, alay, bh, bw, fc);
        } else {
          fd.rows = batch; fd.cols = ad.height * ad.width * ad.channels; fd.layout = alay; fd.bh = bh; fd.bw = bw;
          fc = (uint64_t*)calloc(bo_matrix_words(fd.rows, fd.cols, alay, bh, bw), 8);
          bo_flatten(ad.height, ad.width, ad.batch, ad.channels, tiled, bh, bw, act, alay, bh, bw, fc);
          free(act);
          act = NULL;
        }
        in_fc = 1;
      }
      btnn_matrix_desc wd = {l->in_channels, l->units, tiled ? BTNN_FSB_COL : BTNN_COL_PACKED, bh, bw};
      const int var = tiled ? BTNN_BMM_FSB : BTNN_BMM_BLOCKED;
      if (l->kind == BTNN_BIT_FC) {
        btnn_matrix_desc od = {batch, l->units, alay, bh, bw};
        uint64_t* out = (uint64_t*)calloc(bo_matrix_words(batch, l->units, alay, bh, bw), 8);
        st = bo_bmm_pm1_bin(&fd, fc, &wd, lw->fc_words, var, lw->tau, lw->tkind, lw->n_thresholds, out);
        free(fc);
        fc = out;
        fd = od;
      } else {
        int32_t* v = (int32_t*)malloc(batch * l->units * sizeof(int32_t));
        st = bo_bmm_pm1(&fd, fc, &wd, lw->fc_words, var, v);
        for (size_t n = 0; n < batch; ++n)
          for (size_t j = 0; j < m->classes; ++j)
            logits[n * m->classes + j] = bn_apply(&lw->bn, j, (double)v[n * l->units + j]);
        free(v);
      }
    }
  }
  for (size_t n = 0; n < batch && st == BO_OK; ++n) {
    const double* row = logits + n * m->classes;
    size_t best = 0;
    for (size_t j = 1; j < m->classes; ++j)
      if (row[j] > row[best]) best = j;
    labels[n] = (int32_t)best;
  }
  for (size_t i = 0; i < m->n_layers; ++i) free(taps[i].v);
  free(taps);
  free(act);
  free(fc);
  return st;
}

/* ---------------- oracle.hpp dense references (for the known-answer tests) -------- */

/* ref_matmul (oracle.hpp:43-57): fixed i, l, j order. */
void bo_ref_matmul(const double* a, const double* b, size_t m, size_t n, size_t k, double* out) {
  memset(out, 0, m * k * sizeof(double));
  for (size_t i = 0; i < m; ++i)
    for (size_t l = 0; l < n; ++l) {
      const double av = a[i * n + l];
      for (size_t j = 0; j < k; ++j) out[i * k + j] += av * b[l * k + j];
    }
}

/* ref_conv_zero_pad (oracle.hpp:77-117): x NHWC, wt (r,s,o,c), out PQNO. */
int bo_ref_conv_zero_pad(const double* x, size_t n, size_t h, size_t w, size_t c, const double* wt,
                         size_t o, size_t kh, size_t kw, size_t stride, size_t pad, double* out) {
  if (stride == 0 || h + 2 * pad < kh || w + 2 * pad < kw) return BO_INVALID;
  const size_t P = out_dim(h, kh, stride, pad), Q = out_dim(w, kw, stride, pad);
  for (size_t p = 0; p < P; ++p)
    for (size_t q = 0; q < Q; ++q)
      for (size_t nn = 0; nn < n; ++nn)
        for (size_t oo = 0; oo < o; ++oo) {
          double acc = 0.0;
          for (size_t r = 0; r < kh; ++r)
            for (size_t s = 0; s < kw; ++s) {
              const int64_t hh = (int64_t)(p * stride + r) - (int64_t)pad;
              const int64_t ww = (int64_t)(q * stride + s) - (int64_t)pad;
              if (hh < 0 || ww < 0 || hh >= (int64_t)h || ww >= (int64_t)w) continue;
              const double* xr = x + ((nn * h + (size_t)hh) * w + (size_t)ww) * c;
              const double* wr = wt + ((r * kw + s) * o + oo) * c;
              for (size_t cc = 0; cc < c; ++cc) acc += xr[cc] * wr[cc];
            }
          out[((p * Q + q) * n + nn) * o + oo] = acc;
        }
  return BO_OK;
}

/* ref_max_pool (oracle.hpp:120-142). */
int bo_ref_max_pool(const double* x, size_t p, size_t q, size_t n, size_t o, size_t window, size_t stride,
                    double* out) {
  if (window == 0 || stride == 0 || p < window || q < window || (p - window) % stride || (q - window) % stride)
    return BO_INVALID;
  const size_t oh = (p - window) / stride + 1, ow = (q - window) / stride + 1;
  for (size_t pp = 0; pp < oh; ++pp)
    for (size_t qq = 0; qq < ow; ++qq)
      for (size_t nn = 0; nn < n; ++nn)
        for (size_t oo = 0; oo < o; ++oo) {
          double best = -INFINITY;
          for (size_t r = 0; r < window; ++r)
            for (size_t s = 0; s < window; ++s) {
              const double v = x[(((pp * stride + r) * q + (qq * stride + s)) * n + nn) * o + oo];
              best = v > best ? v : best;
            }
          out[((pp * ow + qq) * n + nn) * o + oo] = best;
        }
  return BO_OK;
}

/* ref_fc (oracle.hpp:146-160). */
void bo_ref_fc(const double* x, size_t n, size_t d, const double* wt, size_t k, double* out) {
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j < k; ++j) {
      double acc = 0.0;
      for (size_t dd = 0; dd < d; ++dd) acc += x[i * d + dd] * wt[j * d + dd];
      out[i * k + j] = acc;
    }
}

/* ref_htanh (oracle.hpp:163). */
double bo_ref_htanh(double x) { return x > 1.0 ? 1.0 : (x < -1.0 ? -1.0 : x); }
