// layout.cuh — bit-layout index math shared by host and device code.
//
// Device tensors use the reference's own byte layouts so the C ABI is zero-copy for the
// plain layouts (bit_matrix.hpp:21-132, tensors.hpp:71-159):
//   - bits are LSB-first in uint64 words (bit_buffer.hpp:14-16); a uint32 view keeps the
//     same bit order on little-endian, which the kernels use for warp ballots;
//   - HWNC activations: per site (h,w) an n_pad x c_pad plane, row n contiguous over c,
//     n_pad = round_up(N, 8), c_pad = round_up(C, 128) (tensors.hpp:86-99);
//   - KKOC filters: per tap (r,s) an o_pad x c_pad plane, row o contiguous over c
//     (tensors.hpp:134-147);
//   - RowPacked/ColPacked matrices pad the packed dimension to 128 bits (bit_matrix.hpp:83-102).
// The fsb (tiled) layouts are converted to plain on ingress and back on egress.
#pragma once
#include <cstddef>
#include <cstdint>

#include "btnn_cuda.h"

#ifdef __CUDACC__
#define BT_HD __host__ __device__ __forceinline__
#else
#define BT_HD inline
#endif

namespace btnn_gpu {

BT_HD size_t ru(size_t v, size_t m) { return (v + m - 1) / m * m; }
BT_HD size_t cdiv(size_t a, size_t b) { return (a + b - 1) / b; }

// BitMatrix::padded_rows/cols (bit_matrix.hpp:83-102).
BT_HD size_t mat_prows(size_t rows, int layout, size_t bh, size_t bw) {
  return layout == BTNN_ROW_PACKED ? rows
         : layout == BTNN_COL_PACKED ? ru(rows, 128)
         : layout == BTNN_FSB_ROW    ? ru(rows, bh)
                                     : ru(rows, bw);
}
BT_HD size_t mat_pcols(size_t cols, int layout, size_t bh, size_t bw) {
  return layout == BTNN_ROW_PACKED ? ru(cols, 128)
         : layout == BTNN_COL_PACKED ? cols
         : layout == BTNN_FSB_ROW    ? ru(cols, bw)
                                     : ru(cols, bh);
}
BT_HD size_t mat_words(size_t rows, size_t cols, int layout, size_t bh, size_t bw) {
  return mat_prows(rows, layout, bh, bw) * mat_pcols(cols, layout, bh, bw) / 64;
}
// BitMatrix::bit_index (bit_matrix.hpp:106-114).
BT_HD size_t mat_bit(size_t rows, size_t cols, int layout, size_t bh, size_t bw, size_t r, size_t c) {
  const size_t pr = mat_prows(rows, layout, bh, bw), pc = mat_pcols(cols, layout, bh, bw);
  if (layout == BTNN_ROW_PACKED) return r * pc + c;
  if (layout == BTNN_COL_PACKED) return c * pr + r;
  if (layout == BTNN_FSB_ROW) return ((r / bh) * (pc / bw) + c / bw) * (bh * bw) + (r % bh) * bw + (c % bw);
  return ((c / bh) * (pr / bw) + r / bw) * (bh * bw) + (c % bh) * bw + (r % bw);
}
// Inverse of mat_bit: storage bit b -> logical (r, c); false for pad bits.
BT_HD bool mat_inv(size_t rows, size_t cols, int layout, size_t bh, size_t bw, size_t b, size_t* r,
                   size_t* c) {
  const size_t pr = mat_prows(rows, layout, bh, bw), pc = mat_pcols(cols, layout, bh, bw);
  size_t rr, cc;
  if (layout == BTNN_ROW_PACKED) {
    rr = b / pc; cc = b % pc;
  } else if (layout == BTNN_COL_PACKED) {
    cc = b / pr; rr = b % pr;
  } else {
    const size_t tile = b / (bh * bw), in = b % (bh * bw);
    if (layout == BTNN_FSB_ROW) {
      const size_t tpr = pc / bw;
      rr = (tile / tpr) * bh + in / bw; cc = (tile % tpr) * bw + in % bw;
    } else {
      const size_t tpc = pr / bw;
      cc = (tile / tpc) * bh + in / bw; rr = (tile % tpc) * bw + in % bw;
    }
  }
  *r = rr; *c = cc;
  return rr < rows && cc < cols;
}

// BitTensorHWNC (tensors.hpp:79-99) — tiled uses FsbGeometry::row_tiled_index over (n, c).
BT_HD size_t act_npad(size_t n, int tiled, size_t bh) { return ru(n, tiled ? bh : 8); }
BT_HD size_t act_cpad(size_t c, int tiled, size_t bw) { return ru(c, tiled ? bw : 128); }
BT_HD size_t act_words(size_t h, size_t w, size_t n, size_t c, int tiled, size_t bh, size_t bw) {
  return h * w * act_npad(n, tiled, bh) * act_cpad(c, tiled, bw) / 64;
}
BT_HD size_t act_bit(size_t w, size_t n, size_t c, int tiled, size_t bh, size_t bw, size_t hh, size_t ww,
                     size_t nn, size_t cc) {
  const size_t np = act_npad(n, tiled, bh), cp = act_cpad(c, tiled, bw);
  const size_t base = (hh * w + ww) * np * cp;
  if (!tiled) return base + nn * cp + cc;
  return base + ((nn / bh) * (cp / bw) + cc / bw) * (bh * bw) + (nn % bh) * bw + (cc % bw);
}
// Inverse within one site plane: plane bit b -> (n, c); false for pad bits.
BT_HD bool act_plane_inv(size_t n, size_t c, int tiled, size_t bh, size_t bw, size_t b, size_t* nn, size_t* cc) {
  const size_t cp = act_cpad(c, tiled, bw);
  size_t a, k;
  if (!tiled) {
    a = b / cp; k = b % cp;
  } else {
    const size_t tile = b / (bh * bw), in = b % (bh * bw), tpr = cp / bw;
    a = (tile / tpr) * bh + in / bw; k = (tile % tpr) * bw + in % bw;
  }
  *nn = a; *cc = k;
  return a < n && k < c;
}

// BitFilterKKOC (tensors.hpp:127-147) — tiled uses col_tiled_index(c, o, c_pad).
BT_HD size_t filt_opad(size_t o, int tiled, size_t bh) { return ru(o, tiled ? bh : 8); }
BT_HD size_t filt_cpad(size_t c, int tiled, size_t bw) { return ru(c, tiled ? bw : 128); }
BT_HD size_t filt_words(size_t kh, size_t kw, size_t o, size_t c, int tiled, size_t bh, size_t bw) {
  return kh * kw * filt_opad(o, tiled, bh) * filt_cpad(c, tiled, bw) / 64;
}
BT_HD size_t filt_bit(size_t kw, size_t o, size_t c, int tiled, size_t bh, size_t bw, size_t r, size_t s,
                      size_t oo, size_t cc) {
  const size_t op = filt_opad(o, tiled, bh), cp = filt_cpad(c, tiled, bw);
  const size_t base = (r * kw + s) * op * cp;
  if (!tiled) return base + oo * cp + cc;
  return base + ((oo / bh) * (cp / bw) + cc / bw) * (bh * bw) + (oo % bh) * bw + (cc % bw);
}

BT_HD int bit_get(const uint64_t* w, size_t b) { return (int)((w[b >> 6] >> (b & 63)) & 1u); }

}  // namespace btnn_gpu
