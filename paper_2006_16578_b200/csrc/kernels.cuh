// kernels.cuh — launchers of the sm_100a kernels behind libbtnn_cuda.
//
// One implicit-GEMM description covers both hot functions of the paper: BConv over HWNC
// activations x KKOC filters (bconv.hpp:76-133), and BMM as the 1x1, single-site special
// case (A RowPacked rows = "images", B ColPacked columns = "output channels",
// bmm.hpp:81-99). Every GEMM row is one output (site, n); every column one output channel.
#pragma once
#include <cuda.h>  // CUtensorMap
#include <cuda_runtime.h>

#include <cstdint>

namespace btnn_gpu {

struct ConvShape {
  int P, Q;              // output grid
  int H, W;              // input grid
  int KH, KW, stride, pad;
  int N;                 // logical rows per site (batch); GEMM rows M = P*Q*N
  int in_rps;            // input row pitch per site, in rows (n_pad)
  int out_rps;           // output bit-tensor row pitch per site (n_pad)
  int cw;                // u64 words per input row (c_pad / 64)
  int C;                 // logical inner channels: v = C * valid_taps - 2 * acc
  int O;                 // logical output channels
  int f_rps;             // filter rows per tap plane (o_pad)
  int cwo;               // u64 words per output bit row (out c_pad / 64)
  int halo_ok = 0;       // layer may use the halo-mode tensor-core kernel (fixes the filter layout;
                         // set for threshold-route convs with C <= 128, where it is faster)
};

// Fused epilogue (bconv.hpp:160-194, bmm.hpp:219-274, inference.hpp:107-118/161-164).
enum EpiMode { EPI_I32 = 0, EPI_BITS = 1, EPI_F64 = 2, EPI_SPLIT = 3 /* tensor-core split-K partial sums (internal) */ };
struct Epi {
  int mode = EPI_I32;
  int raw = 0;                       // EPI_I32: write the raw xor-popcount (bmm_raw)
  int32_t* out_i32 = nullptr;        // PQNO / row-major M x O
  uint64_t* out_bits = nullptr;      // HWNC plain / RowPacked words (pre-zeroed)
  const long long* thr_lo = nullptr; // threshold route: bit = lo <= v <= hi (per channel)
  const long long* thr_hi = nullptr;
  const double* bn_mean = nullptr;   // bn route: y = (v - mean) / s * gamma + beta
  const double* bn_s = nullptr;      //   s = sqrt(var + eps), computed on the host in IEEE f64
  const double* bn_gamma = nullptr;
  const double* bn_beta = nullptr;
  const double* bn_rcp = nullptr;    //   per-channel reciprocal for the division (bnmath.cuh), optional
  const double* rin = nullptr;       // residual_in, PQNO over (rin_P, rin_Q, N, rin_C)
  int rin_P = 0, rin_Q = 0, rin_C = 0, rin_halve = 0;  // type-A adaptation (inference.hpp:43-63)
  double* rout = nullptr;            // residual_out / logits, PQNO over (P, Q, N, O)
  int32_t* split_ws = nullptr;       // optional zeroed-by-callee int32 M x O workspace: lets the
                                     //   tensor-core engine split few-tile FC GEMMs along K
  double* rout_half = nullptr;       // residual_out pre-averaged for a halving consumer,
                                     //   PQNO over (P/2, Q/2, N, O) (tensor-core engine only)
  int32_t* labels = nullptr;         // EPI_F64 (the last layer): kernels that can also write each
  bool* labels_done = nullptr;       //   row's argmax set *labels_done (host flag, at launch)
  int pool = 0;                      // fused or_pool (bconv.hpp:247-272) with window = stride = pool:
                                     //   bits are OR-ed (atomicOr) into the pooled site (p/pool, q/pool)
                                     //   of a zeroed (P/pool, Q/pool) tensor (tensor-core engine only)
};

// CUDA-core LOP3+POPC implicit GEMM (any shape). act/filt are device pointers.
void launch_bgemm_popc(const ConvShape& s, const uint64_t* act, const uint64_t* filt, const Epi& e,
                       cudaStream_t st);

// First layer (bconv.hpp:198-243 + inference.hpp:101-120): f64 (r,s,c)-ordered sums.
struct FirstConvArgs {
  const float* x;         // NHWC
  const float* w_pm1;     // (o, r, s, c) +-1 floats
  int N, H, W, C, O, KH, KW, stride, pad, P, Q;
  double* out_acc;        // optional raw sums, PQNO (first_conv_bwn)
  // optional fused bn -> tap -> sign -> HWNC bits (run_inference's loop)
  const double *bn_mean, *bn_s, *bn_gamma, *bn_beta;
  const double* bn_rcp = nullptr;  // optional per-channel reciprocal (bnmath.cuh)
  double* tap;            // optional, PQNO
  uint64_t* out_bits;     // optional, HWNC plain (pre-zeroed)
  int out_rps, cwo;
  const uint32_t* wbits = nullptr;  // optional per-o sign bits (launch_first_conv_signbits)
  int pool = 0;                     // fused or_pool with window = stride = pool (see Epi::pool)
};
void launch_first_conv(const FirstConvArgs& a, cudaStream_t st);
size_t first_conv_signbits_words(int O, int K);
void launch_first_conv_signbits(const float* w_pm1, int O, int K, uint32_t* out, cudaStream_t st);

// Tensor-core first layer (kernels_first_tc.cu): exact integer-digit MMAs with a
// sequential-f64 fix-up pass for windows whose terms do not fit the tile's grid.
// Encode a 4-D f64 TMA tensor map (dims[0] contiguous; strides in bytes for dims 1..3;
// SWIZZLE_128B or dense boxes, out-of-range elements zero-filled on load and clipped on store).
// False when the driver entry point is missing or the layout is not TMA-compatible.
bool encode_f64_map(CUtensorMap* m, const double* base, const uint64_t dims[4], const uint64_t strides[3],
                    const uint32_t box[4], bool swizzle128 = true);

bool first_conv_tc_supported(const FirstConvArgs& a);
size_t first_conv_tc_weight_bytes(int KH, int KW, int O, int stride);
void launch_first_conv_tc_weights(const float* w_pm1, int O, int KH, int KW, int C, int stride, int8_t* out,
                                  cudaStream_t st);
// Input check per row (n, h) of W*C floats: non-finite flag + largest |x| bit pattern.
void launch_input_rows(const float* x, size_t rows, int row_len, int* flag, uint32_t* rowmax, cudaStream_t st);
// rowmax from launch_input_rows; fix_list holds up to N*P*Q window ids.
// True when the tensor-core first conv can take the tile maxima and the input check itself
// (rowmax == nullptr, flag in nonfinite): stride 4, one pixel column per builder thread, and
// the windows cover every input row (so every input value is checked).
bool first_conv_fused_input(const FirstConvArgs& a);
void launch_first_conv_tc(const FirstConvArgs& a, const uint32_t* rowmax, const int8_t* wblk, int* fix_count,
                          int* fix_list, cudaStream_t st, int* nonfinite = nullptr);
bool try_first_conv_tc_standalone(const FirstConvArgs& a, cudaStream_t st);

// Format stage.
void launch_check_finite(const float* x, size_t n, int* flag, cudaStream_t st);
// Sign-binarize a row-major rows x cols f32 matrix into a plain RowPacked bit matrix
// (pack_matrix, bit_matrix.hpp:135-155). out pre-zeroed; row pitch in u32 words.
void launch_pack_rows(const float* x, size_t rows, size_t cols, size_t row_words32, uint32_t* out,
                      int* nonfinite, cudaStream_t st);
// NHWC f32 -> plain HWNC bits (pack_nhwc, tensors.hpp:162-174). out pre-zeroed.
void launch_pack_nhwc(const float* x, int N, int H, int W, int C, int n_pad, int c_pad, uint32_t* out,
                      int* nonfinite, cudaStream_t st);
// Generic matrix layout conversion (to_fsb/from_fsb/any), one thread per output word.
void launch_convert_matrix(size_t rows, size_t cols, int src_layout, size_t sbh, size_t sbw,
                           const uint64_t* src, int dst_layout, size_t dbh, size_t dbw, uint64_t* dst,
                           cudaStream_t st);
// Activation plane layout conversion (convert_activations, tensors.hpp:203-212).
void launch_convert_act(size_t h, size_t w, size_t n, size_t c, int src_tiled, size_t sbh, size_t sbw,
                        const uint64_t* src, int dst_tiled, size_t dbh, size_t dbw, uint64_t* dst,
                        cudaStream_t st);
// flatten_to_matrix (tensors.hpp:226-237) from plain HWNC to plain RowPacked.
void launch_flatten(const uint64_t* act, int H, int W, int N, int C, int n_pad, int c_pad, uint64_t* out,
                    size_t out_row_words, cudaStream_t st);
// or_pool (bconv.hpp:247-272) over whole plane words.
void launch_or_pool(const uint64_t* in, int H, int W, size_t plane_words, int window, int stride, int OH,
                    int OW, uint64_t* out, cudaStream_t st);
// First-index argmax over logits rows (inference.hpp:177-184).
void launch_argmax(const double* logits, int batch, int classes, int32_t* labels, cudaStream_t st);

}  // namespace btnn_gpu
