// kernels_popc.cu — CUDA-core kernels: the LOP3+POPC implicit GEMM (any shape), the f64
// first layer, and the format-stage kernels.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "common.cuh"
#include "kernels.cuh"
#include "umma.cuh"
#include "layout.cuh"

namespace btnn_gpu {

// ------------------------------------------------------------------------------------
// Shared epilogue math. All f64 steps use explicit round-to-nearest intrinsics so nvcc
// cannot contract them into FMAs: the reference evaluates
// (x - mean) / sqrt(var + eps) * gamma + beta step by step (layer_math.hpp:32-34,
// built with -ffp-contract=off, CMakeLists.txt:16-18).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ double bn_eval(double v, double mean, double s, double gamma, double beta) {
  return __dadd_rn(__dmul_rn(__ddiv_rn(__dsub_rn(v, mean), s), gamma), beta);
}

// Residual value of output (p,q,n,o) from the tap of the shortcut source: same grid ->
// direct, halved grid -> ((a+b)+c)+d then *0.25, channels >= src.C -> 0.0
// (inference.hpp:43-63).
__device__ __forceinline__ double residual_at(const Epi& e, int p, int q, int n, int o, int N) {
  if (o >= e.rin_C) return 0.0;
  if (!e.rin_halve) return e.rin[(((size_t)p * e.rin_Q + q) * N + n) * e.rin_C + o];
  const size_t Qs = e.rin_Q, C = e.rin_C;
  const double a = e.rin[(((size_t)(2 * p) * Qs + 2 * q) * N + n) * C + o];
  const double b = e.rin[(((size_t)(2 * p) * Qs + 2 * q + 1) * N + n) * C + o];
  const double c = e.rin[(((size_t)(2 * p + 1) * Qs + 2 * q) * N + n) * C + o];
  const double d = e.rin[(((size_t)(2 * p + 1) * Qs + 2 * q + 1) * N + n) * C + o];
  return __dmul_rn(__dadd_rn(__dadd_rn(__dadd_rn(a, b), c), d), 0.25);
}

// ------------------------------------------------------------------------------------
// LOP3+POPC implicit GEMM. Tile 64 rows x 64 output channels, 128 threads, each thread
// 8 rows x 4 channels. Per tap (r,s) the 64 row pointers are resolved once; rows whose
// tap falls outside the frame are masked to contribute nothing (the reference skips
// them and counts `exclude`, bconv.hpp:107-117), and v = C * valid_taps - 2 * acc,
// i.e. C*KH*KW - exclude*C - 2*acc (bconv.hpp:127-130). For BMM (1x1, one site) this
// is n - 2*acc (bmm.hpp:219-228).
// ------------------------------------------------------------------------------------
namespace {
constexpr int BM = 64, BN = 64, KC = 8, NT = 128;
}

__global__ void __launch_bounds__(NT) bgemm_popc_kernel(ConvShape s, const uint64_t* __restrict__ act,
                                                        const uint64_t* __restrict__ filt, Epi e) {
  __shared__ uint64_t As[KC][BM];
  __shared__ uint64_t Bs[KC][BN];
  __shared__ const uint64_t* arow[BM];
  __shared__ int rvalid[BM], rsite[BM], rn[BM];

  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const long long M = (long long)s.P * s.Q * s.N;
  const long long m0 = (long long)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;

  if (tid < BM) {
    const long long m = m0 + tid;
    int site = -1, n = 0, cnt = 0;
    if (m < M) {
      site = (int)(m / s.N);
      n = (int)(m % s.N);
      const int p = site / s.Q, q = site % s.Q;
      for (int r = 0; r < s.KH; ++r)
        for (int c = 0; c < s.KW; ++c) {
          const int hh = p * s.stride + r - s.pad, ww = q * s.stride + c - s.pad;
          cnt += (hh >= 0 && ww >= 0 && hh < s.H && ww < s.W);
        }
    }
    rsite[tid] = site;
    rn[tid] = n;
    rvalid[tid] = cnt;
  }

  int acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;

  const int ntaps = s.KH * s.KW;
  for (int t = 0; t < ntaps; ++t) {
    const int r = t / s.KW, c = t % s.KW;
    __syncthreads();
    if (tid < BM) {
      const int site = rsite[tid];
      const uint64_t* ptr = nullptr;
      if (site >= 0) {
        const int p = site / s.Q, q = site % s.Q;
        const int hh = p * s.stride + r - s.pad, ww = q * s.stride + c - s.pad;
        if (hh >= 0 && ww >= 0 && hh < s.H && ww < s.W)
          ptr = act + ((size_t)(hh * s.W + ww) * s.in_rps + rn[tid]) * s.cw;
      }
      arow[tid] = ptr;
    }
    __syncthreads();
    uint32_t msk[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) msk[i] = arow[ty + 8 * i] ? 0xffffffffu : 0u;
    const uint64_t* fplane = filt + (size_t)t * s.f_rps * s.cw;
    for (int k0 = 0; k0 < s.cw; k0 += KC) {
#pragma unroll
      for (int u = 0; u < (BM * KC) / NT; ++u) {
        const int idx = tid + NT * u, row = idx / KC, k = idx % KC;
        const uint64_t* p = arow[row];
        As[k][row] = (p && k0 + k < s.cw) ? __ldg(p + k0 + k) : 0ull;
        const int o = n0 + row;
        Bs[k][row] = (o < s.O && k0 + k < s.cw) ? __ldg(fplane + (size_t)o * s.cw + k0 + k) : 0ull;
      }
      __syncthreads();
      const int kmax = min(KC, s.cw - k0);
      for (int k = 0; k < kmax; ++k) {
        uint64_t a[8], b[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = As[k][ty + 8 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t x = a[i] ^ b[j];
            acc[i][j] += __popc((uint32_t)x & msk[i]) + __popc((uint32_t)(x >> 32) & msk[i]);
          }
      }
      __syncthreads();
    }
  }

  // ---- epilogue ----
  const int lane = tid & 31;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = ty + 8 * i;
    const long long m = m0 + row;
    const bool mvalid = m < M;
    const int site = rsite[row], n = rn[row];
    const int p = mvalid ? site / s.Q : 0, q = mvalid ? site % s.Q : 0;
    const int base = s.C * rvalid[row];
    uint64_t word = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int o = n0 + tx + 16 * j;
      const bool valid = mvalid && o < s.O;
      const int v = base - 2 * acc[i][j];
      bool bit = false;
      if (e.mode == EPI_I32) {
        if (valid) e.out_i32[(size_t)m * s.O + o] = e.raw ? acc[i][j] : v;
      } else if (valid) {
        if (e.bn_mean) {
          double y = bn_eval((double)v, e.bn_mean[o], e.bn_s[o], e.bn_gamma[o], e.bn_beta[o]);
          if (e.rin) y = __dadd_rn(y, residual_at(e, p, q, n, o, s.N));
          if (e.rout) e.rout[(size_t)m * s.O + o] = y;
          bit = y >= 0.0;
        } else if (e.thr_lo) {
          bit = (long long)v >= e.thr_lo[o] && (long long)v <= e.thr_hi[o];
        } else {
          bit = v >= 0;  // bmm_pm1_bin with no thresholds (bmm.hpp:608-610)
        }
      }
      if (e.mode == EPI_BITS) {
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        const uint32_t half = (lane < 16) ? (bal & 0xffffu) : (bal >> 16);
        word |= (uint64_t)half << (16 * j);
      }
    }
    if (e.mode == EPI_BITS && (lane == 0 || lane == 16) && mvalid)
      e.out_bits[((size_t)site * s.out_rps + n) * s.cwo + n0 / 64] = word;
  }
}

void launch_bgemm_popc(const ConvShape& s, const uint64_t* act, const uint64_t* filt, const Epi& e,
                       cudaStream_t st) {
  const long long M = (long long)s.P * s.Q * s.N;
  if (M == 0 || s.O == 0) return;
  dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((s.O + BN - 1) / BN));
  bgemm_popc_kernel<<<grid, NT, 0, st>>>(s, act, filt, e);
  BT_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------------------------
// First layer: f64 sums in the exact (r, s, c) order of the reference
// (bconv.hpp:221-235). x * (+-1) is exact, so each step is one correctly rounded add.
// One thread per output (site, n, o); o fastest so a warp shares its input window.
// ------------------------------------------------------------------------------------
__global__ void first_conv_kernel(FirstConvArgs a) {
  const size_t total = (size_t)a.P * a.Q * a.N * a.O;
  const size_t stride_all = (size_t)gridDim.x * blockDim.x;
  const bool warp_pack = (a.O % 32) == 0;
  for (size_t base = (size_t)blockIdx.x * blockDim.x; base < total; base += stride_all) {
    const size_t idx = base + threadIdx.x;
    const bool live = idx < total;
    double y = 0.0;
    bool bit = false;
    int o = 0, n = 0, site = 0;
    if (live) {
      o = (int)(idx % a.O);
      const size_t rest = idx / a.O;
      n = (int)(rest % a.N);
      site = (int)(rest / a.N);
      const int p = site / a.Q, q = site % a.Q;
      const float* wb = a.w_pm1 + (size_t)o * a.KH * a.KW * a.C;
      double acc = 0.0;
      for (int r = 0; r < a.KH; ++r) {
        const int hh = p * a.stride + r - a.pad;
        if (hh < 0 || hh >= a.H) continue;
        for (int s = 0; s < a.KW; ++s) {
          const int ww = q * a.stride + s - a.pad;
          if (ww < 0 || ww >= a.W) continue;
          const float* xr = a.x + (((size_t)n * a.H + hh) * a.W + ww) * a.C;
          const float* wr = wb + (r * a.KW + s) * a.C;
          for (int c = 0; c < a.C; ++c)
            acc = __dadd_rn(acc, __dmul_rn((double)__ldg(xr + c), (double)__ldg(wr + c)));
        }
      }
      if (a.out_acc) a.out_acc[idx] = acc;
      if (a.out_bits) {
        y = bn_eval(acc, a.bn_mean[o], a.bn_s[o], a.bn_gamma[o], a.bn_beta[o]);
        if (a.tap) a.tap[idx] = y;
        bit = y >= 0.0;
      }
    }
    if (a.out_bits) {
      uint32_t* ob = reinterpret_cast<uint32_t*>(a.out_bits);
      if (warp_pack) {
        // total is a multiple of 32 here, so whole warps are live or dead together.
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        if (live && (threadIdx.x & 31) == 0)
          ob[(((size_t)site * a.out_rps + n) * a.cwo * 64 + o) / 32] = bal;
      } else if (live && bit) {
        const size_t b = ((size_t)site * a.out_rps + n) * a.cwo * 64 + o;
        atomicOr(ob + b / 32, 1u << (b % 32));
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// First layer, register-blocked variant for the stock shapes (KHxKWxC compile-time,
// O % 32 == 0, O <= 128). One block per (image n, output row p); warp w owns sites
// q = 8w..8w+7 of that row, lane l owns channels o = l + 32j (j < J). The KH input rows
// are staged in shared memory as f64 (zero outside the frame: adding +-0.0 to an
// accumulator that starts at +0.0 leaves it unchanged, so zero-fill is bit-identical to
// the reference's skip). Each term is DFMA(x, +-1.0, acc): x * (+-1) is exact, so the
// single rounding equals the reference's add (bconv.hpp:233-234), in the same
// (r, s, c) order. Weight signs live in registers (one bit per (o, k)).
// ------------------------------------------------------------------------------------
template <int KH, int KW, int C, int J>
__global__ void __launch_bounds__(256) first_conv_tiled_kernel(FirstConvArgs a, const uint32_t* __restrict__ wbits) {
  constexpr int K = KH * KW * C, KWORDS = (K + 31) / 32, SQ = 8;
  constexpr int CP = C == 3 ? 4 : C;  // channel pitch in smem: 3 -> 4 so a tap is one 16 B + one 8 B load
  extern __shared__ double patch[];   // [KH][Wp][CP], Wp = W + 2*pad + slack
  const int n = blockIdx.x / a.P, p = blockIdx.x % a.P;
  const int Wp = (a.Q - 1) * a.stride + KW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // stage rows hh = p*stride - pad + r, cols ww = col - pad
  for (int i = threadIdx.x; i < KH * Wp * CP; i += blockDim.x) {
    const int c = i % CP, col = (i / CP) % Wp, r = i / (CP * Wp);
    const int hh = p * a.stride - a.pad + r, ww = col - a.pad;
    double v = 0.0;
    if (c < C && hh >= 0 && hh < a.H && ww >= 0 && ww < a.W)
      v = (double)__ldg(a.x + (((size_t)n * a.H + hh) * a.W + ww) * C + c);
    patch[i] = v;
  }
  uint32_t wb[J][KWORDS];
#pragma unroll
  for (int j = 0; j < J; ++j)
#pragma unroll
    for (int w = 0; w < KWORDS; ++w) wb[j][w] = __ldg(wbits + (size_t)(lane + 32 * j) * KWORDS + w);
  __syncthreads();
  const int q0 = warp * SQ;
  if (q0 >= a.Q) return;  // whole warp idle (no ballots pending)
  double acc[SQ][J];
#pragma unroll
  for (int i = 0; i < SQ; ++i)
#pragma unroll
    for (int j = 0; j < J; ++j) acc[i][j] = 0.0;
  int qoff[SQ];  // smem offset of each site's window column
#pragma unroll
  for (int i = 0; i < SQ; ++i) qoff[i] = min(q0 + i, a.Q - 1) * a.stride * CP;
#pragma unroll
  for (int r = 0; r < KH; ++r)
#pragma unroll
    for (int s = 0; s < KW; ++s) {
      // this tap's +-1 weights once, then per site its C inputs (broadcast loads) and the
      // terms in c order — every accumulator still sees (r, s, c) order.
      double w[C][J];
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const int k = (r * KW + s) * C + c;
          w[c][j] = __hiloint2double((int)(0x3FF00000u | ((~wb[j][k >> 5] >> (k & 31)) & 1u) << 31), 0);
        }
      const double* base = patch + ((size_t)r * Wp + s) * CP;
#pragma unroll
      for (int i = 0; i < SQ; ++i) {
        double x[CP];
        if constexpr (CP == 4) {
          const double2 v01 = *reinterpret_cast<const double2*>(base + qoff[i]);
          x[0] = v01.x;
          x[1] = v01.y;
          x[2] = base[qoff[i] + 2];
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) x[c] = base[qoff[i] + c];
        }
#pragma unroll
        for (int c = 0; c < C; ++c)
#pragma unroll
          for (int j = 0; j < J; ++j) acc[i][j] = __fma_rn(x[c], w[c][j], acc[i][j]);
      }
    }
  uint32_t* ob = reinterpret_cast<uint32_t*>(a.out_bits);
#pragma unroll
  for (int i = 0; i < SQ; ++i) {
    const int q = q0 + i;
    const bool live = q < a.Q;
    const int site = p * a.Q + (live ? q : 0);
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int o = lane + 32 * j;
      const size_t idx = ((size_t)site * a.N + n) * a.O + o;
      if (live && a.out_acc) a.out_acc[idx] = acc[i][j];
      if (a.out_bits) {
        const double y = bn_eval(acc[i][j], a.bn_mean[o], a.bn_s[o], a.bn_gamma[o], a.bn_beta[o]);
        if (live && a.tap) a.tap[idx] = y;
        const uint32_t bal = __ballot_sync(0xffffffffu, y >= 0.0);
        if (live && lane == 0) ob[(((size_t)site * a.out_rps + n) * a.cwo * 64 + 32 * j) / 32] = bal;
      }
    }
  }
}

// (o, r, s, c) +-1 floats -> per-o sign bits, bit k = (w >= 0) in (r, s, c) order.
__global__ void first_conv_signbits_kernel(const float* __restrict__ w, int O, int K, int kwords, uint32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= O * kwords) return;
  const int o = i / kwords, wd = i % kwords;
  uint32_t v = 0;
  for (int b = 0; b < 32; ++b) {
    const int k = wd * 32 + b;
    if (k < K && w[(size_t)o * K + k] >= 0.0f) v |= 1u << b;
  }
  out[i] = v;
}

size_t first_conv_signbits_words(int O, int K) { return (size_t)O * ((K + 31) / 32); }
void launch_first_conv_signbits(const float* w_pm1, int O, int K, uint32_t* out, cudaStream_t st) {
  const int kwords = (K + 31) / 32;
  first_conv_signbits_kernel<<<(O * kwords + 127) / 128, 128, 0, st>>>(w_pm1, O, K, kwords, out);
  BT_CUDA(cudaGetLastError());
}

template <int KH, int KW, int C, int J>
static bool try_first_conv_tiled(const FirstConvArgs& a, cudaStream_t st) {
  if (!a.wbits || a.KH != KH || a.KW != KW || a.C != C || a.O != 32 * J) return false;
  const int Wp = (a.Q - 1) * a.stride + KW;
  const size_t smem = (size_t)KH * Wp * (C == 3 ? 4 : C) * sizeof(double);
  const int warps = (a.Q + 7) / 8;
  if (smem > 200 * 1024 || warps > 8) return false;
  auto kern = first_conv_tiled_kernel<KH, KW, C, J>;
  BT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<(unsigned)(a.N * a.P), 32 * warps, smem, st>>>(a, a.wbits);
  BT_CUDA(cudaGetLastError());
  return true;
}

void launch_first_conv(const FirstConvArgs& a, cudaStream_t st) {
  const size_t total = (size_t)a.P * a.Q * a.N * a.O;
  if (!total) return;
  if (try_first_conv_tiled<7, 7, 3, 2>(a, st) || try_first_conv_tiled<11, 11, 3, 4>(a, st) ||
      try_first_conv_tiled<3, 3, 3, 4>(a, st) || try_first_conv_tiled<3, 3, 3, 2>(a, st) ||
      try_first_conv_tiled<7, 7, 3, 4>(a, st))
    return;
  const int threads = 256;
  const size_t blocks = (total + threads - 1) / threads;
  first_conv_kernel<<<(unsigned)(blocks < 148 * 64 ? blocks : 148 * 64), threads, 0, st>>>(a);
  BT_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------------------------
// Format stage.
// ------------------------------------------------------------------------------------
__global__ void check_finite_kernel(const float* __restrict__ x, size_t n, int* flag) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) atomicExch(flag, 1);
}
void launch_check_finite(const float* x, size_t n, int* flag, cudaStream_t st) {
  if (!n) return;
  const size_t blocks = (n + 255) / 256;
  check_finite_kernel<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, st>>>(x, n, flag);
  BT_CUDA(cudaGetLastError());
}

// One warp per 32 consecutive columns of a row: bit = x >= 0 (bit_buffer.hpp:83), pad
// columns 0, the ballot is the 32-bit word; every word of the padded row is written (no
// clearing pass). The next kernel may launch early (it waits for this grid's writes).
__global__ void pack_rows_kernel(const float* __restrict__ x, size_t rows, size_t cols, size_t row_words32,
                                 uint32_t* out, int* nonfinite) {
  umma::grid_dep_launch();
  const size_t cols32 = row_words32 * 32;
  const size_t total = rows * cols32;
  for (size_t base = (size_t)blockIdx.x * blockDim.x; base < total; base += (size_t)gridDim.x * blockDim.x) {
    const size_t idx = base + threadIdx.x;
    bool bit = false;
    size_t r = 0, c = 0;
    if (idx < total) {
      r = idx / cols32;
      c = idx % cols32;
      if (c < cols) {
        const float v = x[r * cols + c];
        if (!isfinite(v)) atomicExch(nonfinite, 1);
        bit = v >= 0.0f;
      }
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, bit);
    if (idx < total && (threadIdx.x & 31) == 0) out[r * row_words32 + c / 32] = bal;
  }
}
void launch_pack_rows(const float* x, size_t rows, size_t cols, size_t row_words32, uint32_t* out,
                      int* nonfinite, cudaStream_t st) {
  const size_t total = rows * row_words32 * 32;
  if (!total) return;
  const size_t blocks = (total + 255) / 256;
  pack_rows_kernel<<<(unsigned)(blocks < 148 * 32 ? blocks : 148 * 32), 256, 0, st>>>(x, rows, cols, row_words32,
                                                                                      out, nonfinite);
  BT_CUDA(cudaGetLastError());
}

__global__ void pack_nhwc_kernel(const float* __restrict__ x, int N, int H, int W, int C, int n_pad, int c_pad,
                                 uint32_t* out, int* nonfinite) {
  const int C32 = (C + 31) / 32 * 32;
  const size_t total = (size_t)N * H * W * C32;
  for (size_t base = (size_t)blockIdx.x * blockDim.x; base < total; base += (size_t)gridDim.x * blockDim.x) {
    const size_t idx = base + threadIdx.x;
    bool bit = false;
    size_t word = 0;
    if (idx < total) {
      const int c = (int)(idx % C32);
      const size_t pix = idx / C32;  // (n*H + h)*W + w
      const int w = (int)(pix % W), h = (int)((pix / W) % H), n = (int)(pix / ((size_t)W * H));
      if (c < C) {
        const float v = x[pix * C + c];
        if (!isfinite(v)) atomicExch(nonfinite, 1);
        bit = v >= 0.0f;
      }
      word = (((size_t)h * W + w) * n_pad + n) * (c_pad / 32) + c / 32;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, bit);
    if (idx < total && (threadIdx.x & 31) == 0) out[word] = bal;
  }
}
void launch_pack_nhwc(const float* x, int N, int H, int W, int C, int n_pad, int c_pad, uint32_t* out,
                      int* nonfinite, cudaStream_t st) {
  const size_t total = (size_t)N * H * W * ((C + 31) / 32 * 32);
  if (!total) return;
  const size_t blocks = (total + 255) / 256;
  pack_nhwc_kernel<<<(unsigned)(blocks < 148 * 32 ? blocks : 148 * 32), 256, 0, st>>>(x, N, H, W, C, n_pad, c_pad,
                                                                                      out, nonfinite);
  BT_CUDA(cudaGetLastError());
}

// Layout conversions. Word path: when source and destination run along the same fast index
// (RowPacked / fsb_row: columns; ColPacked / fsb_col: rows) and every fsb tile width is a
// multiple of 64, each destination word is one aligned source word (pad bits masked) — one
// load per word. Otherwise bit by bit.
__global__ void convert_matrix_kernel(size_t rows, size_t cols, int sl, size_t sbh, size_t sbw,
                                      const uint64_t* __restrict__ src, int dl, size_t dbh, size_t dbw,
                                      uint64_t* dst, size_t dst_words, int word_path) {
  const bool row_major = dl == BTNN_ROW_PACKED || dl == BTNN_FSB_ROW;
  for (size_t wi = (size_t)blockIdx.x * blockDim.x + threadIdx.x; wi < dst_words;
       wi += (size_t)gridDim.x * blockDim.x) {
    uint64_t word = 0;
    if (word_path) {
      size_t r, c;
      mat_inv(rows, cols, dl, dbh, dbw, wi * 64, &r, &c);  // first bit of the word (fast index % 64 == 0)
      const size_t fast = row_major ? c : r, nfast = row_major ? cols : rows;
      if ((row_major ? r < rows : c < cols) && fast < nfast) {
        word = __ldg(src + mat_bit(rows, cols, sl, sbh, sbw, r, c) / 64);
        if (nfast - fast < 64) word &= (1ull << (nfast - fast)) - 1ull;
      }
    } else {
      for (int b = 0; b < 64; ++b) {
        size_t r, c;
        if (mat_inv(rows, cols, dl, dbh, dbw, wi * 64 + b, &r, &c) &&
            bit_get(src, mat_bit(rows, cols, sl, sbh, sbw, r, c)))
          word |= 1ull << b;
      }
    }
    dst[wi] = word;
  }
}
void launch_convert_matrix(size_t rows, size_t cols, int sl, size_t sbh, size_t sbw, const uint64_t* src, int dl,
                           size_t dbh, size_t dbw, uint64_t* dst, cudaStream_t st) {
  const size_t words = mat_words(rows, cols, dl, dbh, dbw);
  if (!words) return;
  auto rowish = [](int l) { return l == BTNN_ROW_PACKED || l == BTNN_FSB_ROW; };
  auto w64 = [](int l, size_t bw) { return (l != BTNN_FSB_ROW && l != BTNN_FSB_COL) || bw % 64 == 0; };
  const int word_path = rowish(sl) == rowish(dl) && w64(sl, sbw) && w64(dl, dbw);
  const size_t blocks = (words + 255) / 256;
  convert_matrix_kernel<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, st>>>(
      rows, cols, sl, sbh, sbw, src, dl, dbh, dbw, dst, words, word_path);
  BT_CUDA(cudaGetLastError());
}

__global__ void convert_act_kernel(size_t h, size_t w, size_t n, size_t c, int st_, size_t sbh, size_t sbw,
                                   const uint64_t* __restrict__ src, int dt, size_t dbh, size_t dbw, uint64_t* dst,
                                   size_t dst_words, int word_path) {
  const size_t dplane = act_npad(n, dt, dbh) * act_cpad(c, dt, dbw) / 64;
  for (size_t wi = (size_t)blockIdx.x * blockDim.x + threadIdx.x; wi < dst_words;
       wi += (size_t)gridDim.x * blockDim.x) {
    const size_t site = wi / dplane, inw = wi % dplane;
    const size_t hh = site / w, ww = site % w;
    uint64_t word = 0;
    if (word_path) {  // plain and tiled planes both run along channels
      size_t nn, cc;
      act_plane_inv(n, c, dt, dbh, dbw, inw * 64, &nn, &cc);
      if (nn < n && cc < c) {
        word = __ldg(src + act_bit(w, n, c, st_, sbh, sbw, hh, ww, nn, cc) / 64);
        if (c - cc < 64) word &= (1ull << (c - cc)) - 1ull;
      }
    } else {
      for (int b = 0; b < 64; ++b) {
        size_t nn, cc;
        if (act_plane_inv(n, c, dt, dbh, dbw, inw * 64 + b, &nn, &cc) &&
            bit_get(src, act_bit(w, n, c, st_, sbh, sbw, hh, ww, nn, cc)))
          word |= 1ull << b;
      }
    }
    dst[wi] = word;
  }
}
void launch_convert_act(size_t h, size_t w, size_t n, size_t c, int st_, size_t sbh, size_t sbw,
                        const uint64_t* src, int dt, size_t dbh, size_t dbw, uint64_t* dst, cudaStream_t st) {
  const size_t words = act_words(h, w, n, c, dt, dbh, dbw);
  if (!words) return;
  const int word_path = (!st_ || sbw % 64 == 0) && (!dt || dbw % 64 == 0);
  const size_t blocks = (words + 255) / 256;
  convert_act_kernel<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, st>>>(
      h, w, n, c, st_, sbh, sbw, src, dt, dbh, dbw, dst, words, word_path);
  BT_CUDA(cudaGetLastError());
}

// Row n, feature f = (h*W + w)*C + c (tensors.hpp:226-237). Whole-word copies when C is
// a multiple of 64, bit gathers otherwise.
__global__ void flatten_kernel(const uint64_t* __restrict__ act, int H, int W, int N, int C, int n_pad,
                               int c_pad, uint64_t* out, size_t row_words) {
  const size_t features = (size_t)H * W * C;
  const size_t total = (size_t)N * row_words;
  const int cw = c_pad / 64;
  for (size_t wi = (size_t)blockIdx.x * blockDim.x + threadIdx.x; wi < total;
       wi += (size_t)gridDim.x * blockDim.x) {
    const size_t n = wi / row_words, j = wi % row_words;
    uint64_t word = 0;
    if ((C & 63) == 0) {
      const size_t f = j * 64;
      if (f < features) {
        const size_t site = f / C, cword = (f % C) / 64;
        word = act[(site * n_pad + n) * cw + cword];
      }
    } else {
      for (int b = 0; b < 64; ++b) {
        const size_t f = j * 64 + b;
        if (f >= features) break;
        const size_t site = f / C, c = f % C;
        if ((act[(site * n_pad + n) * cw + c / 64] >> (c % 64)) & 1ull) word |= 1ull << b;
      }
    }
    out[wi] = word;
  }
}
void launch_flatten(const uint64_t* act, int H, int W, int N, int C, int n_pad, int c_pad, uint64_t* out,
                    size_t row_words, cudaStream_t st) {
  const size_t total = (size_t)N * row_words;
  if (!total) return;
  const size_t blocks = (total + 255) / 256;
  flatten_kernel<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, st>>>(act, H, W, N, C, n_pad, c_pad,
                                                                                    out, row_words);
  BT_CUDA(cudaGetLastError());
}

__global__ void or_pool_kernel(const uint64_t* __restrict__ in, int W, size_t plane_words, int window, int stride,
                               int OW, size_t total, uint64_t* out) {
  for (size_t wi = (size_t)blockIdx.x * blockDim.x + threadIdx.x; wi < total;
       wi += (size_t)gridDim.x * blockDim.x) {
    const size_t site = wi / plane_words, k = wi % plane_words;
    const int p = (int)(site / OW), q = (int)(site % OW);
    uint64_t v = 0;
    for (int r = 0; r < window; ++r)
      for (int s = 0; s < window; ++s)
        v |= in[((size_t)(p * stride + r) * W + (q * stride + s)) * plane_words + k];
    out[wi] = v;
  }
}
void launch_or_pool(const uint64_t* in, int H, int W, size_t plane_words, int window, int stride, int OH, int OW,
                    uint64_t* out, cudaStream_t st) {
  (void)H;
  const size_t total = (size_t)OH * OW * plane_words;
  if (!total) return;
  const size_t blocks = (total + 255) / 256;
  or_pool_kernel<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, st>>>(in, W, plane_words, window,
                                                                                    stride, OW, total, out);
  BT_CUDA(cudaGetLastError());
}

// One warp per row: each lane keeps the first maximum of its strided classes, then a
// shuffle reduction keeps the larger value and, on ties, the smaller index — the same
// first-index argmax as the sequential scan (inference.hpp:177-184; logits are finite).
__global__ void argmax_kernel(const double* __restrict__ logits, int batch, int classes, int32_t* labels) {
  const int lane = threadIdx.x & 31;
  for (int n = (blockIdx.x * blockDim.x + threadIdx.x) / 32; n < batch; n += gridDim.x * blockDim.x / 32) {
    const double* row = logits + (size_t)n * classes;
    double bv = lane < classes ? row[lane] : -INFINITY;
    int bi = lane < classes ? lane : INT_MAX;
    for (int j = lane + 32; j < classes; j += 32) {
      const double v = row[j];
      if (v > bv) { bv = v; bi = j; }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) labels[n] = bi;
  }
}
void launch_argmax(const double* logits, int batch, int classes, int32_t* labels, cudaStream_t st) {
  if (batch <= 0) return;
  const int blocks = (batch + 7) / 8;
  argmax_kernel<<<blocks < 148 * 8 ? blocks : 148 * 8, 256, 0, st>>>(logits, batch, classes, labels);
  BT_CUDA(cudaGetLastError());
}

}  // namespace btnn_gpu
