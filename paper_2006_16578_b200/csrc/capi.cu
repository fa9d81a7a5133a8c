// capi.cu — kernel-level C ABI of libbtnn_cuda.so (include/btnn_cuda.h).
//
// Each entry point validates its operands host-side exactly where and in the order the
// reference does (so the same inputs raise the same error class), stages the host
// buffers on the device, runs the sm_100a kernels, and copies the result back.
// Synchronous, like the reference calls (common.hpp:53-75 fork/join).
#include <cuda_runtime.h>

#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "api_internal.cuh"
#include "bnmath.cuh"
#include "common.cuh"
#include "kernels.cuh"
#include "layout.cuh"

namespace btnn_gpu {

thread_local std::string g_last_error;
thread_local int g_device = 0;

void set_last_error(const std::string& m) { g_last_error = m; }

// Per-thread device scratch for the kernel-level BMM / BConv entry points. cudaMalloc /
// cudaFree cost 0.1-1 ms per call (and cudaFree synchronizes the device), more than the
// GEMM itself at the reference's sizes. Every kernel-level call is synchronous (its results
// are copied back on the legacy stream before it returns), so a call may reuse the previous
// call's buffers: slots are handed out in call order and only grow.
struct Scratch {
  void* p = nullptr;
  size_t n = 0;
  template <class T = void>
  T* get() const {
    return static_cast<T*>(p);
  }
  size_t bytes() const { return n; }
};
struct ScratchArena {
  int device = -1;
  std::vector<std::unique_ptr<DevBuf>> slots;
  size_t next = 0;
  std::unique_ptr<TcFilter> tcf;  // tensor-core operand of the last kernel-level GEMM
};
static thread_local ScratchArena g_scratch;
static void scratch_begin() {
  int dev = 0;
  BT_CUDA(cudaGetDevice(&dev));
  if (dev != g_scratch.device) {
    g_scratch.slots.clear();
    g_scratch.tcf.reset();
    g_scratch.device = dev;
  }
  g_scratch.next = 0;
}
static Scratch scratch(size_t bytes) {
  if (g_scratch.next == g_scratch.slots.size()) g_scratch.slots.push_back(std::make_unique<DevBuf>());
  DevBuf& b = *g_scratch.slots[g_scratch.next++];
  if (b.bytes() < bytes) b.alloc(bytes + bytes / 4);
  return Scratch{b.get(), bytes};
}
template <class T>
static Scratch scratch_upload(const T* host, size_t count, cudaStream_t st) {
  Scratch b = scratch(count * sizeof(T));
  if (count) BT_CUDA(cudaMemcpyAsync(b.get(), host, count * sizeof(T), cudaMemcpyHostToDevice, st));
  return b;
}

// FsbGeometry validity as enforced by the BitMatrix / tensor constructors
// (bit_matrix.hpp:67-74, tensors.hpp:82-85, 130-133).
static void check_geo(size_t bh, size_t bw, const char* what) {
  require(bh != 0 && bw != 0, BTNN_INVALID_INPUT, std::string(what) + ": zero tile dimension");
  require((bh * bw) % 64 == 0, BTNN_UNSUPPORTED_SHAPE,
          std::string(what) + ": tile size " + std::to_string(bh) + "x" + std::to_string(bw) +
              " is not a whole number of words");
}
void check_matrix_desc(const btnn_matrix_desc* d) {
  require(d != nullptr, BTNN_INVALID_INPUT, "BitMatrix: null descriptor");
  require(d->layout >= 0 && d->layout <= 3, BTNN_INVALID_INPUT, "BitMatrix: unknown layout");
  require(d->rows != 0 && d->cols != 0, BTNN_INVALID_INPUT, "BitMatrix: zero dimension");
  if (d->layout == BTNN_FSB_ROW || d->layout == BTNN_FSB_COL) check_geo(d->bh, d->bw, "BitMatrix");
}
void check_act_desc(const btnn_act_desc* d) {
  require(d != nullptr, BTNN_INVALID_INPUT, "BitTensorHWNC: null descriptor");
  require(d->height && d->width && d->batch && d->channels, BTNN_INVALID_INPUT, "BitTensorHWNC: zero dimension");
  if (d->tiled)
    require(d->bh * d->bw != 0 && (d->bh * d->bw) % 64 == 0, BTNN_UNSUPPORTED_SHAPE,
            "BitTensorHWNC: tile size is not a whole number of words");
}
void check_filter_desc(const btnn_filter_desc* d) {
  require(d != nullptr, BTNN_INVALID_INPUT, "BitFilterKKOC: null descriptor");
  require(d->kh && d->kw && d->out_channels && d->in_channels, BTNN_INVALID_INPUT, "BitFilterKKOC: zero dimension");
  if (d->tiled)
    require(d->bh * d->bw != 0 && (d->bh * d->bw) % 64 == 0, BTNN_UNSUPPORTED_SHAPE,
            "BitFilterKKOC: tile size is not a whole number of words");
}

// Conv2dGeometry::out_h/out_w (tensors.hpp:250-257).
size_t conv_out(size_t x, size_t k, size_t stride, size_t pad, bool height) {
  require(stride != 0, BTNN_INVALID_INPUT, "Conv2dGeometry: zero kernel or stride");
  require(x + 2 * pad >= k, BTNN_UNSUPPORTED_SHAPE,
          height ? "conv: input shorter than kernel" : "conv: input narrower than kernel");
  return (x + 2 * pad - k) / stride + 1;
}

// Threshold::fire (layer_math.hpp:44-52) on an integer v as an inclusive integer range:
// Geq: v >= ceil(tau); Leq: v <= floor(tau); Const*: always / never. Exact for every
// int32 v (values are clamped to +-2^40, far outside any conv/BMM result).
void thresholds_to_int(const double* tau, const uint8_t* kind, size_t n, std::vector<long long>& lo,
                       std::vector<long long>& hi) {
  const long long BIG = 1LL << 40;
  auto clampll = [&](double x) -> long long { return x >= (double)BIG ? BIG : (x <= -(double)BIG ? -BIG : (long long)x); };
  lo.resize(n);
  hi.resize(n);
  for (size_t i = 0; i < n; ++i) {
    switch (kind[i]) {
      case BTNN_GEQ:
        if (std::isnan(tau[i])) { lo[i] = BIG; hi[i] = -BIG; }
        else { lo[i] = clampll(std::ceil(tau[i])); hi[i] = BIG; }
        break;
      case BTNN_LEQ:
        if (std::isnan(tau[i])) { lo[i] = BIG; hi[i] = -BIG; }
        else { lo[i] = -BIG; hi[i] = clampll(std::floor(tau[i])); }
        break;
      case BTNN_CONST_PLUS: lo[i] = -BIG; hi[i] = BIG; break;
      case BTNN_CONST_MINUS: lo[i] = BIG; hi[i] = -BIG; break;
      default: fail(BTNN_INVALID_INPUT, "threshold: unknown kind " + std::to_string(kind[i]));
    }
  }
}

// bn parameters as the device epilogue consumes them: mean, s = sqrt(var + eps) (IEEE
// add then IEEE sqrt, as BnParams::apply computes it), gamma, beta.
void bn_to_device_arrays(const btnn_bn& bn, std::vector<double>& packed) {
  const size_t c = bn.channels;
  packed.assign(kBnArrays * c, 0.0);
  for (size_t i = 0; i < c; ++i) {
    volatile double t = bn.var[i] + bn.eps;  // no contraction, no reassociation
    packed[i] = bn.mean[i];
    packed[c + i] = std::sqrt((double)t);
    packed[2 * c + i] = bn.gamma[i];
    packed[3 * c + i] = bn.beta[i];
  }
}
DevBuf upload_bn(const btnn_bn& bn, cudaStream_t st) {
  std::vector<double> p;
  bn_to_device_arrays(bn, p);
  DevBuf d = upload(p.data(), p.size(), st);
  launch_bn_recip(d.get<double>(), (int)bn.channels, st);
  BT_CUDA(cudaStreamSynchronize(st));  // the host staging vector dies here
  return d;
}

// BnParams::validate (layer_math.hpp:19-30).
void check_bn(const btnn_bn& bn) {
  require(bn.channels != 0 && bn.gamma && bn.beta && bn.mean && bn.var, BTNN_INVALID_INPUT,
          "BnParams: channel arrays must be non-empty and equal length");
  require(bn.eps > 0.0 && std::isfinite(bn.eps), BTNN_INVALID_INPUT, "BnParams: eps must be positive and finite");
  for (size_t i = 0; i < bn.channels; ++i)
    require(std::isfinite(bn.gamma[i]) && std::isfinite(bn.beta[i]) && std::isfinite(bn.mean[i]) &&
                std::isfinite(bn.var[i]) && bn.var[i] >= 0.0,
            BTNN_INVALID_INPUT, "BnParams: bad values at channel " + std::to_string(i));
}

// check_bmm_operands (bmm.hpp:57-76) + bmm_blocked's blocking check (:104-105).
static void check_bmm(const btnn_matrix_desc* a, const btnn_matrix_desc* b, const btnn_bmm_options* opt) {
  const int variant = opt ? opt->variant : BTNN_BMM_BLOCKED;
  require(a->cols == b->rows, BTNN_INVALID_INPUT,
          "bmm: inner dimensions differ: " + std::to_string(a->cols) + " vs " + std::to_string(b->rows));
  if (variant == BTNN_BMM_FSB) {
    require(a->layout == BTNN_FSB_ROW && b->layout == BTNN_FSB_COL, BTNN_INVALID_INPUT,
            "bmm: fsb variant requires fsb_row A and fsb_col B");
    require(a->bh == b->bh && a->bw == b->bw, BTNN_UNSUPPORTED_SHAPE, "bmm: operand tile shapes differ");
    require(a->bw % 64 == 0, BTNN_UNSUPPORTED_SHAPE, "bmm: tile width must be a multiple of 64");
  } else {
    require(variant == BTNN_BMM_NAIVE || variant == BTNN_BMM_BLOCKED, BTNN_INVALID_INPUT, "bmm: unknown variant");
    require(a->layout == BTNN_ROW_PACKED && b->layout == BTNN_COL_PACKED, BTNN_INVALID_INPUT,
            "bmm: word variants require row_packed A and col_packed B");
  }
  require(mat_pcols(a->cols, a->layout, a->bh, a->bw) == mat_prows(b->rows, b->layout, b->bh, b->bw),
          BTNN_UNSUPPORTED_SHAPE, "bmm: padded inner widths differ");
  if (variant == BTNN_BMM_BLOCKED && opt) {
    require(opt->blk_rows && opt->blk_cols && opt->blk_k_bits && opt->blk_k_bits % 64 == 0, BTNN_INVALID_INPUT,
            "bmm: blocking must be nonzero with k_bits a multiple of 64");
  }
}

// Stage A (RowPacked) and B (ColPacked) on the device, converting fsb operands.
struct BmmOperands {
  Scratch a, b;
  ConvShape s{};
};
static BmmOperands stage_bmm(const btnn_matrix_desc* a, const uint64_t* aw, const btnn_matrix_desc* b,
                             const uint64_t* bw, cudaStream_t st) {
  BmmOperands op;
  Scratch ta = scratch_upload(aw, mat_words(a->rows, a->cols, a->layout, a->bh, a->bw), st);
  Scratch tb = scratch_upload(bw, mat_words(b->rows, b->cols, b->layout, b->bh, b->bw), st);
  if (a->layout == BTNN_ROW_PACKED) {
    op.a = ta;
  } else {
    op.a = scratch(mat_words(a->rows, a->cols, BTNN_ROW_PACKED, 0, 0) * 8);
    launch_convert_matrix(a->rows, a->cols, a->layout, a->bh, a->bw, ta.get<uint64_t>(), BTNN_ROW_PACKED, 0, 0,
                          op.a.get<uint64_t>(), st);
  }
  if (b->layout == BTNN_COL_PACKED) {
    op.b = tb;
  } else {
    op.b = scratch(mat_words(b->rows, b->cols, BTNN_COL_PACKED, 0, 0) * 8);
    launch_convert_matrix(b->rows, b->cols, b->layout, b->bh, b->bw, tb.get<uint64_t>(), BTNN_COL_PACKED, 0, 0,
                          op.b.get<uint64_t>(), st);
  }
  ConvShape& s = op.s;
  s.P = s.Q = s.H = s.W = 1;
  s.KH = s.KW = s.stride = 1;
  s.pad = 0;
  s.N = (int)a->rows;
  s.in_rps = s.out_rps = (int)a->rows;
  s.cw = (int)(ru(a->cols, 128) / 64);
  s.C = (int)a->cols;
  s.O = (int)b->cols;
  s.f_rps = (int)b->cols;
  s.cwo = (int)(ru(b->cols, 128) / 64);
  return op;
}

static void use_device() {
  BT_CUDA(cudaSetDevice(g_device));
  scratch_begin();
}

// One implicit GEMM for a kernel-level call: the tensor-core operand is expanded from
// the caller's filter for this call (a plan does it once at creation).
static const char* run_gemm(const ConvShape& s0, const uint64_t* act, const uint64_t* filt, const Epi& e,
                            cudaStream_t st) {
  ConvShape s = s0;
  s.halo_ok = s.C <= 128;
  if (!g_scratch.tcf) g_scratch.tcf = std::make_unique<TcFilter>();
  TcFilter& tcf = *g_scratch.tcf;
  const bool tc = engine_override() != BTNN_ENGINE_POPC && tc_supported(s, e);
  if (tc) tc_prepare_filter(s, filt, tcf, st);
  return launch_bgemm(s, act, filt, e, st, EngineHint::Auto, tc ? &tcf : nullptr);
}

// Kernel-level BMM (bmm.hpp:204-274): one tensor-core kernel on the packed operands
// (bmm_tc.cu: whole-K or K-pipelined); the CUDA-core engine when forced.
static const char* run_bmm(const ConvShape& s, const uint64_t* a, const uint64_t* b, const Epi& e, cudaStream_t st) {
  if (engine_override() != BTNN_ENGINE_POPC) return launch_bmm_packed(s.N, s.O, s.C, a, b, e, st);
  return run_gemm(s, a, b, e, st);
}

}  // namespace btnn_gpu

using namespace btnn_gpu;

extern "C" {

int btnn_cuda_abi_version(void) { return BTNN_CUDA_ABI_VERSION; }
const char* btnn_cuda_last_error(void) { return g_last_error.c_str(); }

int btnn_cuda_device_count(int* n) {
  return guard([&] {
    int c = 0;
    BT_CUDA(cudaGetDeviceCount(&c));
    *n = c;
  });
}
int btnn_cuda_set_device(int device) {
  return guard([&] {
    int c = 0;
    BT_CUDA(cudaGetDeviceCount(&c));
    require(device >= 0 && device < c, BTNN_INVALID_INPUT, "set_device: no such device");
    g_device = device;
  });
}

size_t btnn_cuda_matrix_words(const btnn_matrix_desc* d) { return mat_words(d->rows, d->cols, d->layout, d->bh, d->bw); }
size_t btnn_cuda_act_words(const btnn_act_desc* d) {
  return act_words(d->height, d->width, d->batch, d->channels, d->tiled, d->bh, d->bw);
}
size_t btnn_cuda_filter_words(const btnn_filter_desc* d) {
  return filt_words(d->kh, d->kw, d->out_channels, d->in_channels, d->tiled, d->bh, d->bw);
}

// ---------------------------------------------------------------- format stage
int btnn_cuda_pack_matrix(const float* values, size_t n_values, const btnn_matrix_desc* d, uint64_t* out) {
  return guard([&] {
    require(n_values == d->rows * d->cols, BTNN_INVALID_INPUT, "pack_matrix: value count does not match rows*cols");
    check_matrix_desc(d);
    use_device();
    cudaStream_t st = 0;
    DevBuf x = upload(values, n_values, st);
    DevBuf flag(sizeof(int));
    BT_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), st));
    const size_t pc = ru(d->cols, 128);
    DevBuf rp(d->rows * pc / 8);
    BT_CUDA(cudaMemsetAsync(rp.get(), 0, rp.bytes(), st));
    launch_pack_rows(x.get<float>(), d->rows, d->cols, pc / 32, rp.get<uint32_t>(), flag.get<int>(), st);
    int bad = 0;
    BT_CUDA(cudaMemcpyAsync(&bad, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaStreamSynchronize(st));
    require(!bad, BTNN_INVALID_INPUT, "pack_matrix: non-finite value");
    const size_t words = mat_words(d->rows, d->cols, d->layout, d->bh, d->bw);
    if (d->layout == BTNN_ROW_PACKED) {
      BT_CUDA(cudaMemcpy(out, rp.get(), words * 8, cudaMemcpyDeviceToHost));
      return;
    }
    DevBuf o(words * 8);
    launch_convert_matrix(d->rows, d->cols, BTNN_ROW_PACKED, 0, 0, rp.get<uint64_t>(), d->layout, d->bh, d->bw,
                          o.get<uint64_t>(), st);
    BT_CUDA(cudaMemcpy(out, o.get(), words * 8, cudaMemcpyDeviceToHost));
  });
}

int btnn_cuda_pack_nhwc(const float* x, size_t batch, size_t height, size_t width, size_t channels, int tiled,
                        size_t bh, size_t bw, uint64_t* out) {
  return guard([&] {
    btnn_act_desc d{height, width, batch, channels, tiled, bh, bw};
    check_act_desc(&d);
    use_device();
    cudaStream_t st = 0;
    const size_t n = batch * height * width * channels;
    DevBuf dx = upload(x, n, st);
    DevBuf flag(sizeof(int));
    BT_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), st));
    const size_t np = act_npad(batch, 0, 0), cp = act_cpad(channels, 0, 0);
    DevBuf plain(act_words(height, width, batch, channels, 0, 0, 0) * 8);
    BT_CUDA(cudaMemsetAsync(plain.get(), 0, plain.bytes(), st));
    launch_pack_nhwc(dx.get<float>(), (int)batch, (int)height, (int)width, (int)channels, (int)np, (int)cp,
                     plain.get<uint32_t>(), flag.get<int>(), st);
    int bad = 0;
    BT_CUDA(cudaMemcpyAsync(&bad, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaStreamSynchronize(st));
    require(!bad, BTNN_INVALID_INPUT, "pack_nhwc: non-finite value");
    const size_t words = act_words(height, width, batch, channels, tiled, bh, bw);
    if (!tiled) {
      BT_CUDA(cudaMemcpy(out, plain.get(), words * 8, cudaMemcpyDeviceToHost));
      return;
    }
    DevBuf o(words * 8);
    launch_convert_act(height, width, batch, channels, 0, 0, 0, plain.get<uint64_t>(), 1, bh, bw, o.get<uint64_t>(),
                       st);
    BT_CUDA(cudaMemcpy(out, o.get(), words * 8, cudaMemcpyDeviceToHost));
  });
}

static int convert_matrix_entry(const btnn_matrix_desc* src, const uint64_t* sw, int dst_layout, size_t bh, size_t bw,
                                uint64_t* out) {
  return guard([&] {
    use_device();
    cudaStream_t st = 0;
    DevBuf s = upload(sw, mat_words(src->rows, src->cols, src->layout, src->bh, src->bw), st);
    const size_t words = mat_words(src->rows, src->cols, dst_layout, bh, bw);
    DevBuf o(words * 8);
    launch_convert_matrix(src->rows, src->cols, src->layout, src->bh, src->bw, s.get<uint64_t>(), dst_layout, bh, bw,
                          o.get<uint64_t>(), st);
    BT_CUDA(cudaMemcpy(out, o.get(), words * 8, cudaMemcpyDeviceToHost));
  });
}

// to_fsb (bit_matrix.hpp:224-237).
int btnn_cuda_to_fsb(const btnn_matrix_desc* src, const uint64_t* sw, size_t bh, size_t bw, uint64_t* out) {
  int target = -1;
  int st = guard([&] {
    check_matrix_desc(src);
    require(src->layout == BTNN_ROW_PACKED || src->layout == BTNN_COL_PACKED, BTNN_INVALID_INPUT,
            "to_fsb: source is already tiled");
    check_geo(bh, bw, "BitMatrix");
    target = src->layout == BTNN_ROW_PACKED ? BTNN_FSB_ROW : BTNN_FSB_COL;
  });
  return st ? st : convert_matrix_entry(src, sw, target, bh, bw, out);
}
// from_fsb (bit_matrix.hpp:240-253).
int btnn_cuda_from_fsb(const btnn_matrix_desc* src, const uint64_t* sw, uint64_t* out) {
  int target = -1;
  int st = guard([&] {
    check_matrix_desc(src);
    require(src->layout == BTNN_FSB_ROW || src->layout == BTNN_FSB_COL, BTNN_INVALID_INPUT,
            "from_fsb: source is not tiled");
    target = src->layout == BTNN_FSB_ROW ? BTNN_ROW_PACKED : BTNN_COL_PACKED;
  });
  return st ? st : convert_matrix_entry(src, sw, target, 8, 128, out);
}

int btnn_cuda_convert_activations(const btnn_act_desc* src, const uint64_t* sw, int tiled, size_t bh, size_t bw,
                                  uint64_t* out) {
  return guard([&] {
    check_act_desc(src);
    btnn_act_desc d{src->height, src->width, src->batch, src->channels, tiled, bh, bw};
    check_act_desc(&d);
    use_device();
    cudaStream_t st = 0;
    DevBuf s = upload(sw, btnn_cuda_act_words(src), st);
    const size_t words = btnn_cuda_act_words(&d);
    DevBuf o(words * 8);
    launch_convert_act(src->height, src->width, src->batch, src->channels, src->tiled, src->bh, src->bw,
                       s.get<uint64_t>(), tiled, bh, bw, o.get<uint64_t>(), st);
    BT_CUDA(cudaMemcpy(out, o.get(), words * 8, cudaMemcpyDeviceToHost));
  });
}

int btnn_cuda_flatten_to_matrix(const btnn_act_desc* src, const uint64_t* sw, const btnn_matrix_desc* od,
                                uint64_t* out) {
  return guard([&] {
    check_act_desc(src);
    btnn_matrix_desc d = *od;
    d.rows = src->batch;
    d.cols = src->height * src->width * src->channels;
    check_matrix_desc(&d);
    use_device();
    cudaStream_t st = 0;
    DevBuf s = upload(sw, btnn_cuda_act_words(src), st);
    DevBuf plain;
    const uint64_t* act = s.get<uint64_t>();
    if (src->tiled) {
      plain.alloc(act_words(src->height, src->width, src->batch, src->channels, 0, 0, 0) * 8);
      launch_convert_act(src->height, src->width, src->batch, src->channels, 1, src->bh, src->bw, act, 0, 0, 0,
                         plain.get<uint64_t>(), st);
      act = plain.get<uint64_t>();
    }
    const size_t row_words = ru(d.cols, 128) / 64;
    DevBuf rp(d.rows * row_words * 8);
    launch_flatten(act, (int)src->height, (int)src->width, (int)src->batch, (int)src->channels,
                   (int)act_npad(src->batch, 0, 0), (int)act_cpad(src->channels, 0, 0), rp.get<uint64_t>(), row_words,
                   st);
    const size_t words = mat_words(d.rows, d.cols, d.layout, d.bh, d.bw);
    if (d.layout == BTNN_ROW_PACKED) {
      BT_CUDA(cudaMemcpy(out, rp.get(), words * 8, cudaMemcpyDeviceToHost));
      return;
    }
    DevBuf o(words * 8);
    launch_convert_matrix(d.rows, d.cols, BTNN_ROW_PACKED, 0, 0, rp.get<uint64_t>(), d.layout, d.bh, d.bw,
                          o.get<uint64_t>(), st);
    BT_CUDA(cudaMemcpy(out, o.get(), words * 8, cudaMemcpyDeviceToHost));
  });
}

// ---------------------------------------------------------------- BMM
static int bmm_entry(int which, const btnn_matrix_desc* a, const uint64_t* aw, const btnn_matrix_desc* b,
                     const uint64_t* bw, const btnn_bmm_options* opt, const double* tau, const uint8_t* kind,
                     size_t n_thr, void* out) {
  return guard([&] {
    check_matrix_desc(a);
    check_matrix_desc(b);
    if (which == 0)
      require(a->cols % 128 == 0, BTNN_UNSUPPORTED_SHAPE, "bmm_raw: inner dimension must be a multiple of 128");
    if (which == 2)
      require(n_thr == 0 || n_thr == b->cols, BTNN_INVALID_INPUT, "bmm_pm1_bin: need one threshold per output column");
    check_bmm(a, b, opt);
    std::vector<long long> lo, hi;
    if (which == 2 && n_thr) thresholds_to_int(tau, kind, n_thr, lo, hi);
    use_device();
    cudaStream_t st = 0;
    BmmOperands op = stage_bmm(a, aw, b, bw, st);
    Epi e;
    if (which < 2) {
      Scratch o = scratch(a->rows * b->cols * 4);
      e.mode = EPI_I32;
      e.raw = which == 0;
      e.out_i32 = o.get<int32_t>();
      run_bmm(op.s, op.a.get<uint64_t>(), op.b.get<uint64_t>(), e, st);
      BT_CUDA(cudaMemcpy(out, o.get(), a->rows * b->cols * 4, cudaMemcpyDeviceToHost));
      return;
    }
    Scratch dlo, dhi;
    if (n_thr) {
      dlo = scratch_upload(lo.data(), n_thr, st);
      dhi = scratch_upload(hi.data(), n_thr, st);
      e.thr_lo = dlo.get<long long>();
      e.thr_hi = dhi.get<long long>();
    }
    const size_t rp_words = a->rows * (size_t)op.s.cwo;
    Scratch rp = scratch(rp_words * 8);
    BT_CUDA(cudaMemsetAsync(rp.get(), 0, rp.bytes(), st));
    e.mode = EPI_BITS;
    e.out_bits = rp.get<uint64_t>();
    run_bmm(op.s, op.a.get<uint64_t>(), op.b.get<uint64_t>(), e, st);
    const int out_layout = a->layout == BTNN_FSB_ROW ? BTNN_FSB_ROW : BTNN_ROW_PACKED;
    const size_t words = mat_words(a->rows, b->cols, out_layout, a->bh, a->bw);
    if (out_layout == BTNN_ROW_PACKED) {
      BT_CUDA(cudaMemcpy(out, rp.get(), words * 8, cudaMemcpyDeviceToHost));
      return;
    }
    Scratch o = scratch(words * 8);
    launch_convert_matrix(a->rows, b->cols, BTNN_ROW_PACKED, 0, 0, rp.get<uint64_t>(), out_layout, a->bh, a->bw,
                          o.get<uint64_t>(), st);
    BT_CUDA(cudaMemcpy(out, o.get(), words * 8, cudaMemcpyDeviceToHost));
  });
}

int btnn_cuda_bmm_raw(const btnn_matrix_desc* a, const uint64_t* aw, const btnn_matrix_desc* b, const uint64_t* bw,
                      const btnn_bmm_options* opt, int32_t* out) {
  return bmm_entry(0, a, aw, b, bw, opt, nullptr, nullptr, 0, out);
}
int btnn_cuda_bmm_pm1(const btnn_matrix_desc* a, const uint64_t* aw, const btnn_matrix_desc* b, const uint64_t* bw,
                      const btnn_bmm_options* opt, int32_t* out) {
  return bmm_entry(1, a, aw, b, bw, opt, nullptr, nullptr, 0, out);
}
int btnn_cuda_bmm_pm1_bin(const btnn_matrix_desc* a, const uint64_t* aw, const btnn_matrix_desc* b,
                          const uint64_t* bw, const btnn_bmm_options* opt, const double* tau, const uint8_t* kind,
                          size_t n_thr, uint64_t* out) {
  return bmm_entry(2, a, aw, b, bw, opt, tau, kind, n_thr, out);
}

// ---------------------------------------------------------------- BConv
// Operand checks of bconv_sites (bconv.hpp:79-91).
static void check_conv(const btnn_act_desc* in, const btnn_filter_desc* f, const btnn_conv_geom* g) {
  require(g->kh && g->kw && g->stride, BTNN_INVALID_INPUT, "Conv2dGeometry: zero kernel or stride");
  require(g->kh == f->kh && g->kw == f->kw, BTNN_INVALID_INPUT, "bconv: geometry kernel does not match filter");
  require(in->channels == f->in_channels, BTNN_INVALID_INPUT, "bconv: channel counts differ");
  require((in->tiled != 0) == (f->tiled != 0), BTNN_INVALID_INPUT, "bconv: operand layouts differ");
  if (in->tiled) {
    require(in->bh == f->bh && in->bw == f->bw, BTNN_UNSUPPORTED_SHAPE, "bconv: operand tile shapes differ");
    require(in->bw % 64 == 0, BTNN_UNSUPPORTED_SHAPE, "bconv: tile width must be a multiple of 64");
  }
}

struct ConvOperands {
  Scratch in, filt;
  ConvShape s{};
};
static ConvOperands stage_conv(const btnn_act_desc* in, const uint64_t* iw, const btnn_filter_desc* f,
                               const uint64_t* fw, const btnn_conv_geom* g, size_t P, size_t Q, cudaStream_t st) {
  ConvOperands op;
  Scratch ti = scratch_upload(iw, btnn_cuda_act_words(in), st);
  Scratch tf = scratch_upload(fw, btnn_cuda_filter_words(f), st);
  if (!in->tiled) {
    op.in = ti;
    op.filt = tf;
  } else {
    op.in = scratch(act_words(in->height, in->width, in->batch, in->channels, 0, 0, 0) * 8);
    launch_convert_act(in->height, in->width, in->batch, in->channels, 1, in->bh, in->bw, ti.get<uint64_t>(), 0, 0, 0,
                       op.in.get<uint64_t>(), st);
    // Filter planes share the activation plane geometry with n -> o (tensors.hpp:143-147).
    op.filt = scratch(filt_words(f->kh, f->kw, f->out_channels, f->in_channels, 0, 0, 0) * 8);
    launch_convert_act(f->kh, f->kw, f->out_channels, f->in_channels, 1, f->bh, f->bw, tf.get<uint64_t>(), 0, 0, 0,
                       op.filt.get<uint64_t>(), st);
    BT_CUDA(cudaStreamSynchronize(st));
  }
  ConvShape& s = op.s;
  s.P = (int)P; s.Q = (int)Q;
  s.H = (int)in->height; s.W = (int)in->width;
  s.KH = (int)g->kh; s.KW = (int)g->kw; s.stride = (int)g->stride; s.pad = (int)g->pad;
  s.N = (int)in->batch;
  s.in_rps = s.out_rps = (int)act_npad(in->batch, 0, 0);
  s.cw = (int)(act_cpad(in->channels, 0, 0) / 64);
  s.C = (int)in->channels;
  s.O = (int)f->out_channels;
  s.f_rps = (int)filt_opad(f->out_channels, 0, 0);
  s.cwo = (int)(act_cpad(f->out_channels, 0, 0) / 64);
  return op;
}

int btnn_cuda_bconv_pm1(const btnn_act_desc* in, const uint64_t* iw, const btnn_filter_desc* f, const uint64_t* fw,
                        const btnn_conv_geom* g, int32_t* out) {
  return guard([&] {
    check_act_desc(in);
    check_filter_desc(f);
    // IntTensorPQNO out(geo.out_h(...), ...) is built before bconv_sites (bconv.hpp:140-141).
    const size_t P = conv_out(in->height, g->kh, g->stride, g->pad, true);
    const size_t Q = conv_out(in->width, g->kw, g->stride, g->pad, false);
    check_conv(in, f, g);
    use_device();
    cudaStream_t st = 0;
    ConvOperands op = stage_conv(in, iw, f, fw, g, P, Q, st);
    const size_t n_out = P * Q * in->batch * f->out_channels;
    Scratch o = scratch(n_out * 4);
    Epi e;
    e.mode = EPI_I32;
    e.out_i32 = o.get<int32_t>();
    run_gemm(op.s, op.in.get<uint64_t>(), op.filt.get<uint64_t>(), e, st);
    BT_CUDA(cudaMemcpy(out, o.get(), n_out * 4, cudaMemcpyDeviceToHost));
  });
}

int btnn_cuda_bconv_fused(const btnn_act_desc* in, const uint64_t* iw, const btnn_filter_desc* f, const uint64_t* fw,
                          const btnn_conv_geom* g, const btnn_conv_fused* fu, uint64_t* out) {
  return guard([&] {
    check_act_desc(in);
    check_filter_desc(f);
    const size_t O = f->out_channels;
    const bool thresholded = fu->n_thresholds != 0;
    // bconv_fused's own checks (bconv.hpp:163-171), then output dims (:172-173).
    require(thresholded != (fu->bn != nullptr), BTNN_INVALID_INPUT, "bconv_fused: need exactly one of thresholds or bn");
    require(!thresholded || fu->n_thresholds == O, BTNN_INVALID_INPUT, "bconv_fused: need one threshold per output channel");
    require(!fu->bn || fu->bn->channels == O, BTNN_INVALID_INPUT, "bconv_fused: bn channel count does not match filter");
    require(!((fu->residual_in || fu->residual_out) && !fu->bn), BTNN_INVALID_INPUT,
            "bconv_fused: residual ports require the bn route");
    const size_t P = conv_out(in->height, g->kh, g->stride, g->pad, true);
    const size_t Q = conv_out(in->width, g->kw, g->stride, g->pad, false);
    check_conv(in, f, g);
    std::vector<long long> lo, hi;
    std::vector<double> bnp;
    if (thresholded) thresholds_to_int(fu->tau, fu->kind, O, lo, hi);
    if (fu->bn) bn_to_device_arrays(*fu->bn, bnp);
    use_device();
    cudaStream_t st = 0;
    ConvOperands op = stage_conv(in, iw, f, fw, g, P, Q, st);
    const size_t n_out = P * Q * in->batch * O;
    Scratch dlo, dhi, dbn, drin, drout;
    Epi e;
    e.mode = EPI_BITS;
    if (thresholded) {
      dlo = scratch_upload(lo.data(), O, st);
      dhi = scratch_upload(hi.data(), O, st);
      e.thr_lo = dlo.get<long long>();
      e.thr_hi = dhi.get<long long>();
    } else {
      dbn = scratch_upload(bnp.data(), bnp.size(), st);
      launch_bn_recip(dbn.get<double>(), (int)O, st);
      e.bn_mean = dbn.get<double>();
      e.bn_s = e.bn_mean + O;
      e.bn_gamma = e.bn_mean + 2 * O;
      e.bn_beta = e.bn_mean + 3 * O;
      e.bn_rcp = e.bn_mean + 4 * O;
    }
    if (fu->residual_in) {
      drin = scratch_upload(fu->residual_in, n_out, st);
      e.rin = drin.get<double>();
      e.rin_P = (int)P; e.rin_Q = (int)Q; e.rin_C = (int)O; e.rin_halve = 0;
    }
    if (fu->residual_out) {
      drout = scratch(n_out * 8);
      e.rout = drout.get<double>();
    }
    const size_t plain_words = act_words(P, Q, in->batch, O, 0, 0, 0);
    Scratch ob = scratch(plain_words * 8);
    BT_CUDA(cudaMemsetAsync(ob.get(), 0, ob.bytes(), st));
    e.out_bits = ob.get<uint64_t>();
    run_gemm(op.s, op.in.get<uint64_t>(), op.filt.get<uint64_t>(), e, st);
    if (fu->residual_out) BT_CUDA(cudaMemcpyAsync(fu->residual_out, drout.get(), n_out * 8, cudaMemcpyDeviceToHost, st));
    if (!in->tiled) {
      BT_CUDA(cudaMemcpyAsync(out, ob.get(), plain_words * 8, cudaMemcpyDeviceToHost, st));
    } else {
      const size_t words = act_words(P, Q, in->batch, O, 1, in->bh, in->bw);
      Scratch t = scratch(words * 8);
      launch_convert_act(P, Q, in->batch, O, 0, 0, 0, ob.get<uint64_t>(), 1, in->bh, in->bw, t.get<uint64_t>(), st);
      BT_CUDA(cudaMemcpyAsync(out, t.get(), words * 8, cudaMemcpyDeviceToHost, st));
      BT_CUDA(cudaStreamSynchronize(st));
    }
    BT_CUDA(cudaStreamSynchronize(st));
  });
}

int btnn_cuda_first_conv_bwn(const float* x, size_t batch, size_t height, size_t width, size_t channels,
                             const float* weights_pm1, size_t n_weights, size_t kh, size_t kw, size_t out_channels,
                             const btnn_conv_geom* g, double* out) {
  return guard([&] {
    // bconv.hpp:202-208
    require(g->kh && g->kw && g->stride, BTNN_INVALID_INPUT, "Conv2dGeometry: zero kernel or stride");
    require(g->kh == kh && g->kw == kw, BTNN_INVALID_INPUT, "first_conv_bwn: geometry kernel does not match filter");
    require(n_weights == kh * kw * out_channels * channels, BTNN_INVALID_INPUT,
            "first_conv_bwn: weight count does not match dimensions");
    const size_t P = conv_out(height, kh, g->stride, g->pad, true);
    const size_t Q = conv_out(width, kw, g->stride, g->pad, false);
    use_device();
    cudaStream_t st = 0;
    DevBuf dx = upload(x, batch * height * width * channels, st);
    DevBuf dw = upload(weights_pm1, n_weights, st);
    const size_t n_out = P * Q * batch * out_channels;
    DevBuf o(n_out * 8);
    FirstConvArgs a{};
    a.x = dx.get<float>();
    a.w_pm1 = dw.get<float>();
    a.N = (int)batch; a.H = (int)height; a.W = (int)width; a.C = (int)channels; a.O = (int)out_channels;
    a.KH = (int)kh; a.KW = (int)kw; a.stride = (int)g->stride; a.pad = (int)g->pad; a.P = (int)P; a.Q = (int)Q;
    a.out_acc = o.get<double>();
    const int K = (int)(kh * kw * channels);
    DevBuf wb(first_conv_signbits_words((int)out_channels, K) * 4);
    launch_first_conv_signbits(dw.get<float>(), (int)out_channels, K, wb.get<uint32_t>(), st);
    a.wbits = wb.get<uint32_t>();
    if (!try_first_conv_tc_standalone(a, st)) launch_first_conv(a, st);
    BT_CUDA(cudaMemcpy(out, o.get(), n_out * 8, cudaMemcpyDeviceToHost));
  });
}

int btnn_cuda_or_pool(const btnn_act_desc* in, const uint64_t* iw, size_t window, size_t stride, uint64_t* out) {
  return guard([&] {
    check_act_desc(in);
    // bconv.hpp:249-253
    require(window && stride, BTNN_INVALID_INPUT, "or_pool: zero window or stride");
    require(in->height >= window && in->width >= window, BTNN_UNSUPPORTED_SHAPE, "or_pool: input smaller than window");
    require((in->height - window) % stride == 0 && (in->width - window) % stride == 0, BTNN_UNSUPPORTED_SHAPE,
            "or_pool: window placement does not cover the input exactly");
    const size_t oh = (in->height - window) / stride + 1, ow = (in->width - window) / stride + 1;
    use_device();
    cudaStream_t st = 0;
    DevBuf d = upload(iw, btnn_cuda_act_words(in), st);
    const size_t pw = act_npad(in->batch, in->tiled, in->bh) * act_cpad(in->channels, in->tiled, in->bw) / 64;
    DevBuf o(oh * ow * pw * 8);
    launch_or_pool(d.get<uint64_t>(), (int)in->height, (int)in->width, pw, (int)window, (int)stride, (int)oh, (int)ow,
                   o.get<uint64_t>(), st);
    BT_CUDA(cudaMemcpy(out, o.get(), oh * ow * pw * 8, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
