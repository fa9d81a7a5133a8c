// bench_api.cu — device-timed versions of the reference benchmark suites
// (bench.hpp:129-299): bmm / bmm-bin over n x n x n, bconv / bconv-bin over
// input x input x batch x C -> O with a k x k kernel, stride 1, pad k/2.
//
//   bmm        packed operands + bmm_pm1 (int32), B's tensor-core operand re-expanded per call
//   bmm-bin    packed operands + bmm_pm1_bin with the sign rule (bit output)
//   bconv      float input binarized (pack_nhwc) + bconv_pm1 (int32 PQNO)
//   bconv-bin  packed input + bconv_fused with sign thresholds (tau = 0, Geq; bench.hpp:238)
//
// Operands are random on the device, timing is CUDA events around each launch sequence
// after `warmup` untimed repetitions; median and min over `reps` (bench.hpp:51-70).
// Throughput (reported by the caller) uses the reference's op counts: 2n^3 and
// 2*P*Q*N*C*O*K^2 (bench.hpp:207-209, 290-292).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "api_internal.cuh"
#include "bnmath.cuh"
#include "layout.cuh"

namespace btnn_gpu {

__global__ void rand_words_kernel(uint64_t* w, size_t n, uint64_t seed) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + i * 0x9E3779B97F4A7C15ull;  // splitmix64
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    w[i] = z ^ (z >> 31);
  }
}
__global__ void rand_floats_kernel(float* x, size_t n, uint64_t seed) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    x[i] = (float)((int64_t)(z ^ (z >> 31)) >> 40) * (1.0f / 8388608.0f);  // symmetric, zero-mean
  }
}
static void rand_words(uint64_t* w, size_t n, uint64_t seed, cudaStream_t st) {
  rand_words_kernel<<<148 * 8, 256, 0, st>>>(w, n, seed);
  BT_CUDA(cudaGetLastError());
}
// Zero the bits past `cols` of each of `rows` rows of `kw` words (matrix pad bits are 0,
// bit_buffer.hpp:62-66).
__global__ void clear_pad_kernel(uint64_t* w, size_t rows, size_t kw, size_t cols) {
  for (size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (size_t)gridDim.x * blockDim.x)
    for (size_t i = cols / 64; i < kw; ++i) {
      const size_t lo = i * 64;
      w[r * kw + i] &= cols > lo ? (cols - lo >= 64 ? ~0ull : ((1ull << (cols - lo)) - 1ull)) : 0ull;
    }
}
static void clear_pad_bits(uint64_t* w, size_t rows, size_t kw, size_t cols, cudaStream_t st) {
  clear_pad_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(w, rows, kw, cols);
  BT_CUDA(cudaGetLastError());
}
static void rand_floats(float* x, size_t n, uint64_t seed, cudaStream_t st) {
  rand_floats_kernel<<<148 * 8, 256, 0, st>>>(x, n, seed);
  BT_CUDA(cudaGetLastError());
}

template <class F>
static void time_reps(int reps, int warmup, cudaStream_t st, F&& fn, double* median_ns, double* min_ns) {
  require(reps >= 1, BTNN_INVALID_INPUT, "bench: need at least one repetition");
  for (int i = 0; i < warmup; ++i) fn();
  cudaEvent_t a, b;
  BT_CUDA(cudaEventCreate(&a));
  BT_CUDA(cudaEventCreate(&b));
  std::vector<double> ns(reps);
  for (int r = 0; r < reps; ++r) {
    BT_CUDA(cudaEventRecord(a, st));
    fn();
    BT_CUDA(cudaEventRecord(b, st));
    BT_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    BT_CUDA(cudaEventElapsedTime(&ms, a, b));
    ns[r] = ms * 1e6;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  std::sort(ns.begin(), ns.end());
  *median_ns = reps % 2 ? ns[reps / 2] : 0.5 * (ns[reps / 2 - 1] + ns[reps / 2]);
  *min_ns = ns.front();
}

// Average device time of `reps` launches of fn issued back to back between two events.
template <class F>
static double time_stream(int reps, int warmup, cudaStream_t st, F&& fn) {
  for (int i = 0; i < warmup; ++i) fn();
  cudaEvent_t a, b;
  BT_CUDA(cudaEventCreate(&a));
  BT_CUDA(cudaEventCreate(&b));
  BT_CUDA(cudaEventRecord(a, st));
  for (int i = 0; i < reps; ++i) fn();
  BT_CUDA(cudaEventRecord(b, st));
  BT_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  BT_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms * 1e6 / reps;
}

// Average device time per call of `reps` calls captured back to back in one CUDA graph and
// replayed (after `warmup` direct calls and one untimed replay).
template <class F>
static double time_graph(int reps, int warmup, cudaStream_t st, F&& fn) {
  for (int i = 0; i < warmup; ++i) fn();
  BT_CUDA(cudaStreamSynchronize(st));
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  BT_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < reps; ++i) fn();
  BT_CUDA(cudaStreamEndCapture(st, &graph));
  BT_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  BT_CUDA(cudaGraphLaunch(exec, st));
  cudaEvent_t a, b;
  BT_CUDA(cudaEventCreate(&a));
  BT_CUDA(cudaEventCreate(&b));
  BT_CUDA(cudaEventRecord(a, st));
  BT_CUDA(cudaGraphLaunch(exec, st));
  BT_CUDA(cudaEventRecord(b, st));
  BT_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  BT_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  return ms * 1e6 / reps;
}

}  // namespace btnn_gpu

using namespace btnn_gpu;

// Self-test of bnmath.cuh: the bn division with the per-channel reciprocal against
// __ddiv_rn (and hence IEEE a/b) on caller-supplied operands.
__global__ void div_selftest_kernel(const double* a, const double* b, size_t n, double* fast, double* ref) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double y = bn_recip(b[i]);
    fast[i] = div_rn_with_recip(a[i], b[i], y);
    ref[i] = __ddiv_rn(a[i], b[i]);
  }
}

extern "C" {

int btnn_cuda_selftest_div(const double* a, const double* b, size_t n, double* fast, double* ref) {
  return guard([&] {
    cudaStream_t st = 0;
    DevBuf da = upload(a, n, st), db = upload(b, n, st), df(n * 8), dr(n * 8);
    div_selftest_kernel<<<1184, 256, 0, st>>>(da.get<double>(), db.get<double>(), n, df.get<double>(), dr.get<double>());
    BT_CUDA(cudaGetLastError());
    BT_CUDA(cudaMemcpyAsync(fast, df.get(), n * 8, cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaMemcpyAsync(ref, dr.get(), n * 8, cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaStreamSynchronize(st));
  });
}


static int bench_bmm_impl(size_t n, int bin, int fsb, int reps, int warmup, double* median_ns, double* min_ns,
                          char* engine, size_t engine_len, const btnn_bench_readback* rb) {
  return guard([&] {
    require(n > 0, BTNN_INVALID_INPUT, "bench_bmm: zero size");
    int dev = 0;
    BT_CUDA(cudaGetDevice(&dev));
    cudaStream_t st;
    BT_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const size_t kw = ru(n, 128) / 64;
    DevBuf a(n * kw * 8), b(n * kw * 8), out_i(bin ? 0 : n * n * 4), out_b(bin ? n * kw * 8 : 0);
    ConvShape s{};
    s.P = s.Q = s.H = s.W = 1;
    s.KH = s.KW = s.stride = 1;
    s.N = (int)n;
    s.in_rps = s.out_rps = (int)n;
    s.cw = (int)kw;
    s.C = (int)n;
    s.O = (int)n;
    s.f_rps = (int)n;
    s.cwo = (int)kw;
    // random packed words with the pad bits of every row / column cleared
    rand_words(a.get<uint64_t>(), n * kw, 1, st);
    rand_words(b.get<uint64_t>(), n * kw, 2, st);
    if (n % 128) {
      clear_pad_bits(a.get<uint64_t>(), n, kw, n, st);
      clear_pad_bits(b.get<uint64_t>(), n, kw, n, st);
    }
    Epi e;
    if (bin) {
      e.mode = EPI_BITS;
      e.out_bits = out_b.get<uint64_t>();
    } else {
      e.mode = EPI_I32;
      e.out_i32 = out_i.get<int32_t>();
    }
    // fsb layout (the reference's "fsb" rows, bench.hpp:140-156): the call's operands are FSB
    // tiles (8 x 128), converted to RowPacked / ColPacked on the device inside every timed
    // call, and a bit result converted back to FSB rows
    constexpr size_t kBh = 8, kBw = 128;
    DevBuf af, bf, tmp_a, tmp_b, of;
    if (fsb) {
      af.alloc(mat_words(n, n, BTNN_FSB_ROW, kBh, kBw) * 8);
      bf.alloc(mat_words(n, n, BTNN_FSB_COL, kBh, kBw) * 8);
      tmp_a.alloc(a.bytes());
      tmp_b.alloc(b.bytes());
      launch_convert_matrix(n, n, BTNN_ROW_PACKED, 0, 0, a.get<uint64_t>(), BTNN_FSB_ROW, kBh, kBw, af.get<uint64_t>(), st);
      launch_convert_matrix(n, n, BTNN_COL_PACKED, 0, 0, b.get<uint64_t>(), BTNN_FSB_COL, kBh, kBw, bf.get<uint64_t>(), st);
      if (bin) of.alloc(mat_words(n, n, BTNN_FSB_ROW, kBh, kBw) * 8);
    }
    const uint64_t* opa = fsb ? tmp_a.get<uint64_t>() : a.get<uint64_t>();
    const uint64_t* opb = fsb ? tmp_b.get<uint64_t>() : b.get<uint64_t>();
    auto to_plain = [&] {
      if (!fsb) return;
      launch_convert_matrix(n, n, BTNN_FSB_ROW, kBh, kBw, af.get<uint64_t>(), BTNN_ROW_PACKED, 0, 0, tmp_a.get<uint64_t>(), st);
      launch_convert_matrix(n, n, BTNN_FSB_COL, kBh, kBw, bf.get<uint64_t>(), BTNN_COL_PACKED, 0, 0, tmp_b.get<uint64_t>(), st);
    };
    auto to_fsb_out = [&] {
      if (fsb && bin)
        launch_convert_matrix(n, n, BTNN_ROW_PACKED, 0, 0, out_b.get<uint64_t>(), BTNN_FSB_ROW, kBh, kBw, of.get<uint64_t>(), st);
    };
    TcFilter tcf;
    const bool packed = engine_override() != BTNN_ENGINE_POPC;
    const bool tc = !packed && engine_override() != BTNN_ENGINE_POPC && tc_supported(s, e);
    if (tc) tc_prepare_filter(s, b.get<uint64_t>(), tcf, st);
    const char* used = "popc";
    // the whole bmm_pm1 / bmm_pm1_bin call from packed operands: one kernel that expands both
    // operands on chip (bmm_tc.cu, whole-K or K-pipelined)
    auto step = [&] {
      to_plain();
      if (packed) {
        used = launch_bmm_packed((int)n, (int)n, (int)n, opa, opb, e, st);
      } else {
        if (tc) tc_prepare_filter(s, opb, tcf, st);
        used = launch_bgemm(s, opa, opb, e, st, EngineHint::Auto, &tcf);
      }
      to_fsb_out();
    };
    BT_CUDA(cudaStreamSynchronize(st));
    time_reps(reps, warmup, st, step, median_ns, min_ns);
    // Back-to-back averages (the host launch cost overlapped, as a GEMM inside a plan or a
    // stream of calls sees it; the per-call median above also pays each call's host launch):
    // the GEMM alone with B prepared, and the whole call.
    if (rb && rb->kernel_ns)
      *rb->kernel_ns = time_graph(reps, warmup, st, [&] {
        if (packed) launch_bmm_packed((int)n, (int)n, (int)n, opa, opb, e, st);
        else launch_bgemm(s, opa, opb, e, st, EngineHint::Auto, &tcf);
      });
    if (rb && rb->stream_ns) *rb->stream_ns = time_stream(reps, warmup, st, step);
    if (rb && rb->graph_ns) *rb->graph_ns = time_graph(reps, warmup, st, step);
    if (rb) {
      BT_CUDA(cudaStreamSynchronize(st));
      if (rb->a_words) BT_CUDA(cudaMemcpy(rb->a_words, a.get(), a.bytes(), cudaMemcpyDeviceToHost));
      if (rb->b_words) BT_CUDA(cudaMemcpy(rb->b_words, b.get(), b.bytes(), cudaMemcpyDeviceToHost));
      if (rb->out) BT_CUDA(cudaMemcpy(rb->out, bin ? out_b.get() : out_i.get(), bin ? out_b.bytes() : out_i.bytes(),
                                      cudaMemcpyDeviceToHost));
    }
    if (engine && engine_len) {
      std::snprintf(engine, engine_len, "%s", used);
    }
    cudaStreamDestroy(st);
  });
}

static int bench_bconv_impl(size_t input_hw, size_t batch, size_t c, size_t o, size_t k, int bin, int fsb, int reps,
                            int warmup, double* median_ns, double* min_ns, char* engine, size_t engine_len,
                            const btnn_bench_readback* rb) {
  return guard([&] {
    require(input_hw && batch && c && o && k, BTNN_INVALID_INPUT, "bench_bconv: zero size");
    cudaStream_t st;
    BT_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const size_t H = input_hw, pad = k / 2;
    const size_t P = (H + 2 * pad - k) + 1;
    const size_t np = act_npad(batch, 0, 0), cp = act_cpad(c, 0, 0), op = act_cpad(o, 0, 0);
    DevBuf in(H * H * np * cp / 8), filt(k * k * filt_opad(o, 0, 0) * cp / 8), x, flag(4);
    DevBuf out_b(bin ? P * P * np * op / 8 : 0), out_i(bin ? 0 : P * P * batch * o * 4), lo, hi;
    ConvShape s{};
    s.P = s.Q = (int)P;
    s.H = s.W = (int)H;
    s.KH = s.KW = (int)k;
    s.stride = 1;
    s.pad = (int)pad;
    s.N = (int)batch;
    s.in_rps = s.out_rps = (int)np;
    s.cw = (int)(cp / 64);
    s.C = (int)c;
    s.O = (int)o;
    s.f_rps = (int)filt_opad(o, 0, 0);
    s.cwo = (int)(op / 64);
    // filter words: random, pad bits cleared by packing random floats per plane row
    {
      DevBuf fw(k * k * filt_opad(o, 0, 0) * c * 4);
      rand_floats(fw.get<float>(), k * k * filt_opad(o, 0, 0) * c, 7, st);
      BT_CUDA(cudaMemsetAsync(filt.get(), 0, filt.bytes(), st));
      launch_pack_rows(fw.get<float>(), k * k * filt_opad(o, 0, 0), c, cp / 32, filt.get<uint32_t>(), flag.get<int>(), st);
      BT_CUDA(cudaStreamSynchronize(st));
    }
    Epi e;
    if (bin) {
      BT_CUDA(cudaMemsetAsync(in.get(), 0, in.bytes(), st));
      DevBuf fx(batch * H * H * c * 4);
      rand_floats(fx.get<float>(), batch * H * H * c, 3, st);
      launch_pack_nhwc(fx.get<float>(), (int)batch, (int)H, (int)H, (int)c, (int)np, (int)cp, in.get<uint32_t>(),
                       flag.get<int>(), st);
      BT_CUDA(cudaStreamSynchronize(st));
      std::vector<long long> l(o, 0), h(o, 1LL << 40);  // sign rule: v >= 0 (tau = 0, Geq)
      lo = upload(l.data(), o, st);
      hi = upload(h.data(), o, st);
      e.mode = EPI_BITS;
      e.out_bits = out_b.get<uint64_t>();
      e.thr_lo = lo.get<long long>();
      e.thr_hi = hi.get<long long>();
    } else {
      x.alloc(batch * H * H * c * 4);
      rand_floats(x.get<float>(), batch * H * H * c, 3, st);
      e.mode = EPI_I32;
      e.out_i32 = out_i.get<int32_t>();
    }
    s.halo_ok = s.C <= 128;
    TcFilter tcf;
    if (engine_override() != BTNN_ENGINE_POPC && tc_supported(s, e)) tc_prepare_filter(s, filt.get<uint64_t>(), tcf, st);
    const char* used = "popc";
    // fsb layout (bench.hpp:230-245): the call's input is the tiled activation tensor
    // (convert_activations, 8 x 128 tiles), converted to plain HWNC on the device every call;
    // a bit output goes back to tiles. (The filter is a layer constant: converted and expanded
    // once, as in the plain rows.)
    constexpr size_t kBh = 8, kBw = 128;
    DevBuf in_t, out_t;
    if (fsb) {
      in_t.alloc(act_words(H, H, batch, c, 1, kBh, kBw) * 8);
      if (bin) {
        launch_convert_act(H, H, batch, c, 0, 0, 0, in.get<uint64_t>(), 1, kBh, kBw, in_t.get<uint64_t>(), st);
        out_t.alloc(act_words(P, P, batch, o, 1, kBh, kBw) * 8);
      }
    }
    auto step = [&] {
      if (!bin) {
        BT_CUDA(cudaMemsetAsync(in.get(), 0, in.bytes(), st));
        launch_pack_nhwc(x.get<float>(), (int)batch, (int)H, (int)H, (int)c, (int)np, (int)cp, in.get<uint32_t>(),
                         flag.get<int>(), st);
        if (fsb) {  // binarize into tiles (pack_nhwc then convert), then back to plain for the GEMM
          launch_convert_act(H, H, batch, c, 0, 0, 0, in.get<uint64_t>(), 1, kBh, kBw, in_t.get<uint64_t>(), st);
          launch_convert_act(H, H, batch, c, 1, kBh, kBw, in_t.get<uint64_t>(), 0, 0, 0, in.get<uint64_t>(), st);
        }
      } else if (fsb) {
        launch_convert_act(H, H, batch, c, 1, kBh, kBw, in_t.get<uint64_t>(), 0, 0, 0, in.get<uint64_t>(), st);
      }
      used = launch_bgemm(s, in.get<uint64_t>(), filt.get<uint64_t>(), e, st, EngineHint::Auto, &tcf);
      if (fsb && bin)
        launch_convert_act(P, P, batch, o, 0, 0, 0, out_b.get<uint64_t>(), 1, kBh, kBw, out_t.get<uint64_t>(), st);
    };
    BT_CUDA(cudaStreamSynchronize(st));
    time_reps(reps, warmup, st, step, median_ns, min_ns);
    if (rb) {
      BT_CUDA(cudaStreamSynchronize(st));
      if (rb->a_words) BT_CUDA(cudaMemcpy(rb->a_words, in.get(), in.bytes(), cudaMemcpyDeviceToHost));
      if (rb->b_words) BT_CUDA(cudaMemcpy(rb->b_words, filt.get(), filt.bytes(), cudaMemcpyDeviceToHost));
      if (rb->out) BT_CUDA(cudaMemcpy(rb->out, bin ? out_b.get() : out_i.get(), bin ? out_b.bytes() : out_i.bytes(),
                                      cudaMemcpyDeviceToHost));
    }
    if (engine && engine_len) std::snprintf(engine, engine_len, "%s", used);
    cudaStreamDestroy(st);
  });
}

int btnn_cuda_bench_bmm(size_t n, int bin, int reps, int warmup, double* median_ns, double* min_ns, char* engine,
                        size_t engine_len, const btnn_bench_readback* rb) {
  return bench_bmm_impl(n, bin, 0, reps, warmup, median_ns, min_ns, engine, engine_len, rb);
}
int btnn_cuda_bench_bmm_fsb(size_t n, int bin, int reps, int warmup, double* median_ns, double* min_ns, char* engine,
                            size_t engine_len, const btnn_bench_readback* rb) {
  return bench_bmm_impl(n, bin, 1, reps, warmup, median_ns, min_ns, engine, engine_len, rb);
}
int btnn_cuda_bench_bconv(size_t input_hw, size_t batch, size_t c, size_t o, size_t k, int bin, int reps, int warmup,
                          double* median_ns, double* min_ns, char* engine, size_t engine_len,
                          const btnn_bench_readback* rb) {
  return bench_bconv_impl(input_hw, batch, c, o, k, bin, 0, reps, warmup, median_ns, min_ns, engine, engine_len, rb);
}
int btnn_cuda_bench_bconv_fsb(size_t input_hw, size_t batch, size_t c, size_t o, size_t k, int bin, int reps,
                              int warmup, double* median_ns, double* min_ns, char* engine, size_t engine_len,
                              const btnn_bench_readback* rb) {
  return bench_bconv_impl(input_hw, batch, c, o, k, bin, 1, reps, warmup, median_ns, min_ns, engine, engine_len, rb);
}

}  // extern "C"
