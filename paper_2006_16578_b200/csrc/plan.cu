// plan.cu — the model driver: run_inference (inference.hpp:67-186) as a device plan.
//
// A plan holds, per device ("shard"), the weights converted once to the device formats,
// the activation / tap / FC buffers sized for the shard's max batch, and a CUDA graph
// per (batch, pointers) that replays the whole layer sequence. The batch is split into
// contiguous per-device chunks; no sample couples to another (bn uses frozen statistics,
// layer_math.hpp:32-34), so the shards need no collective and the result is identical
// to a single-device run.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "api_internal.cuh"
#include "common.cuh"
#include "kernels.cuh"
#include "layout.cuh"

namespace btnn_gpu {

constexpr size_t kMaxChunks = 16;  // run_shard_host input pipelining (chunk_schedule)

struct LayerDev {
  btnn_layer_spec spec{};
  DevBuf filt;          // plain KKOC filter / ColPacked fc matrix
  TcFilter tc;          // tensor-core operand (bit conv / fc when covered)
  DevBuf wpm1;          // first conv (o,r,s,c) floats
  DevBuf wbits;         // first conv per-o sign bits
  DevBuf wblk;          // first conv tensor-core weight blocks (kernels_first_tc.cu)
  DevBuf fix_list, fix_count;  // first conv windows left to the sequential kernel
  DevBuf thr_lo, thr_hi;
  DevBuf bn;            // mean | s | gamma | beta
  bool has_thr = false, has_bn = false;
  DevBuf tap;           // residual_out, PQNO f64 sized for max batch
  DevBuf tap_half;      // residual_out pre-averaged 2x2 for a halving consumer (P/2, Q/2, N, O)
  DevBuf split_ws;      // fc layers: int32 batch x units workspace for split-K (tensor-core engine)
  bool feeds_full = false, feeds_half = false;  // consumers read the tap as is / halved
  bool wrote_half = false;                      // last enqueue stored tap_half instead of tap
  bool halo_ok = false;                         // conv may run the halo-mode kernel (filter layout)
  bool pool_fused = false;                      // or_pool layer folded into the previous conv's epilogue
  std::string engine = "-";
  // Measured geometry choice (tune_shard): the candidates of the layer's shape, their
  // measured ms at the shard's max batch, and the pick.
  TcChoice choice;
  std::vector<TcChoice> cands;
  std::vector<std::string> cand_names;
  std::vector<double> cand_ms;
};

struct Shard {
  int device = 0;
  cudaStream_t stream = nullptr;
  size_t max_batch = 0;
  std::vector<LayerDev> layers;
  DevBuf x, act[2], fc[2], logits, labels, flag;
  DevBuf rowmax;        // per input row (n, h): largest |x| (tensor-core first conv)
  size_t act_words = 0, fc_words = 0;
  // Captured graphs per (batch, pointers, engine override). Host-side choices are frozen in
  // each graph, including which layers stored a pre-averaged tap (restored on replay so
  // plan_tap_dims / plan_read_tap describe the graph that ran last).
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    std::vector<char> wrote_half;
  };
  std::map<std::tuple<size_t, const void*, const void*, const void*, int>, Graph> graphs;
  std::vector<cudaEvent_t> events;  // breakdown
  cudaStream_t copy_stream = nullptr;    // host->device input chunks (run_shard_host)
  cudaStream_t d2h_stream = nullptr;     // device->host results per chunk (pinned outputs)
  std::vector<cudaEvent_t> in_ready;     // per chunk: input resident
  std::vector<cudaEvent_t> out_ready;    // per chunk: logits / labels computed
  // e2e chunk model (calibrate_e2e, measured once per shard on its first host run): host ->
  // device copy time per image (us) and the graph's time t(b) = t0 + b * s (us) for b images
  bool e2e_cal = false;
  bool e2e_cal_pinned = false;  // the input buffer kind the model was measured on
  double e2e_c = 0.0, e2e_t0 = 0.0, e2e_s = 0.0;
  size_t launches = 0;
  int tune_pass = -1;  // >= 0 while tune_shard runs candidate pass k of every layer
  ~Shard() {
    if (device >= 0) cudaSetDevice(device);
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    for (auto ev : events) cudaEventDestroy(ev);
    for (auto ev : in_ready) cudaEventDestroy(ev);
    for (auto ev : out_ready) cudaEventDestroy(ev);
    if (d2h_stream) cudaStreamDestroy(d2h_stream);
    if (stream) cudaStreamDestroy(stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
  }
};

}  // namespace btnn_gpu

struct btnn_plan {
  std::string name;
  size_t in_h = 0, in_w = 0, in_c = 0, classes = 0;
  std::vector<btnn_layer_spec> specs;
  std::vector<std::unique_ptr<btnn_gpu::Shard>> shards;
  bool breakdown = false;
  std::vector<double> layer_ms;
};

namespace btnn_gpu {

static ConvShape conv_shape(const btnn_layer_spec& l, size_t batch, bool halo_ok) {
  ConvShape s{};
  s.halo_ok = halo_ok && l.in_channels <= 128;
  s.P = (int)l.out_h; s.Q = (int)l.out_w;
  s.H = (int)l.in_h; s.W = (int)l.in_w;
  s.KH = (int)l.kh; s.KW = (int)l.kw; s.stride = (int)l.stride; s.pad = (int)l.pad;
  s.N = (int)batch;
  s.in_rps = s.out_rps = (int)act_npad(batch, 0, 0);
  s.cw = (int)(act_cpad(l.in_channels, 0, 0) / 64);
  s.C = (int)l.in_channels;
  s.O = (int)l.out_channels;
  s.f_rps = (int)filt_opad(l.out_channels, 0, 0);
  s.cwo = (int)(act_cpad(l.out_channels, 0, 0) / 64);
  return s;
}

static ConvShape fc_shape(const btnn_layer_spec& l, size_t batch) {
  ConvShape s{};
  s.P = s.Q = s.H = s.W = 1;
  s.KH = s.KW = s.stride = 1;
  s.pad = 0;
  s.N = (int)batch;
  s.in_rps = s.out_rps = (int)batch;
  s.cw = (int)(ru(l.in_channels, 128) / 64);
  s.C = (int)l.in_channels;
  s.O = (int)l.units;
  s.f_rps = (int)l.units;
  s.cwo = (int)(ru(l.units, 128) / 64);
  return s;
}

// Validation of the (model, store) pair; run_inference checks the layer count
// (inference.hpp:69-70), the rest guards the raw C ABI against short buffers.
static void check_plan_inputs(const btnn_model_spec* m, const btnn_weight_store* ws) {
  require(m && ws && m->layers && ws->layers, BTNN_INVALID_INPUT, "plan: null model or weights");
  require(ws->n_layers == m->n_layers, BTNN_INVALID_INPUT, "run_inference: weight store does not match model");
  require(m->n_layers > 0, BTNN_VALIDATION_ERROR, "model: no layers");
  if (ws->tiled)
    require(ws->bh * ws->bw != 0 && (ws->bh * ws->bw) % 64 == 0 && ws->bw % 64 == 0, BTNN_UNSUPPORTED_SHAPE,
            "plan: unsupported tile geometry");
  for (size_t i = 0; i < m->n_layers; ++i) {
    const btnn_layer_spec& l = m->layers[i];
    const btnn_layer_weights& w = ws->layers[i];
    const std::string tag = "layer " + std::to_string(i);
    require(w.kind == l.kind, BTNN_VALIDATION_ERROR, tag + ": weight record kind does not match model");
    const bool conv = l.kind == BTNN_FIRST_CONV_BWN || l.kind == BTNN_BIT_CONV;
    const bool fc = l.kind == BTNN_BIT_FC || l.kind == BTNN_LAST_FC;
    if (l.kind == BTNN_FIRST_CONV_BWN)
      require(w.conv_pm1 && w.conv_pm1_n == l.kh * l.kw * l.out_channels * l.in_channels, BTNN_VALIDATION_ERROR,
              tag + ": first conv weights missing");
    if (l.kind == BTNN_BIT_CONV)
      require(w.filter_words &&
                  w.filter_n_words == filt_words(l.kh, l.kw, l.out_channels, l.in_channels, ws->tiled, ws->bh, ws->bw),
              BTNN_VALIDATION_ERROR, tag + ": filter word count does not match");
    if (fc)
      require(w.fc_words && w.fc_n_words == mat_words(l.in_channels, l.units, ws->tiled ? BTNN_FSB_COL : BTNN_COL_PACKED,
                                                      ws->bh, ws->bw),
              BTNN_VALIDATION_ERROR, tag + ": fc word count does not match");
    const size_t outc = conv ? l.out_channels : (fc ? l.units : 0);
    const bool bn_route = l.kind == BTNN_FIRST_CONV_BWN || l.kind == BTNN_LAST_FC || l.residual_in || l.residual_out;
    if (l.kind != BTNN_OR_POOL) {
      if (bn_route || w.n_thresholds == 0) {
        require(w.has_bn && w.bn.channels == outc, BTNN_VALIDATION_ERROR, tag + ": bn parameters missing");
        check_bn(w.bn);
      } else {
        require(w.n_thresholds == outc && w.tau && w.tkind, BTNN_VALIDATION_ERROR, tag + ": threshold count does not match");
      }
    }
    if (l.residual_in)
      require(l.shortcut_from >= 0 && (size_t)l.shortcut_from < i && m->layers[l.shortcut_from].residual_out,
              BTNN_VALIDATION_ERROR, tag + ": bad shortcut source");
  }
}

static void build_shard(Shard& sh, const btnn_model_spec* m, const btnn_weight_store* ws) {
  BT_CUDA(cudaSetDevice(sh.device));
  BT_CUDA(cudaStreamCreateWithFlags(&sh.stream, cudaStreamNonBlocking));
  BT_CUDA(cudaStreamCreateWithFlags(&sh.copy_stream, cudaStreamNonBlocking));
  BT_CUDA(cudaStreamCreateWithFlags(&sh.d2h_stream, cudaStreamNonBlocking));
  cudaStream_t st = sh.stream;
  const size_t B = sh.max_batch;
  sh.layers.resize(m->n_layers);
  size_t act_max = 1, fc_max = 1;
  for (size_t i = 0; i < m->n_layers; ++i) {
    const btnn_layer_spec& l = m->layers[i];
    const btnn_layer_weights& w = ws->layers[i];
    LayerDev& L = sh.layers[i];
    L.spec = l;
    if (l.kind == BTNN_FIRST_CONV_BWN || l.kind == BTNN_BIT_CONV || l.kind == BTNN_OR_POOL)
      act_max = std::max(act_max, act_words(l.out_h, l.out_w, B, l.out_channels, 0, 0, 0));
    if (l.kind == BTNN_BIT_FC || l.kind == BTNN_LAST_FC) {
      fc_max = std::max(fc_max, B * ru(l.in_channels, 128) / 64);
      fc_max = std::max(fc_max, B * ru(l.units, 128) / 64);
      L.split_ws.alloc(B * l.units * sizeof(int32_t));
    }
    if (l.kind == BTNN_FIRST_CONV_BWN) {
      L.wpm1 = upload(w.conv_pm1, w.conv_pm1_n, st);
      const int K = (int)(l.kh * l.kw * l.in_channels);
      L.wbits.alloc(first_conv_signbits_words((int)l.out_channels, K) * 4);
      launch_first_conv_signbits(L.wpm1.get<float>(), (int)l.out_channels, K, L.wbits.get<uint32_t>(), st);
      L.wblk.alloc(first_conv_tc_weight_bytes((int)l.kh, (int)l.kw, (int)l.out_channels, (int)l.stride));
      launch_first_conv_tc_weights(L.wpm1.get<float>(), (int)l.out_channels, (int)l.kh, (int)l.kw,
                                   (int)l.in_channels, (int)l.stride, L.wblk.get<int8_t>(), st);
      L.fix_list.alloc(B * l.out_h * l.out_w * sizeof(int));
      L.fix_count.alloc(sizeof(int));
      sh.rowmax.alloc(B * l.in_h * sizeof(uint32_t));
    } else if (l.kind == BTNN_BIT_CONV) {
      DevBuf raw = upload(w.filter_words, w.filter_n_words, st);
      if (!ws->tiled) {
        L.filt = std::move(raw);
      } else {
        L.filt.alloc(filt_words(l.kh, l.kw, l.out_channels, l.in_channels, 0, 0, 0) * 8);
        launch_convert_act(l.kh, l.kw, l.out_channels, l.in_channels, 1, ws->bh, ws->bw, raw.get<uint64_t>(), 0, 0, 0,
                           L.filt.get<uint64_t>(), st);
        BT_CUDA(cudaStreamSynchronize(st));
      }
      // Halo-mode kernels for every conv except a tap producer whose consumer halves it
      // (that one writes the pre-averaged tap in 2x2-blocked row order, TMEM-A path).
      L.halo_ok = true;
      if (l.residual_out)
        for (size_t j = i + 1; j < m->n_layers; ++j)
          if (m->layers[j].residual_in && m->layers[j].shortcut_from == (int)i && m->layers[j].out_h != l.out_h)
            L.halo_ok = false;
      tc_prepare_filter(conv_shape(l, B, L.halo_ok), L.filt.get<uint64_t>(), L.tc, st);
    } else if (l.kind == BTNN_BIT_FC || l.kind == BTNN_LAST_FC) {
      DevBuf raw = upload(w.fc_words, w.fc_n_words, st);
      if (!ws->tiled) {
        L.filt = std::move(raw);
      } else {
        L.filt.alloc(mat_words(l.in_channels, l.units, BTNN_COL_PACKED, 0, 0) * 8);
        launch_convert_matrix(l.in_channels, l.units, BTNN_FSB_COL, ws->bh, ws->bw, raw.get<uint64_t>(),
                              BTNN_COL_PACKED, 0, 0, L.filt.get<uint64_t>(), st);
        BT_CUDA(cudaStreamSynchronize(st));
      }
      tc_prepare_filter(fc_shape(l, B), L.filt.get<uint64_t>(), L.tc, st);
    }
    if (l.kind != BTNN_OR_POOL) {
      if (w.n_thresholds && !(l.kind == BTNN_LAST_FC || l.kind == BTNN_FIRST_CONV_BWN || l.residual_in || l.residual_out)) {
        std::vector<long long> lo, hi;
        thresholds_to_int(w.tau, w.tkind, w.n_thresholds, lo, hi);
        L.thr_lo = upload(lo.data(), lo.size(), st);
        L.thr_hi = upload(hi.data(), hi.size(), st);
        L.has_thr = true;
      } else {
        L.bn = upload_bn(w.bn, st);
        L.has_bn = true;
      }
    }
    if (l.residual_out) {
      // Who reads this tap: adapt_shortcut halves it when the consumer's grid is smaller
      // (inference.hpp:46). A producer whose every consumer halves may store only the
      // pre-averaged tap (kernels_tc.cu, blocked row order); the full one stays allocated
      // for engines or grids that cannot.
      for (size_t j = i + 1; j < m->n_layers; ++j) {
        const btnn_layer_spec& c = m->layers[j];
        if (!c.residual_in || c.shortcut_from != (int)i) continue;
        (c.out_h != l.out_h ? L.feeds_half : L.feeds_full) = true;
      }
      L.tap.alloc(l.out_h * l.out_w * B * l.out_channels * sizeof(double));
      if (L.feeds_half && !L.feeds_full && l.kind == BTNN_BIT_CONV && l.out_h % 2 == 0 && l.out_w % 2 == 0)
        L.tap_half.alloc((l.out_h / 2) * (l.out_w / 2) * B * l.out_channels * sizeof(double));
    }
    BT_CUDA(cudaStreamSynchronize(st));  // host staging vectors die here
  }
  sh.act_words = act_max;
  sh.fc_words = fc_max;
  for (auto& a : sh.act) a.alloc(act_max * 8);
  for (auto& f : sh.fc) f.alloc(fc_max * 8);
  sh.x.alloc(B * m->in_h * m->in_w * m->in_c * sizeof(float));
  sh.logits.alloc(B * m->classes * sizeof(double));
  sh.labels.alloc(B * sizeof(int32_t));
  sh.flag.alloc(sizeof(int));
  sh.events.resize(m->n_layers + 1);
  for (auto& ev : sh.events) BT_CUDA(cudaEventCreate(&ev));
  sh.in_ready.resize(kMaxChunks);
  for (auto& ev : sh.in_ready) BT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  sh.out_ready.resize(kMaxChunks);
  for (auto& ev : sh.out_ready) BT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  BT_CUDA(cudaStreamSynchronize(st));
}

// Window of an or_pool layer i + 1 that the conv layer i can fold into its epilogue
// (non-overlapping windows that tile the conv's grid exactly: each output site feeds one
// pooled site), else 0.
static int fusable_pool(const Shard& sh, size_t i) {
  if (i + 1 >= sh.layers.size()) return 0;
  const btnn_layer_spec& l = sh.layers[i].spec;
  const btnn_layer_spec& nx = sh.layers[i + 1].spec;
  if (nx.kind != BTNN_OR_POOL || nx.window != nx.pool_stride || nx.window < 2) return 0;
  if (l.out_h % nx.window || l.out_w % nx.window || nx.out_h * nx.window != l.out_h || nx.out_w * nx.window != l.out_w)
    return 0;
  return (int)nx.window;
}

// Enqueues the whole layer sequence for `batch` samples of x (device) on the shard's
// stream. Returns the number of kernels launched.
static size_t enqueue_forward(btnn_plan* plan, Shard& sh, const float* d_x, size_t batch, double* d_logits,
                              int32_t* d_labels, bool timed) {
  cudaStream_t st = sh.stream;
  size_t launches = 0;
  // (sh.flag is cleared by the host-side caller, so one flag covers all chunks of a run.)
  // The tensor-core first conv needs per-row input maxima; that input pass doubles as the
  // non-finite check (inference.hpp:69-75).
  FirstConvArgs fa{};
  bool first_tc = false;
  if (!sh.layers.empty() && sh.layers[0].spec.kind == BTNN_FIRST_CONV_BWN) {
    const btnn_layer_spec& l = sh.layers[0].spec;
    fa.N = (int)batch; fa.H = (int)l.in_h; fa.W = (int)l.in_w; fa.C = (int)l.in_channels; fa.O = (int)l.out_channels;
    fa.KH = (int)l.kh; fa.KW = (int)l.kw; fa.stride = (int)l.stride; fa.pad = (int)l.pad;
    fa.P = (int)l.out_h; fa.Q = (int)l.out_w;
    fa.tap = l.residual_out ? sh.layers[0].tap.get<double>() : nullptr;  // (sizes the tap stage)
    first_tc = engine_override() != BTNN_ENGINE_POPC && first_conv_tc_supported(fa);
  }
  if (timed) BT_CUDA(cudaEventRecord(sh.events[0], st));  // layer 0's time includes the input pass
  // the first conv's own builders check the input and take the tile maxima where they cover it
  const bool fused_in = first_tc && first_conv_fused_input(fa);
  if (fused_in) {
  } else if (first_tc) {
    launch_input_rows(d_x, batch * plan->in_h, (int)(plan->in_w * plan->in_c), sh.flag.get<int>(),
                      sh.rowmax.get<uint32_t>(), st);
    ++launches;
  } else if ((sh.layers[0].spec.kind != BTNN_BIT_FC && sh.layers[0].spec.kind != BTNN_LAST_FC) ||
             sh.layers[0].spec.in_channels != plan->in_h * plan->in_w * plan->in_c) {
    // (an FC-first model's pack_rows pass checks every input value itself)
    launch_check_finite(d_x, batch * plan->in_h * plan->in_w * plan->in_c, sh.flag.get<int>(), st);
    ++launches;
  }
  const size_t np = act_npad(batch, 0, 0);
  bool labels_done = false;  // the last layer's kernel wrote the argmax labels
  int cur = 0;              // act buffer holding the current activations
  int fcur = 0;             // fc buffer holding the current fc activations
  bool in_fc = false;
  size_t H = plan->in_h, W = plan->in_w, C = plan->in_c;
  for (size_t i = 0; i < sh.layers.size(); ++i) {
    LayerDev& L = sh.layers[i];
    const btnn_layer_spec& l = L.spec;
    if (timed && i > 0) BT_CUDA(cudaEventRecord(sh.events[i], st));
    if (l.kind == BTNN_FIRST_CONV_BWN) {
      uint64_t* out = sh.act[cur].get<uint64_t>();
      const int pool = first_tc ? fusable_pool(sh, i) : 0;
      if (i + 1 < sh.layers.size()) sh.layers[i + 1].pool_fused = pool != 0;
      // the tensor-core kernel writes every word of its packed output when N % 8 == 0; a fused
      // pool ORs into a zeroed pooled tensor
      if (pool)
        BT_CUDA(cudaMemsetAsync(out, 0, act_words(l.out_h / pool, l.out_w / pool, batch, l.out_channels, 0, 0, 0) * 8, st));
      else if (!(first_tc && np == batch))
        BT_CUDA(cudaMemsetAsync(out, 0, act_words(l.out_h, l.out_w, batch, l.out_channels, 0, 0, 0) * 8, st));
      FirstConvArgs a{};
      a.x = d_x;
      a.w_pm1 = L.wpm1.get<float>();
      a.N = (int)batch; a.H = (int)l.in_h; a.W = (int)l.in_w; a.C = (int)l.in_channels; a.O = (int)l.out_channels;
      a.KH = (int)l.kh; a.KW = (int)l.kw; a.stride = (int)l.stride; a.pad = (int)l.pad;
      a.P = (int)l.out_h; a.Q = (int)l.out_w;
      const size_t C4 = l.out_channels;
      a.bn_mean = L.bn.get<double>(); a.bn_s = a.bn_mean + C4; a.bn_gamma = a.bn_mean + 2 * C4; a.bn_beta = a.bn_mean + 3 * C4;
      a.bn_rcp = a.bn_mean + 4 * C4;
      a.tap = l.residual_out ? L.tap.get<double>() : nullptr;
      a.out_bits = out;
      a.wbits = L.wbits.get<uint32_t>();
      a.out_rps = (int)np;
      a.cwo = (int)(act_cpad(l.out_channels, 0, 0) / 64);
      a.pool = pool;
      if (first_tc) {
        launch_first_conv_tc(a, fused_in ? nullptr : sh.rowmax.get<uint32_t>(), L.wblk.get<int8_t>(), L.fix_count.get<int>(),
                             L.fix_list.get<int>(), st, sh.flag.get<int>());
        launches += 2;
        L.engine = pool ? "tc_i8_exact+pool" : "tc_i8_exact";
      } else {
        launch_first_conv(a, st);
        ++launches;
        L.engine = "fp64";
      }
      H = l.out_h; W = l.out_w; C = l.out_channels;
    } else if (l.kind == BTNN_BIT_CONV) {
      const uint64_t* in = sh.act[cur].get<uint64_t>();
      uint64_t* out = sh.act[cur ^ 1].get<uint64_t>();
      const ConvShape s = conv_shape(l, batch, L.halo_ok);
      Epi e;
      e.mode = EPI_BITS;
      e.out_bits = out;
      if (L.has_thr) {
        e.thr_lo = L.thr_lo.get<long long>();
        e.thr_hi = L.thr_hi.get<long long>();
      } else {
        const size_t O = l.out_channels;
        e.bn_mean = L.bn.get<double>(); e.bn_s = e.bn_mean + O; e.bn_gamma = e.bn_mean + 2 * O; e.bn_beta = e.bn_mean + 3 * O;
        e.bn_rcp = e.bn_mean + 4 * O;
      }
      if (l.residual_in) {
        const LayerDev& src = sh.layers[l.shortcut_from];
        e.rin_C = (int)src.spec.out_channels;
        if (src.wrote_half) {  // already averaged by the producer: read as is
          e.rin = src.tap_half.get<double>();
          e.rin_P = (int)l.out_h;
          e.rin_Q = (int)l.out_w;
          e.rin_halve = 0;
        } else {
          e.rin = src.tap.get<double>();
          e.rin_P = (int)src.spec.out_h;
          e.rin_Q = (int)src.spec.out_w;
          e.rin_halve = src.spec.out_h != l.out_h;  // adapt_shortcut's `halve` (inference.hpp:46)
        }
      }
      L.wrote_half = false;
      if (l.residual_out) {
        e.rout = L.tap.get<double>();
        if (L.tap_half.get()) {
          Epi eh = e;
          eh.rout = nullptr;
          eh.rout_half = L.tap_half.get<double>();
          if (will_use_tc(s, eh, EngineHint::Auto, &L.tc)) {
            e = eh;
            L.wrote_half = true;
          }
        }
      }
      // The packed output is cleared first unless the tensor-core epilogue writes every word of
      // it (channel-pad words included): no image padding (N a multiple of 8). A following
      // or_pool is folded into the tensor-core epilogue (atomic OR into the zeroed pooled tensor).
      const bool tc = will_use_tc(s, e, EngineHint::Auto, &L.tc);
      e.pool = tc ? fusable_pool(sh, i) : 0;
      if (i + 1 < sh.layers.size()) sh.layers[i + 1].pool_fused = e.pool != 0;
      if (e.pool)
        BT_CUDA(cudaMemsetAsync(out, 0, act_words(l.out_h / e.pool, l.out_w / e.pool, batch, l.out_channels, 0, 0, 0) * 8, st));
      else if (!(tc && np == batch))
        BT_CUDA(cudaMemsetAsync(out, 0, act_words(l.out_h, l.out_w, batch, l.out_channels, 0, 0, 0) * 8, st));
      if (sh.tune_pass >= 0 && tc) {  // plan tuner: this pass's candidate geometry
        if (L.cands.empty()) {
          L.cands = tc_choices(s, e);
          for (const TcChoice& c : L.cands) L.cand_names.push_back(tc_choice_name(s, e, c));
          L.cand_ms.assign(L.cands.size(), 0.0);
        }
        L.choice = L.cands[std::min((size_t)sh.tune_pass, L.cands.size() - 1)];
      }
      L.engine = launch_bgemm(s, in, L.filt.get<uint64_t>(), e, st, EngineHint::Auto, &L.tc, &L.choice);
      if (e.pool) L.engine += "+pool";
      ++launches;
      cur ^= 1;
      H = l.out_h; W = l.out_w; C = l.out_channels;
    } else if (l.kind == BTNN_OR_POOL && L.pool_fused) {
      L.engine = "fused";  // done by the previous conv's epilogue
      H = l.out_h; W = l.out_w;
    } else if (l.kind == BTNN_OR_POOL) {
      const size_t pw = np * act_cpad(C, 0, 0) / 64;
      launch_or_pool(sh.act[cur].get<uint64_t>(), (int)H, (int)W, pw, (int)l.window, (int)l.pool_stride, (int)l.out_h,
                     (int)l.out_w, sh.act[cur ^ 1].get<uint64_t>(), st);
      ++launches;
      L.engine = "orpool";
      cur ^= 1;
      H = l.out_h; W = l.out_w;
    } else {
      if (!in_fc) {
        uint64_t* dst = sh.fc[fcur].get<uint64_t>();
        const size_t row_words = ru(l.in_channels, 128) / 64;
        if (i == 0) {
          // FC-first model: binarize the raw input (inference.hpp:149-151) and flag
          // non-finite values (the input check of inference.hpp:69-75, no separate pass).
          launch_pack_rows(d_x, batch, l.in_channels, row_words * 2, reinterpret_cast<uint32_t*>(dst),
                           sh.flag.get<int>(), st);
        } else {
          launch_flatten(sh.act[cur].get<uint64_t>(), (int)H, (int)W, (int)batch, (int)C, (int)np,
                         (int)act_cpad(C, 0, 0), dst, row_words, st);
        }
        ++launches;
        in_fc = true;
      }
      const ConvShape s = fc_shape(l, batch);
      Epi e;
      if (l.kind == BTNN_BIT_FC) {
        uint64_t* out = sh.fc[fcur ^ 1].get<uint64_t>();
        // every engine writes whole 64-bit words of its output columns: only rows with pad
        // words past O need clearing
        if (s.O % 128) BT_CUDA(cudaMemsetAsync(out, 0, batch * (size_t)s.cwo * 8, st));
        e.mode = EPI_BITS;
        e.out_bits = out;
        e.thr_lo = L.thr_lo.get<long long>();
        e.thr_hi = L.thr_hi.get<long long>();
        e.split_ws = L.split_ws.get<int32_t>();
        L.engine = launch_bgemm(s, sh.fc[fcur].get<uint64_t>(), L.filt.get<uint64_t>(), e, st, EngineHint::Auto, &L.tc);
        fcur ^= 1;
      } else {
        const size_t O = l.units;
        e.mode = EPI_F64;
        e.bn_mean = L.bn.get<double>(); e.bn_s = e.bn_mean + O; e.bn_gamma = e.bn_mean + 2 * O; e.bn_beta = e.bn_mean + 3 * O;
        e.bn_rcp = e.bn_mean + 4 * O;
        e.rout = d_logits;  // logits = bn(v) (inference.hpp:161-164)
        e.split_ws = L.split_ws.get<int32_t>();
        if (i + 1 == sh.layers.size() && !timed) {  // the packed BMM may write the labels too
          e.labels = d_labels;
          e.labels_done = &labels_done;
        }
        L.engine = launch_bgemm(s, sh.fc[fcur].get<uint64_t>(), L.filt.get<uint64_t>(), e, st, EngineHint::Auto, &L.tc);
      }
      launches += L.engine == std::string("tc_i8_splitk") ? 2 : 1;
    }
  }
  if (timed) BT_CUDA(cudaEventRecord(sh.events[sh.layers.size()], st));
  if (!labels_done) {
    launch_argmax(d_logits, (int)batch, (int)plan->classes, d_labels, st);
    ++launches;
  }
  return launches;
}

// Enqueue via a cached CUDA graph (or eagerly when timing layers). The graph is
// captured on the shard's stream and launched on `launch_stream` (the caller's stream
// for run_device, the shard's own stream otherwise).
static void run_shard_device(btnn_plan* plan, Shard& sh, const float* d_x, size_t batch, double* d_logits,
                             int32_t* d_labels, bool timed, cudaStream_t launch_stream = nullptr) {
  if (timed) {
    sh.launches = enqueue_forward(plan, sh, d_x, batch, d_logits, d_labels, true);
    return;
  }
  auto key = std::make_tuple(batch, (const void*)d_x, (const void*)d_logits, (const void*)d_labels, engine_override());
  auto it = sh.graphs.find(key);
  if (it == sh.graphs.end()) {
    cudaGraph_t g;
    BT_CUDA(cudaStreamBeginCapture(sh.stream, cudaStreamCaptureModeThreadLocal));
    size_t n = 0;
    try {
      n = enqueue_forward(plan, sh, d_x, batch, d_logits, d_labels, false);
    } catch (...) {
      cudaStreamEndCapture(sh.stream, &g);
      throw;
    }
    BT_CUDA(cudaStreamEndCapture(sh.stream, &g));
    Shard::Graph gr;
    BT_CUDA(cudaGraphInstantiate(&gr.exec, g, 0));
    cudaGraphDestroy(g);
    sh.launches = n;
    for (const LayerDev& L : sh.layers) gr.wrote_half.push_back(L.wrote_half);
    it = sh.graphs.emplace(key, std::move(gr)).first;
  }
  for (size_t i = 0; i < sh.layers.size(); ++i) sh.layers[i].wrote_half = it->second.wrote_half[i];
  BT_CUDA(cudaGraphLaunch(it->second.exec, launch_stream ? launch_stream : sh.stream));
}

// Host-buffer run (the C ABI's run_inference). The input copy is the long pole end to end
// (602 KB per ImageNet image over PCIe, ~55 GB/s measured: ~90 K img/s), so the batch is cut
// into chunks: chunk k+1's host->device copy runs on the copy stream while chunk k's graph
// runs on the compute stream, and chunk k's logits / labels go back to the host right behind
// its graph. Samples are independent, so chunking does not change any result.
//
// The schedule comes from measurements, not constants (calibrate_e2e): the copy time per image
// c from a timed copy of the caller's own buffer, and the graph's time t(b) = t0 + b * s from
// two timed replays (ResNet-18 on a B200: t0 ~ 0.29 ms, s ~ 4.8 us, c ~ 10.9 us). The step ends
// when the last chunk's copy and then its compute finish, so the last chunk wants to be small —
// but a chunk's graph must also finish before the next chunk's copy does, or the compute stream
// backs up: walking backwards, chunk k may be as large as (b_{k+1} * c - t0) / s, so chunks
// grow geometrically from a small last one. Every candidate (each last-chunk size, uniform
// chunks, one chunk) is simulated with the model and the fastest kept.
#ifndef BTNN_E2E_MIN_BYTES
#define BTNN_E2E_MIN_BYTES (64 * 1024)
#endif
static bool host_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// kChunkIssueUs: host issue cost of one chunk (copy, event record and wait, graph launch, two
// result copies: ~6 runtime calls), which paces the pipeline when a chunk's device work is
// short (MNIST-MLP: ~20 us graphs).
constexpr double kChunkIssueUs = 25.0;
static double simulate_chunks(const std::vector<size_t>& sizes, double c, double t0, double s) {
  double copy_done = 0.0, comp_end = 0.0, issued = 0.0;
  for (size_t b : sizes) {
    issued += kChunkIssueUs;
    copy_done = std::max(copy_done, issued) + (double)b * c;
    comp_end = std::max(copy_done, comp_end) + t0 + (double)b * s;
  }
  return comp_end;
}

static std::vector<size_t> chunk_schedule(const Shard& sh, size_t batch) {
  static const size_t fixed = (size_t)timing_knob("BTNN_E2E_CHUNK", 0);  // timing experiments
  if (fixed) {
    std::vector<size_t> sizes;
    for (size_t b0 = 0; b0 < batch; b0 += fixed) sizes.push_back(std::min(fixed, batch - b0));
    return sizes;
  }
  if (!sh.e2e_cal || batch < 16) return {batch};
  const double c = sh.e2e_c, t0 = sh.e2e_t0, sl = sh.e2e_s;
  std::vector<size_t> best{batch};
  double best_t = simulate_chunks(best, c, t0, sl);
  auto consider = [&](std::vector<size_t> v) {
    if (v.empty() || v.size() > kMaxChunks) return;
    const double t = simulate_chunks(v, c, t0, sl);
    if (t < best_t) best_t = t, best = std::move(v);
  };
  const size_t cap = std::min<size_t>(batch, 512);
  for (size_t last = 8; last <= std::min<size_t>(batch, 256); last += 8) {
    // backwards from the last chunk: each earlier chunk as large as its successor's copy hides
    std::vector<size_t> rev{last};
    size_t tot = last;
    while (tot < batch && rev.size() < kMaxChunks) {
      const double lim = ((double)rev.back() * c - t0) / sl;
      size_t b = lim <= (double)rev.back() ? 2 * rev.back() : (size_t)lim / 8 * 8;  // (compute-bound: double)
      b = std::max<size_t>(8, std::min(b, cap));
      b = std::min(b, batch - tot);
      rev.push_back(b);
      tot += b;
    }
    if (tot < batch) continue;
    consider(std::vector<size_t>(rev.rbegin(), rev.rend()));
  }
  for (size_t u = 16; u <= std::min<size_t>(batch, 256); u += 16) {  // uniform chunks
    std::vector<size_t> v;
    for (size_t b0 = 0; b0 < batch; b0 += u) v.push_back(std::min(u, batch - b0));
    consider(v);
  }
  return best;
}

// One-time measurement of the chunk model on the caller's buffer (first host run of a shard):
// a timed copy of up to 64 images (after one untimed), and two timed replays of the graph at
// b = 16 and b = 128 (or the largest batch the shard holds) on whatever the device input buffer
// holds — the graph's speed does not depend on the values; any non-finite flag raised here is
// cleared by the run that follows.
static void calibrate_e2e(btnn_plan* plan, Shard& sh, const float* x, size_t batch) {
  const size_t xin = plan->in_h * plan->in_w * plan->in_c;
  cudaEvent_t e0, e1;
  BT_CUDA(cudaEventCreate(&e0));
  BT_CUDA(cudaEventCreate(&e1));
  auto elapsed_us = [&](cudaStream_t st) {
    BT_CUDA(cudaEventRecord(e1, st));
    BT_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    BT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    return 1e3 * (double)ms;
  };
  const size_t nb = std::min<size_t>(batch, 64);
  const size_t b1 = std::min<size_t>(16, sh.max_batch), b2 = std::min<size_t>(128, sh.max_batch);
  BT_CUDA(cudaMemsetAsync(sh.x.get(), 0, b2 * xin * sizeof(float), sh.copy_stream));  // (finite values)
  BT_CUDA(cudaMemcpyAsync(sh.x.get(), x, nb * xin * sizeof(float), cudaMemcpyHostToDevice, sh.copy_stream));
  BT_CUDA(cudaEventRecord(e0, sh.copy_stream));
  BT_CUDA(cudaMemcpyAsync(sh.x.get(), x, nb * xin * sizeof(float), cudaMemcpyHostToDevice, sh.copy_stream));
  const double c = elapsed_us(sh.copy_stream) / (double)nb;
  double t[2] = {0.0, 0.0};
  const size_t bs[2] = {b1, b2};
  for (int i = 0; i < 2; ++i) {
    run_shard_device(plan, sh, sh.x.get<float>(), bs[i], sh.logits.get<double>(), sh.labels.get<int32_t>(), false);
    BT_CUDA(cudaEventRecord(e0, sh.stream));
    run_shard_device(plan, sh, sh.x.get<float>(), bs[i], sh.logits.get<double>(), sh.labels.get<int32_t>(), false);
    t[i] = elapsed_us(sh.stream);
  }
  BT_CUDA(cudaEventDestroy(e0));
  BT_CUDA(cudaEventDestroy(e1));
  const double sl = b2 > b1 ? std::max(0.0, (t[1] - t[0]) / (double)(b2 - b1)) : t[0] / (double)b1;
  sh.e2e_c = c;
  sh.e2e_s = sl;
  sh.e2e_t0 = std::max(0.0, t[0] - sl * (double)b1);
  sh.e2e_cal = true;
}

static void run_shard_host(btnn_plan* plan, Shard& sh, const float* x, size_t batch, double* logits, int32_t* labels) {
  BT_CUDA(cudaSetDevice(sh.device));
  const size_t xin = plan->in_h * plan->in_w * plan->in_c;
  const bool timed = plan->breakdown && &sh == plan->shards[0].get();
  // Small inputs (Cifar 12 KB, MNIST 3 KB per image) copy in a fraction of the compute time and
  // each extra chunk costs more host and launch time than it hides (measured with the model's
  // schedules, XDEFS=-DBTNN_E2E_MIN_BYTES=0: Cifar-VGG b1024 700 K -> 668 K img/s, MNIST-MLP
  // 7.7 M -> 5.8 M with 3-4 chunks): one graph each.
  const bool pipelined = batch >= 16 && xin * sizeof(float) >= BTNN_E2E_MIN_BYTES;
  // (re-measured when the caller switches between pinned and pageable input buffers: the copy
  // rate differs by ~2-4x)
  const bool x_pinned = pipelined && host_pinned(x);
  if (!timed && pipelined && (!sh.e2e_cal || sh.e2e_cal_pinned != x_pinned) && !timing_knob("BTNN_E2E_CHUNK", 0)) {
    calibrate_e2e(plan, sh, x, batch);
    sh.e2e_cal_pinned = x_pinned;
  }
  const std::vector<size_t> sizes = timed || !pipelined ? std::vector<size_t>{batch} : chunk_schedule(sh, batch);
  BT_CUDA(cudaMemsetAsync(sh.flag.get(), 0, sizeof(int), sh.stream));
  const bool pinned_out = sizes.size() > 1 && host_pinned(logits) && host_pinned(labels);
  size_t b0 = 0;
  for (size_t k = 0; k < sizes.size(); ++k) {
    const size_t bn = sizes[k];
    float* dx = sh.x.get<float>() + b0 * xin;
    BT_CUDA(cudaMemcpyAsync(dx, x + b0 * xin, bn * xin * sizeof(float), cudaMemcpyHostToDevice, sh.copy_stream));
    BT_CUDA(cudaEventRecord(sh.in_ready[k], sh.copy_stream));
    BT_CUDA(cudaStreamWaitEvent(sh.stream, sh.in_ready[k], 0));
    double* dl = sh.logits.get<double>() + b0 * plan->classes;
    int32_t* db = sh.labels.get<int32_t>() + b0;
    run_shard_device(plan, sh, dx, bn, dl, db, timed);
    if (pinned_out) {  // this chunk's results leave (own stream) while the next chunk computes
      BT_CUDA(cudaEventRecord(sh.out_ready[k], sh.stream));
      BT_CUDA(cudaStreamWaitEvent(sh.d2h_stream, sh.out_ready[k], 0));
      BT_CUDA(cudaMemcpyAsync(logits + b0 * plan->classes, dl, bn * plan->classes * sizeof(double),
                              cudaMemcpyDeviceToHost, sh.d2h_stream));
      BT_CUDA(cudaMemcpyAsync(labels + b0, db, bn * sizeof(int32_t), cudaMemcpyDeviceToHost, sh.d2h_stream));
    }
    b0 += bn;
  }
  if (!pinned_out) {  // (a copy to pageable memory blocks the host: once, at the end)
    BT_CUDA(cudaMemcpyAsync(logits, sh.logits.get(), batch * plan->classes * sizeof(double), cudaMemcpyDeviceToHost,
                            sh.stream));
    BT_CUDA(cudaMemcpyAsync(labels, sh.labels.get(), batch * sizeof(int32_t), cudaMemcpyDeviceToHost, sh.stream));
  }
  int bad = 0;
  BT_CUDA(cudaMemcpyAsync(&bad, sh.flag.get(), sizeof(int), cudaMemcpyDeviceToHost, sh.stream));
  BT_CUDA(cudaStreamSynchronize(sh.stream));
  if (pinned_out) BT_CUDA(cudaStreamSynchronize(sh.d2h_stream));
  require(!bad, BTNN_INVALID_INPUT, "run_inference: non-finite input");
  if (plan->breakdown && &sh == plan->shards[0].get()) {
    plan->layer_ms.assign(sh.layers.size(), 0.0);
    for (size_t i = 0; i < sh.layers.size(); ++i) {
      float ms = 0.f;
      BT_CUDA(cudaEventElapsedTime(&ms, sh.events[i], sh.events[i + 1]));
      plan->layer_ms[i] = ms;
    }
  }
}

}  // namespace btnn_gpu

using namespace btnn_gpu;

extern "C" {

namespace btnn_gpu {
// Plan tuner (north star (2): the variant per layer shape from measured throughput). Every
// tensor-core conv layer lists the distinct geometries its shape allows (tc_choices: the cost
// model's pick, halo mode at each feasible sites-per-tile, the TMEM-A path); pass k runs
// candidate k of every layer in one eager forward at the shard's max batch (an all-zero
// input) with per-layer events, twice (the first warms up), and each layer keeps its fastest.
// Every candidate computes the same exact sums, so the pick changes speed only.
static std::atomic<int> g_autotune{[] {
  const char* v = std::getenv("BTNN_AUTOTUNE");
  return v ? std::atoi(v) : 1;
}()};

static void tune_shard(btnn_plan* plan, Shard& sh) {
  BT_CUDA(cudaSetDevice(sh.device));
  const size_t B = sh.max_batch;
  BT_CUDA(cudaMemsetAsync(sh.x.get(), 0, sh.x.bytes(), sh.stream));
  size_t passes = 1;
  for (size_t pass = 0; pass < passes; ++pass) {
    sh.tune_pass = (int)pass;
    for (int rep = 0; rep < 2; ++rep) {
      BT_CUDA(cudaMemsetAsync(sh.flag.get(), 0, sizeof(int), sh.stream));
      enqueue_forward(plan, sh, sh.x.get<float>(), B, sh.logits.get<double>(), sh.labels.get<int32_t>(), true);
    }
    BT_CUDA(cudaStreamSynchronize(sh.stream));
    for (size_t i = 0; i < sh.layers.size(); ++i) {
      LayerDev& L = sh.layers[i];
      passes = std::max(passes, L.cands.size());
      if (pass < L.cands.size()) {
        float ms = 0.f;
        BT_CUDA(cudaEventElapsedTime(&ms, sh.events[i], sh.events[i + 1]));
        L.cand_ms[pass] = ms;
      }
    }
  }
  sh.tune_pass = -1;
  for (LayerDev& L : sh.layers) {
    if (L.cands.empty()) continue;
    size_t best = 0;
    for (size_t k = 1; k < L.cands.size(); ++k)
      if (L.cand_ms[k] < L.cand_ms[best]) best = k;
    L.choice = L.cands[best];
  }
}
}  // namespace btnn_gpu

int btnn_cuda_set_autotune(int enabled) {
  return guard([&] { g_autotune.store(enabled != 0); });
}

int btnn_cuda_plan_layer_choice(btnn_plan* plan, size_t i, char* buf, size_t n, double* ms, size_t n_ms) {
  return guard([&] {
    require(plan && !plan->shards.empty() && i < plan->specs.size(), BTNN_INVALID_INPUT, "plan_layer_choice: bad layer");
    const LayerDev& L = plan->shards[0]->layers[i];
    std::string out;
    size_t pick = 0;
    for (size_t k = 0; k < L.cands.size(); ++k)
      if (L.cands[k].spt == L.choice.spt && L.cands[k].tmem_a == L.choice.tmem_a && L.cands[k].groups == L.choice.groups)
        pick = k;
    for (size_t k = 0; k < L.cands.size(); ++k) {
      out += (k ? "," : "") + std::string(k == pick ? "*" : "") + L.cand_names[k];
      if (ms && k < n_ms) ms[k] = L.cand_ms[k];
    }
    if (buf && n) {
      const size_t c = std::min(n - 1, out.size());
      std::memcpy(buf, out.data(), c);
      buf[c] = 0;
    }
  });
}

int btnn_cuda_plan_set_layer_choice(btnn_plan* plan, size_t i, size_t k) {
  return guard([&] {
    require(plan && !plan->shards.empty() && i < plan->specs.size(), BTNN_INVALID_INPUT, "plan_set_layer_choice: bad layer");
    for (auto& sh : plan->shards) {
      LayerDev& L = sh->layers[i];
      require(k < L.cands.size(), BTNN_INVALID_INPUT, "plan_set_layer_choice: no such candidate");
      L.choice = L.cands[k];
      BT_CUDA(cudaSetDevice(sh->device));
      for (auto& kv : sh->graphs) cudaGraphExecDestroy(kv.second.exec);  // captured with the old choice
      sh->graphs.clear();
    }
  });
}

int btnn_cuda_plan_create(const btnn_model_spec* m, const btnn_weight_store* ws, size_t max_batch, const int* devices,
                          int n_devices, btnn_plan** out) {
  return guard([&] {
    require(out != nullptr, BTNN_INVALID_INPUT, "plan_create: null out");
    *out = nullptr;
    check_plan_inputs(m, ws);
    require(max_batch > 0, BTNN_INVALID_INPUT, "plan_create: zero max_batch");
    int count = 0;
    BT_CUDA(cudaGetDeviceCount(&count));
    std::vector<int> devs;
    if (devices && n_devices > 0)
      devs.assign(devices, devices + n_devices);
    else
      devs.push_back(0);
    for (int d : devs) require(d >= 0 && d < count, BTNN_INVALID_INPUT, "plan_create: no such device");
    auto plan = std::make_unique<btnn_plan>();
    plan->name = m->name ? m->name : "";
    plan->in_h = m->in_h; plan->in_w = m->in_w; plan->in_c = m->in_c; plan->classes = m->classes;
    plan->specs.assign(m->layers, m->layers + m->n_layers);
    const size_t per = cdiv(max_batch, devs.size());
    for (int d : devs) {
      auto sh = std::make_unique<Shard>();
      sh->device = d;
      sh->max_batch = per;
      build_shard(*sh, m, ws);
      plan->shards.push_back(std::move(sh));
    }
    if (g_autotune.load())
      for (auto& sh : plan->shards) tune_shard(plan.get(), *sh);
    *out = plan.release();
  });
}

int btnn_cuda_plan_run(btnn_plan* plan, const float* x, size_t batch, double* logits, int32_t* labels) {
  return guard([&] {
    require(plan != nullptr, BTNN_INVALID_INPUT, "plan_run: null plan");
    require(batch > 0, BTNN_INVALID_INPUT, "run_inference: empty batch");
    const size_t n = plan->shards.size();
    const size_t per = cdiv(batch, n);
    require(per <= plan->shards[0]->max_batch, BTNN_INVALID_INPUT, "plan_run: batch exceeds the plan's max_batch");
    const size_t xin = plan->in_h * plan->in_w * plan->in_c;
    std::vector<int> codes(n, BTNN_OK);
    std::vector<std::string> msgs(n);
    auto work = [&](size_t k) {
      const size_t b0 = k * per;
      if (b0 >= batch) return;
      const size_t bn = std::min(per, batch - b0);
      try {
        run_shard_host(plan, *plan->shards[k], x + b0 * xin, bn, logits + b0 * plan->classes, labels + b0);
      } catch (const Error& e) {
        codes[k] = e.code;
        msgs[k] = e.what();
      } catch (const std::exception& e) {
        codes[k] = BTNN_CUDA_ERROR;
        msgs[k] = e.what();
      }
    };
    if (n == 1) {
      work(0);
    } else {
      std::vector<std::thread> th;
      for (size_t k = 0; k < n; ++k) th.emplace_back(work, k);
      for (auto& t : th) t.join();
    }
    // Report the lowest-numbered failing code (invalid input beats device errors).
    int best = BTNN_OK;
    std::string msg;
    for (size_t k = 0; k < n; ++k)
      if (codes[k] != BTNN_OK && (best == BTNN_OK || codes[k] < best)) { best = codes[k]; msg = msgs[k]; }
    if (best != BTNN_OK) fail(best, msg);
  });
}

int btnn_cuda_plan_run_device(btnn_plan* plan, int shard, const float* d_x, size_t batch, double* d_logits,
                              int32_t* d_labels, void* stream) {
  return guard([&] {
    require(plan && shard >= 0 && (size_t)shard < plan->shards.size(), BTNN_INVALID_INPUT, "plan_run_device: bad shard");
    Shard& sh = *plan->shards[shard];
    require(batch > 0 && batch <= sh.max_batch, BTNN_INVALID_INPUT, "plan_run_device: batch out of range");
    BT_CUDA(cudaSetDevice(sh.device));
    // stream == NULL: the plan's own stream (caller synchronizes via the device);
    // otherwise the graph is launched straight onto the caller's stream. The input check's
    // non-finite flag is cleared first and read back by btnn_cuda_plan_input_status.
    cudaStream_t ls = stream ? static_cast<cudaStream_t>(stream) : sh.stream;
    BT_CUDA(cudaMemsetAsync(sh.flag.get(), 0, sizeof(int), ls));
    run_shard_device(plan, sh, d_x, batch, d_logits ? d_logits : sh.logits.get<double>(),
                     d_labels ? d_labels : sh.labels.get<int32_t>(), false, static_cast<cudaStream_t>(stream));
  });
}

int btnn_cuda_plan_e2e_schedule(btnn_plan* plan, int shard, size_t batch, double* model, size_t* sizes, size_t cap,
                                size_t* n_sizes) {
  return guard([&] {
    require(plan && shard >= 0 && (size_t)shard < plan->shards.size() && model && sizes && n_sizes, BTNN_INVALID_INPUT,
            "plan_e2e_schedule: bad arguments");
    const Shard& sh = *plan->shards[shard];
    model[0] = sh.e2e_cal ? 1.0 : 0.0;
    model[1] = sh.e2e_c;
    model[2] = sh.e2e_t0;
    model[3] = sh.e2e_s;
    const std::vector<size_t> v = chunk_schedule(sh, batch);
    model[4] = sh.e2e_cal ? simulate_chunks(v, sh.e2e_c, sh.e2e_t0, sh.e2e_s) : 0.0;
    *n_sizes = v.size();
    for (size_t i = 0; i < v.size() && i < cap; ++i) sizes[i] = v[i];
  });
}

int btnn_cuda_plan_input_status(btnn_plan* plan, int shard, int* nonfinite) {
  return guard([&] {
    require(plan && shard >= 0 && (size_t)shard < plan->shards.size() && nonfinite, BTNN_INVALID_INPUT,
            "plan_input_status: bad arguments");
    Shard& sh = *plan->shards[shard];
    BT_CUDA(cudaSetDevice(sh.device));
    int f = 0;
    BT_CUDA(cudaMemcpy(&f, sh.flag.get(), sizeof(int), cudaMemcpyDeviceToHost));
    *nonfinite = f != 0;
  });
}

int btnn_cuda_plan_layer_ms(btnn_plan* plan, double* ms, size_t n_layers) {
  return guard([&] {
    require(plan && n_layers == plan->specs.size(), BTNN_INVALID_INPUT, "plan_layer_ms: size mismatch");
    for (size_t i = 0; i < n_layers; ++i) ms[i] = i < plan->layer_ms.size() ? plan->layer_ms[i] : 0.0;
  });
}

int btnn_cuda_plan_set_breakdown(btnn_plan* plan, int enabled) {
  return guard([&] {
    require(plan != nullptr, BTNN_INVALID_INPUT, "null plan");
    plan->breakdown = enabled != 0;
  });
}

int btnn_cuda_plan_launches(btnn_plan* plan, size_t batch, size_t* launches) {
  return guard([&] {
    require(plan != nullptr, BTNN_INVALID_INPUT, "null plan");
    (void)batch;
    *launches = plan->shards[0]->launches;
  });
}

int btnn_cuda_plan_read_tap(btnn_plan* plan, size_t i, size_t batch, double* out) {
  return guard([&] {
    require(plan && !plan->shards.empty() && i < plan->specs.size(), BTNN_INVALID_INPUT, "plan_read_tap: bad layer");
    Shard& sh = *plan->shards[0];
    const LayerDev& L = sh.layers[i];
    require(L.spec.residual_out && L.tap.get(), BTNN_INVALID_INPUT, "plan_read_tap: layer has no residual_out");
    require(batch > 0 && batch <= sh.max_batch, BTNN_INVALID_INPUT, "plan_read_tap: bad batch");
    BT_CUDA(cudaSetDevice(sh.device));
    BT_CUDA(cudaStreamSynchronize(sh.stream));
    // The tap as the last run stored it: full resolution, or pre-averaged (see tap_dims).
    const size_t hw = L.wrote_half ? (L.spec.out_h / 2) * (L.spec.out_w / 2) : L.spec.out_h * L.spec.out_w;
    BT_CUDA(cudaMemcpy(out, L.wrote_half ? L.tap_half.get() : L.tap.get(),
                       hw * batch * L.spec.out_channels * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

int btnn_cuda_plan_tap_dims(btnn_plan* plan, size_t i, size_t* dims) {
  return guard([&] {
    require(plan && !plan->shards.empty() && i < plan->specs.size() && dims, BTNN_INVALID_INPUT,
            "plan_tap_dims: bad layer");
    const LayerDev& L = plan->shards[0]->layers[i];
    require(L.spec.residual_out, BTNN_INVALID_INPUT, "plan_tap_dims: layer has no residual_out");
    dims[0] = L.wrote_half ? L.spec.out_h / 2 : L.spec.out_h;
    dims[1] = L.wrote_half ? L.spec.out_w / 2 : L.spec.out_w;
    dims[2] = L.wrote_half ? 1 : 0;  // 1: 2x2-averaged (adapt_shortcut's halve, inference.hpp:43-63)
    dims[3] = L.spec.out_channels;
  });
}

const char* btnn_cuda_plan_layer_engine(btnn_plan* plan, size_t i) {
  if (!plan || plan->shards.empty() || i >= plan->shards[0]->layers.size()) return "";
  return plan->shards[0]->layers[i].engine.c_str();
}

int btnn_cuda_plan_destroy(btnn_plan* plan) {
  return guard([&] { delete plan; });
}

}  // extern "C"
