// btnn/cuda.hpp — drop-in B200 (sm_100a) twins of the btnn layer/model API.
//
// Include it next to the reference headers (proj/include/btnn) and link
// libbtnn_cuda.so. Every function has the signature, value types, output layout and
// error classes of the reference function it replaces (file:line below), and runs on the
// GPU through the C ABI in btnn_cuda.h:
//
//   btnn::bmm_raw / bmm_pm1 / bmm_pm1_bin   -> btnn::cuda::bmm_raw / ...   (bmm.hpp:204-274)
//   btnn::bconv_pm1 / bconv_fused           -> btnn::cuda::bconv_pm1 / ... (bconv.hpp:138-194)
//   btnn::first_conv_bwn / or_pool          -> btnn::cuda::...             (bconv.hpp:198-272)
//   btnn::pack_matrix / to_fsb / from_fsb   -> btnn::cuda::...             (bit_matrix.hpp:135-253)
//   btnn::pack_nhwc / flatten_to_matrix     -> btnn::cuda::...             (tensors.hpp:162-237)
//   btnn::run_inference                     -> btnn::cuda::run_inference   (inference.hpp:67)
//
// `threads` arguments are accepted and ignored (the GPU grid replaces parallel_chunks,
// common.hpp:56-75); results are identical to the CPU engine bit for bit. For repeated
// inference, btnn::cuda::Engine keeps the weights resident and replays a CUDA graph.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "btnn/bconv.hpp"
#include "btnn/bit_matrix.hpp"
#include "btnn/bmm.hpp"
#include "btnn/inference.hpp"
#include "btnn/layer_math.hpp"
#include "btnn/model.hpp"
#include "btnn/tensors.hpp"
#include "btnn/weights.hpp"
#include "btnn_cuda.h"

namespace btnn::cuda {

namespace detail {

// Status code -> the reference's exception taxonomy (common.hpp:14-32).
[[noreturn]] inline void rethrow(int code) {
  const std::string msg = btnn_cuda_last_error();
  switch (code) {
    case BTNN_INVALID_INPUT: throw invalid_input(msg);
    case BTNN_UNSUPPORTED_SHAPE: throw unsupported_shape(msg);
    case BTNN_IO_ERROR: throw io_error(msg);
    case BTNN_VALIDATION_ERROR: throw validation_error(msg);
    default: throw std::runtime_error("btnn::cuda: " + msg);
  }
}
inline void check(int code) {
  if (code != BTNN_OK) rethrow(code);
}

inline btnn_matrix_desc desc(const BitMatrix& m) {
  return {m.rows(), m.cols(), static_cast<int>(m.layout()), m.geometry().bh, m.geometry().bw};
}
inline btnn_act_desc desc(const BitTensorHWNC& t) {
  return {t.height, t.width, t.batch, t.channels, t.tiled ? 1 : 0, t.geo.bh, t.geo.bw};
}
inline btnn_filter_desc desc(const BitFilterKKOC& f) {
  return {f.kh, f.kw, f.out_channels, f.in_channels, f.tiled ? 1 : 0, f.geo.bh, f.geo.bw};
}
inline btnn_bmm_options opts(const BmmOptions& o) {
  return {static_cast<int>(o.variant), o.blocking.rows, o.blocking.cols, o.blocking.k_bits, o.threads};
}
inline btnn_conv_geom geom(const Conv2dGeometry& g) { return {g.kh, g.kw, g.stride, g.pad}; }

struct ThresholdArrays {
  std::vector<double> tau;
  std::vector<std::uint8_t> kind;
  explicit ThresholdArrays(std::span<const Threshold> t) {
    for (const auto& x : t) {
      tau.push_back(x.tau);
      kind.push_back(static_cast<std::uint8_t>(x.kind));
    }
  }
};

inline btnn_bn bn_view(const BnParams& bn) {
  return {bn.gamma.data(), bn.beta.data(), bn.mean.data(), bn.var.data(), bn.gamma.size(), bn.eps};
}

}  // namespace detail

// ---- BMM (bmm.hpp:204-274) ----------------------------------------------------------------
inline IntMatrix bmm_raw(const BitMatrix& a, const BitMatrix& b, const BmmOptions& opt = {}) {
  IntMatrix out(a.rows(), b.cols());
  const auto da = detail::desc(a), db = detail::desc(b);
  const auto o = detail::opts(opt);
  detail::check(btnn_cuda_bmm_raw(&da, a.data(), &db, b.data(), &o, out.v.data()));
  return out;
}

inline IntMatrix bmm_pm1(const BitMatrix& a, const BitMatrix& b, const BmmOptions& opt = {}) {
  IntMatrix out(a.rows(), b.cols());
  const auto da = detail::desc(a), db = detail::desc(b);
  const auto o = detail::opts(opt);
  detail::check(btnn_cuda_bmm_pm1(&da, a.data(), &db, b.data(), &o, out.v.data()));
  return out;
}

inline BitMatrix bmm_pm1_bin(const BitMatrix& a, const BitMatrix& b, const BmmOptions& opt = {},
                             std::span<const Threshold> thresholds = {}) {
  if (!thresholds.empty() && thresholds.size() != b.cols())
    throw invalid_input("bmm_pm1_bin: need one threshold per output column");
  const Layout out_layout = a.layout() == Layout::FsbRow ? Layout::FsbRow : Layout::RowPacked;
  BitMatrix out(a.rows(), b.cols(), out_layout, a.geometry());
  const detail::ThresholdArrays t(thresholds);
  const auto da = detail::desc(a), db = detail::desc(b);
  const auto o = detail::opts(opt);
  detail::check(btnn_cuda_bmm_pm1_bin(&da, a.data(), &db, b.data(), &o, t.tau.data(), t.kind.data(), t.tau.size(),
                                      out.data()));
  return out;
}

// ---- BConv (bconv.hpp:138-272) ------------------------------------------------------------
inline IntTensorPQNO bconv_pm1(const BitTensorHWNC& in, const BitFilterKKOC& filt, const Conv2dGeometry& geo,
                               int threads = 0) {
  (void)threads;
  IntTensorPQNO out(geo.out_h(in.height), geo.out_w(in.width), in.batch, filt.out_channels);
  const auto di = detail::desc(in);
  const auto df = detail::desc(filt);
  const auto g = detail::geom(geo);
  detail::check(btnn_cuda_bconv_pm1(&di, in.bits.data(), &df, filt.bits.data(), &g, out.v.data()));
  return out;
}

inline BitTensorHWNC bconv_fused(const BitTensorHWNC& in, const BitFilterKKOC& filt, const Conv2dGeometry& geo,
                                 const ConvFused& f) {
  const std::size_t o = filt.out_channels;
  const bool thresholded = !f.thresholds.empty();
  if (thresholded == (f.bn != nullptr)) throw invalid_input("bconv_fused: need exactly one of thresholds or bn");
  if (thresholded && f.thresholds.size() != o) throw invalid_input("bconv_fused: need one threshold per output channel");
  if (f.bn && f.bn->channels() != o) throw invalid_input("bconv_fused: bn channel count does not match filter");
  if ((f.residual_in || f.residual_out) && !f.bn) throw invalid_input("bconv_fused: residual ports require the bn route");
  const std::size_t p = geo.out_h(in.height), q = geo.out_w(in.width);
  if (f.residual_in) {
    const auto& t = *f.residual_in;
    if (t.p != p || t.q != q || t.batch != in.batch || t.channels != o)
      throw invalid_input("bconv_fused: residual_in dims do not match output");
  }
  if (f.residual_out) *f.residual_out = RealTensorPQNO(p, q, in.batch, o);
  BitTensorHWNC out(p, q, in.batch, o, in.tiled, in.geo);
  const detail::ThresholdArrays t(f.thresholds);
  btnn_bn bnv{};
  btnn_conv_fused cf{};
  if (thresholded) {
    cf.tau = t.tau.data();
    cf.kind = t.kind.data();
    cf.n_thresholds = t.tau.size();
  } else {
    bnv = detail::bn_view(*f.bn);
    cf.bn = &bnv;
  }
  cf.residual_in = f.residual_in ? f.residual_in->v.data() : nullptr;
  cf.residual_out = f.residual_out ? f.residual_out->v.data() : nullptr;
  const auto di = detail::desc(in);
  const auto df = detail::desc(filt);
  const auto g = detail::geom(geo);
  detail::check(btnn_cuda_bconv_fused(&di, in.bits.data(), &df, filt.bits.data(), &g, &cf, out.bits.data()));
  return out;
}

inline RealTensorPQNO first_conv_bwn(const RealTensorNHWC& x, std::span<const float> weights_pm1, std::size_t kh,
                                     std::size_t kw, std::size_t o, const Conv2dGeometry& geo, int threads = 0) {
  (void)threads;
  geo.validate();
  if (geo.kh != kh || geo.kw != kw) throw invalid_input("first_conv_bwn: geometry kernel does not match filter");
  if (weights_pm1.size() != kh * kw * o * x.channels)
    throw invalid_input("first_conv_bwn: weight count does not match dimensions");
  RealTensorPQNO out(geo.out_h(x.height), geo.out_w(x.width), x.batch, o);
  const auto g = detail::geom(geo);
  detail::check(btnn_cuda_first_conv_bwn(x.v.data(), x.batch, x.height, x.width, x.channels, weights_pm1.data(),
                                         weights_pm1.size(), kh, kw, o, &g, out.v.data()));
  return out;
}

inline BitTensorHWNC or_pool(const BitTensorHWNC& in, std::size_t window, std::size_t stride, int threads = 0) {
  (void)threads;
  if (window == 0 || stride == 0) throw invalid_input("or_pool: zero window or stride");
  if (in.height < window || in.width < window) throw unsupported_shape("or_pool: input smaller than window");
  if ((in.height - window) % stride != 0 || (in.width - window) % stride != 0)
    throw unsupported_shape("or_pool: window placement does not cover the input exactly");
  BitTensorHWNC out((in.height - window) / stride + 1, (in.width - window) / stride + 1, in.batch, in.channels,
                    in.tiled, in.geo);
  const auto di = detail::desc(in);
  detail::check(btnn_cuda_or_pool(&di, in.bits.data(), window, stride, out.bits.data()));
  return out;
}

// ---- format stage (bit_matrix.hpp, tensors.hpp) -----------------------------------------
inline BitMatrix pack_matrix(std::span<const float> values, std::size_t rows, std::size_t cols, Layout layout,
                             FsbGeometry geo = {}) {
  if (values.size() != rows * cols) throw invalid_input("pack_matrix: value count does not match rows*cols");
  BitMatrix out(rows, cols, layout, geo);
  const auto d = detail::desc(out);
  detail::check(btnn_cuda_pack_matrix(values.data(), values.size(), &d, out.data()));
  return out;
}

inline BitTensorHWNC pack_nhwc(const RealTensorNHWC& x, bool tiled = false, FsbGeometry geo = {}) {
  BitTensorHWNC out(x.height, x.width, x.batch, x.channels, tiled, geo);
  detail::check(btnn_cuda_pack_nhwc(x.v.data(), x.batch, x.height, x.width, x.channels, tiled ? 1 : 0, geo.bh, geo.bw,
                                    out.bits.data()));
  return out;
}

inline BitMatrix to_fsb(const BitMatrix& src, FsbGeometry geo = {}) {
  Layout target;
  switch (src.layout()) {
    case Layout::RowPacked: target = Layout::FsbRow; break;
    case Layout::ColPacked: target = Layout::FsbCol; break;
    default: throw invalid_input("to_fsb: source is already tiled");
  }
  BitMatrix out(src.rows(), src.cols(), target, geo);
  const auto d = detail::desc(src);
  detail::check(btnn_cuda_to_fsb(&d, src.data(), geo.bh, geo.bw, out.data()));
  return out;
}

inline BitMatrix from_fsb(const BitMatrix& src) {
  Layout target;
  switch (src.layout()) {
    case Layout::FsbRow: target = Layout::RowPacked; break;
    case Layout::FsbCol: target = Layout::ColPacked; break;
    default: throw invalid_input("from_fsb: source is not tiled");
  }
  BitMatrix out(src.rows(), src.cols(), target);
  const auto d = detail::desc(src);
  detail::check(btnn_cuda_from_fsb(&d, src.data(), out.data()));
  return out;
}

inline BitMatrix flatten_to_matrix(const BitTensorHWNC& t, Layout layout, FsbGeometry geo = {}) {
  BitMatrix out(t.batch, t.height * t.width * t.channels, layout, geo);
  const auto di = detail::desc(t);
  const auto dm = detail::desc(out);
  detail::check(btnn_cuda_flatten_to_matrix(&di, t.bits.data(), &dm, out.data()));
  return out;
}

// ---- model driver (inference.hpp:67-186) --------------------------------------------------
// Holds a device plan for one (ModelSpec, WeightStore): weights converted and uploaded
// once per device, the layer sequence replayed from a CUDA graph; the batch is split
// across `devices` (one shard per GPU, no collective).
class Engine {
 public:
  Engine(const ModelSpec& m, const WeightStore& ws, std::size_t max_batch, std::vector<int> devices = {0})
      : m_(m) {
    if (ws.layers.size() != m.layers.size()) throw invalid_input("run_inference: weight store does not match model");
    for (const auto& l : m.layers) {
      btnn_layer_spec s{};
      s.kind = static_cast<int>(l.kind);
      s.kh = l.kh; s.kw = l.kw; s.out_channels = l.out_channels; s.stride = l.stride; s.pad = l.pad;
      s.window = l.window; s.pool_stride = l.pool_stride; s.units = l.units;
      s.in_h = l.in_h; s.in_w = l.in_w; s.in_channels = l.in_channels; s.out_h = l.out_h; s.out_w = l.out_w;
      s.residual_out = l.residual_out; s.residual_in = l.residual_in; s.shortcut_from = l.shortcut_from;
      specs_.push_back(s);
    }
    const btnn_model_spec spec{m.name.c_str(), m.in_h, m.in_w, m.in_c, m.classes, m.epsilon, specs_.data(), specs_.size()};
    std::vector<btnn_layer_weights> lw(ws.layers.size());
    std::vector<detail::ThresholdArrays> thr;
    thr.reserve(ws.layers.size());
    for (std::size_t i = 0; i < ws.layers.size(); ++i) {
      const LayerWeights& w = ws.layers[i];
      btnn_layer_weights& o = lw[i];
      o = btnn_layer_weights{};
      o.kind = static_cast<int>(w.kind);
      if (w.filter.bits.n_words()) { o.filter_words = w.filter.bits.data(); o.filter_n_words = w.filter.bits.n_words(); }
      if (!w.conv_pm1.empty()) { o.conv_pm1 = w.conv_pm1.data(); o.conv_pm1_n = w.conv_pm1.size(); }
      if (w.fc.rows()) { o.fc_words = w.fc.data(); o.fc_n_words = w.fc.bits().n_words(); }
      thr.emplace_back(w.thresholds);
      o.tau = thr.back().tau.data();
      o.tkind = thr.back().kind.data();
      o.n_thresholds = thr.back().tau.size();
      o.has_bn = w.has_bn ? 1 : 0;
      if (w.has_bn) o.bn = detail::bn_view(w.bn);
    }
    const btnn_weight_store store{ws.tiled ? 1 : 0, ws.geo.bh, ws.geo.bw, lw.data(), lw.size()};
    detail::check(btnn_cuda_plan_create(&spec, &store, max_batch, devices.data(), static_cast<int>(devices.size()),
                                        &plan_));
  }
  ~Engine() {
    if (plan_) btnn_cuda_plan_destroy(plan_);
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  RunResult run(const RealTensorNHWC& input, const RunOptions& opt = {}) {
    if (input.batch == 0) throw invalid_input("run_inference: empty batch");
    if (input.height != m_.in_h || input.width != m_.in_w || input.channels != m_.in_c)
      throw invalid_input("run_inference: input dims do not match model '" + m_.name + "'");
    RunResult res;
    res.batch = input.batch;
    res.classes = m_.classes;
    res.logits.assign(input.batch * m_.classes, 0.0);
    std::vector<std::int32_t> labels(input.batch);
    detail::check(btnn_cuda_plan_set_breakdown(plan_, opt.breakdown ? 1 : 0));
    detail::check(btnn_cuda_plan_run(plan_, input.v.data(), input.batch, res.logits.data(), labels.data()));
    res.labels.assign(labels.begin(), labels.end());
    if (opt.breakdown) {
      std::vector<double> ms(specs_.size());
      detail::check(btnn_cuda_plan_layer_ms(plan_, ms.data(), ms.size()));
      for (std::size_t i = 0; i < ms.size(); ++i) res.timings.push_back({layer_label(m_, i), ms[i]});
    }
    return res;
  }

 private:
  ModelSpec m_;
  std::vector<btnn_layer_spec> specs_;
  btnn_plan* plan_ = nullptr;
};

// One-shot run_inference: plan, run, release. Same validation and results as the
// reference (inference.hpp:67-186).
inline RunResult run_inference(const ModelSpec& m, const WeightStore& ws, const RealTensorNHWC& input,
                               const RunOptions& opt = {}) {
  if (ws.layers.size() != m.layers.size()) throw invalid_input("run_inference: weight store does not match model");
  if (input.batch == 0) throw invalid_input("run_inference: empty batch");
  Engine e(m, ws, input.batch);
  return e.run(input, opt);
}

}  // namespace btnn::cuda
