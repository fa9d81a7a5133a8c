// ref_shim.cpp — TEST INFRASTRUCTURE ONLY. A thin extern "C" wrapper around the
// UNMODIFIED reference btnn headers, compiled where they lie
// (-I/root/reference/proj/include) by oracle/Makefile into oracle/_ref/libbtnn_ref.so.
// Nothing from the reference is copied here: every function forwards to the reference
// implementation (file:line cited) and marshals plain arrays in and out.
//
// Used by: tests (golden fixtures, parity of the C oracle and of the CUDA path against
// the reference itself) and bench.py's --impl reference / cpu_baseline arm (times
// btnn::run_inference on the host cores). The product never loads it.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "btnn/bconv.hpp"
#include "btnn/bit_matrix.hpp"
#include "btnn/bmm.hpp"
#include "btnn/inference.hpp"
#include "btnn/io.hpp"
#include "btnn/layer_math.hpp"
#include "btnn/model.hpp"
#include "btnn/oracle.hpp"
#include "btnn/tensors.hpp"
#include "btnn/weights.hpp"

#include "../include/btnn_cuda.h"

namespace {

thread_local std::string g_err;

template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    g_err.clear();
    return 0;
  } catch (const btnn::invalid_input& e) {
    g_err = e.what();
    return BTNN_INVALID_INPUT;
  } catch (const btnn::unsupported_shape& e) {
    g_err = e.what();
    return BTNN_UNSUPPORTED_SHAPE;
  } catch (const btnn::io_error& e) {
    g_err = e.what();
    return BTNN_IO_ERROR;
  } catch (const btnn::validation_error& e) {
    g_err = e.what();
    return BTNN_VALIDATION_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

btnn::Layout layout_of(int l) { return static_cast<btnn::Layout>(l); }

btnn::BitMatrix make_matrix(const btnn_matrix_desc* d, const uint64_t* words) {
  btnn::BitMatrix m(d->rows, d->cols, layout_of(d->layout), btnn::FsbGeometry{d->bh ? d->bh : 8, d->bw ? d->bw : 128});
  std::memcpy(m.data(), words, m.bits().n_words() * 8);
  return m;
}

btnn::BitTensorHWNC make_act(const btnn_act_desc* d, const uint64_t* words) {
  btnn::BitTensorHWNC t(d->height, d->width, d->batch, d->channels, d->tiled != 0,
                        btnn::FsbGeometry{d->bh ? d->bh : 8, d->bw ? d->bw : 128});
  std::memcpy(t.bits.data(), words, t.bits.n_words() * 8);
  return t;
}

btnn::BitFilterKKOC make_filter(const btnn_filter_desc* d, const uint64_t* words) {
  btnn::BitFilterKKOC f(d->kh, d->kw, d->out_channels, d->in_channels, d->tiled != 0,
                        btnn::FsbGeometry{d->bh ? d->bh : 8, d->bw ? d->bw : 128});
  std::memcpy(f.bits.data(), words, f.bits.n_words() * 8);
  return f;
}

btnn::BmmOptions bmm_opt(int variant, int threads) {
  btnn::BmmOptions o;
  o.variant = static_cast<btnn::BmmVariant>(variant);
  o.threads = threads;
  return o;
}

std::vector<btnn::Threshold> thresholds(const double* tau, const uint8_t* kind, size_t n) {
  std::vector<btnn::Threshold> t(n);
  for (size_t i = 0; i < n; ++i) t[i] = {tau[i], static_cast<btnn::ThresholdKind>(kind[i])};
  return t;
}

btnn::BnParams bn_of(const btnn_bn* b) {
  btnn::BnParams p;
  p.gamma.assign(b->gamma, b->gamma + b->channels);
  p.beta.assign(b->beta, b->beta + b->channels);
  p.mean.assign(b->mean, b->mean + b->channels);
  p.var.assign(b->var, b->var + b->channels);
  p.eps = b->eps;
  return p;
}

struct Model {
  btnn::ModelSpec m;
  std::vector<btnn_layer_spec> specs;
  btnn_model_spec view{};
};

void export_model(Model& h) {
  h.specs.clear();
  for (const auto& l : h.m.layers) {
    btnn_layer_spec s{};
    s.kind = static_cast<int>(l.kind);
    s.kh = l.kh; s.kw = l.kw; s.out_channels = l.out_channels; s.stride = l.stride; s.pad = l.pad;
    s.window = l.window; s.pool_stride = l.pool_stride; s.units = l.units;
    s.in_h = l.in_h; s.in_w = l.in_w; s.in_channels = l.in_channels; s.out_h = l.out_h; s.out_w = l.out_w;
    s.residual_out = l.residual_out; s.residual_in = l.residual_in; s.shortcut_from = l.shortcut_from;
    h.specs.push_back(s);
  }
  h.view.name = h.m.name.c_str();
  h.view.in_h = h.m.in_h; h.view.in_w = h.m.in_w; h.view.in_c = h.m.in_c;
  h.view.classes = h.m.classes; h.view.epsilon = h.m.epsilon;
  h.view.layers = h.specs.data(); h.view.n_layers = h.specs.size();
}

struct Store {
  btnn::WeightStore ws;
  std::vector<btnn_layer_weights> lw;
  std::vector<std::vector<double>> tau;
  std::vector<std::vector<uint8_t>> kind;
  btnn_weight_store view{};
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- models (model.hpp:299-343) ----
void* ref_model_parse_json(const char* text, int* status) {
  auto h = std::make_unique<Model>();
  *status = guard([&] { h->m = btnn::parse_model_text(text); export_model(*h); });
  return *status ? nullptr : h.release();
}
void* ref_make_model(const char* name, const char* tokens, size_t in_h, size_t in_w, size_t in_c,
                     size_t classes, const size_t* sc_from, const size_t* sc_to, size_t n_sc,
                     double epsilon, int* status) {
  auto h = std::make_unique<Model>();
  *status = guard([&] {
    std::vector<btnn::Shortcut> sc;
    for (size_t i = 0; i < n_sc; ++i) sc.push_back({sc_from[i], sc_to[i]});
    h->m = btnn::make_model(name, tokens, in_h, in_w, in_c, classes, sc, epsilon);
    export_model(*h);
  });
  return *status ? nullptr : h.release();
}
const btnn_model_spec* ref_model_view(void* model) { return &static_cast<Model*>(model)->view; }
void ref_model_free(void* model) { delete static_cast<Model*>(model); }

// ---- float weights (weights.hpp:34-73) ----
void* ref_random_weights(void* model, uint64_t seed) {
  return new btnn::FloatWeights(btnn::random_weights(static_cast<Model*>(model)->m, seed));
}
// Float weights from caller arrays: one record per layer (pool records empty).
void* ref_float_weights_new(size_t n_layers) {
  auto* fw = new btnn::FloatWeights();
  fw->layers.resize(n_layers);
  return fw;
}
void ref_float_weights_set(void* fwp, size_t i, const float* w, size_t n, const double* gamma,
                           const double* beta, const double* mean, const double* var, size_t ch, double eps) {
  auto& l = static_cast<btnn::FloatWeights*>(fwp)->layers[i];
  l.weights.assign(w, w + n);
  l.has_bn = ch > 0;
  l.bn.gamma.assign(gamma, gamma + ch);
  l.bn.beta.assign(beta, beta + ch);
  l.bn.mean.assign(mean, mean + ch);
  l.bn.var.assign(var, var + ch);
  l.bn.eps = eps;
}
// Export one record: pointers stay valid while the handle lives.
void ref_float_weights_get(void* fwp, size_t i, const float** w, size_t* n, const double** gamma,
                           const double** beta, const double** mean, const double** var, size_t* ch) {
  auto& l = static_cast<btnn::FloatWeights*>(fwp)->layers[i];
  *w = l.weights.data(); *n = l.weights.size();
  *gamma = l.bn.gamma.data(); *beta = l.bn.beta.data(); *mean = l.bn.mean.data(); *var = l.bn.var.data();
  *ch = l.has_bn ? l.bn.gamma.size() : 0;
}
void ref_float_weights_free(void* fw) { delete static_cast<btnn::FloatWeights*>(fw); }

// ---- weight store (weights.hpp:255-296) ----
void* ref_build_weights(void* model, void* fwp, int tiled, size_t bh, size_t bw, int* status) {
  auto h = std::make_unique<Store>();
  auto& m = static_cast<Model*>(model)->m;
  *status = guard([&] {
    h->ws = btnn::build_weights(m, *static_cast<btnn::FloatWeights*>(fwp), tiled != 0, btnn::FsbGeometry{bh, bw});
    const size_t L = h->ws.layers.size();
    h->lw.resize(L);
    h->tau.resize(L);
    h->kind.resize(L);
    for (size_t i = 0; i < L; ++i) {
      auto& s = h->ws.layers[i];
      auto& o = h->lw[i];
      std::memset(&o, 0, sizeof o);
      o.kind = static_cast<int>(s.kind);
      if (s.filter.bits.n_words()) { o.filter_words = s.filter.bits.data(); o.filter_n_words = s.filter.bits.n_words(); }
      if (!s.conv_pm1.empty()) { o.conv_pm1 = s.conv_pm1.data(); o.conv_pm1_n = s.conv_pm1.size(); }
      if (s.fc.rows()) { o.fc_words = s.fc.data(); o.fc_n_words = s.fc.bits().n_words(); }
      for (auto& t : s.thresholds) { h->tau[i].push_back(t.tau); h->kind[i].push_back(static_cast<uint8_t>(t.kind)); }
      o.tau = h->tau[i].data(); o.tkind = h->kind[i].data(); o.n_thresholds = s.thresholds.size();
      o.has_bn = s.has_bn;
      o.bn.gamma = s.bn.gamma.data(); o.bn.beta = s.bn.beta.data(); o.bn.mean = s.bn.mean.data();
      o.bn.var = s.bn.var.data(); o.bn.channels = s.has_bn ? s.bn.gamma.size() : 0; o.bn.eps = s.bn.eps;
    }
    h->view.tiled = tiled; h->view.bh = bh; h->view.bw = bw;
    h->view.layers = h->lw.data(); h->view.n_layers = L;
  });
  return *status ? nullptr : h.release();
}
const btnn_weight_store* ref_store_view(void* ws) { return &static_cast<Store*>(ws)->view; }
void ref_store_free(void* ws) { delete static_cast<Store*>(ws); }

// ---- files: save_weights (weights.hpp:302-352), write_batch (io.hpp:71-80), and the
// `btnn infer` flow load_weights + read_batch + run_inference (btnn_cli.cpp:69-110) ----
int ref_save_weights(void* model, void* ws, const char* path) {
  return guard([&] { btnn::save_weights(path, static_cast<Model*>(model)->m, static_cast<Store*>(ws)->ws); });
}
int ref_write_batch(const float* x, size_t n, size_t h, size_t w, size_t c, const char* path) {
  return guard([&] {
    btnn::RealTensorNHWC t(n, h, w, c);
    std::memcpy(t.v.data(), x, t.v.size() * sizeof(float));
    btnn::write_batch(path, t);
  });
}
int ref_infer_files(void* model, const char* wpath, int tiled, const char* bpath, size_t max_batch, double* logits,
                    int32_t* labels, size_t* n_out) {
  auto& m = static_cast<Model*>(model)->m;
  return guard([&] {
    const btnn::WeightStore ws = btnn::load_weights(wpath, m, tiled != 0);
    const btnn::RealTensorNHWC in = btnn::read_batch(bpath);
    if (in.batch > max_batch) throw btnn::invalid_input("ref_infer_files: batch larger than the output buffers");
    auto r = btnn::run_inference(m, ws, in, {});
    std::memcpy(logits, r.logits.data(), r.logits.size() * sizeof(double));
    for (size_t i = 0; i < r.labels.size(); ++i) labels[i] = r.labels[i];
    *n_out = in.batch;
  });
}

// ---- inputs: the CLI's seeded N(0,1) floats (btnn_cli.cpp:76-79) ----
void ref_normal_floats(uint64_t seed, float* out, size_t n) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<float> dist(0.0f, 1.0f);
  for (size_t i = 0; i < n; ++i) out[i] = dist(rng);
}
void ref_mt19937_64(uint64_t seed, uint64_t* out, size_t n) {
  std::mt19937_64 rng(seed);
  for (size_t i = 0; i < n; ++i) out[i] = rng();
}

// ---- model driver (inference.hpp:67) and dense oracle (oracle.hpp:176) ----
int ref_run_inference(void* model, void* ws, const float* x, size_t batch, int threads, double* logits,
                      int32_t* labels, double* layer_ms) {
  auto& m = static_cast<Model*>(model)->m;
  return guard([&] {
    btnn::RealTensorNHWC in(batch, m.in_h, m.in_w, m.in_c);
    std::memcpy(in.v.data(), x, in.v.size() * sizeof(float));
    btnn::RunOptions opt;
    opt.threads = threads;
    opt.breakdown = layer_ms != nullptr;
    auto r = btnn::run_inference(m, static_cast<Store*>(ws)->ws, in, opt);
    std::memcpy(logits, r.logits.data(), r.logits.size() * sizeof(double));
    for (size_t i = 0; i < r.labels.size(); ++i) labels[i] = r.labels[i];
    if (layer_ms)
      for (size_t i = 0; i < r.timings.size(); ++i) layer_ms[i] = r.timings[i].ms;
  });
}
int ref_pipeline(void* model, void* fwp, const float* x, size_t batch, double* logits, int32_t* labels) {
  auto& m = static_cast<Model*>(model)->m;
  return guard([&] {
    btnn::RealTensorNHWC in(batch, m.in_h, m.in_w, m.in_c);
    std::memcpy(in.v.data(), x, in.v.size() * sizeof(float));
    auto r = btnn::oracle::ref_pipeline(m, *static_cast<btnn::FloatWeights*>(fwp), in);
    std::memcpy(logits, r.logits.data(), r.logits.size() * sizeof(double));
    for (size_t i = 0; i < r.labels.size(); ++i) labels[i] = r.labels[i];
  });
}

// ---- kernel level ----
size_t ref_matrix_words(const btnn_matrix_desc* d) {
  btnn::BitMatrix m(d->rows, d->cols, layout_of(d->layout), btnn::FsbGeometry{d->bh ? d->bh : 8, d->bw ? d->bw : 128});
  return m.bits().n_words();
}
int ref_pack_matrix(const float* v, size_t n, const btnn_matrix_desc* d, uint64_t* out) {
  return guard([&] {
    auto m = btnn::pack_matrix(std::span<const float>(v, n), d->rows, d->cols, layout_of(d->layout),
                               btnn::FsbGeometry{d->bh ? d->bh : 8, d->bw ? d->bw : 128});
    std::memcpy(out, m.data(), m.bits().n_words() * 8);
  });
}
int ref_to_fsb(const btnn_matrix_desc* d, const uint64_t* w, size_t bh, size_t bw, uint64_t* out) {
  return guard([&] {
    auto m = btnn::to_fsb(make_matrix(d, w), btnn::FsbGeometry{bh, bw});
    std::memcpy(out, m.data(), m.bits().n_words() * 8);
  });
}
int ref_from_fsb(const btnn_matrix_desc* d, const uint64_t* w, uint64_t* out) {
  return guard([&] {
    auto m = btnn::from_fsb(make_matrix(d, w));
    std::memcpy(out, m.data(), m.bits().n_words() * 8);
  });
}
int ref_bmm(int which, const btnn_matrix_desc* a, const uint64_t* aw, const btnn_matrix_desc* b,
            const uint64_t* bw, int variant, int threads, const double* tau, const uint8_t* kind, size_t n_thr,
            void* out) {
  return guard([&] {
    auto A = make_matrix(a, aw);
    auto B = make_matrix(b, bw);
    auto opt = bmm_opt(variant, threads);
    if (which == 0) {
      auto r = btnn::bmm_raw(A, B, opt);
      std::memcpy(out, r.v.data(), r.v.size() * 4);
    } else if (which == 1) {
      auto r = btnn::bmm_pm1(A, B, opt);
      std::memcpy(out, r.v.data(), r.v.size() * 4);
    } else {
      auto t = thresholds(tau, kind, n_thr);
      auto r = btnn::bmm_pm1_bin(A, B, opt, t);
      std::memcpy(out, r.data(), r.bits().n_words() * 8);
    }
  });
}
int ref_pack_nhwc(const float* x, size_t n, size_t h, size_t w, size_t c, int tiled, size_t bh, size_t bw,
                  uint64_t* out) {
  return guard([&] {
    btnn::RealTensorNHWC t(n, h, w, c);
    std::memcpy(t.v.data(), x, t.v.size() * 4);
    auto b = btnn::pack_nhwc(t, tiled != 0, btnn::FsbGeometry{bh, bw});
    std::memcpy(out, b.bits.data(), b.bits.n_words() * 8);
  });
}
int ref_pack_filter(const float* wt, size_t kh, size_t kw, size_t o, size_t c, int tiled, size_t bh, size_t bw,
                    uint64_t* out) {
  return guard([&] {
    auto f = btnn::pack_filter(std::span<const float>(wt, kh * kw * o * c), kh, kw, o, c, tiled != 0,
                               btnn::FsbGeometry{bh, bw});
    std::memcpy(out, f.bits.data(), f.bits.n_words() * 8);
  });
}
int ref_flatten(const btnn_act_desc* d, const uint64_t* w, int layout, size_t bh, size_t bw, uint64_t* out) {
  return guard([&] {
    auto m = btnn::flatten_to_matrix(make_act(d, w), layout_of(layout), btnn::FsbGeometry{bh, bw});
    std::memcpy(out, m.data(), m.bits().n_words() * 8);
  });
}
int ref_convert_activations(const btnn_act_desc* d, const uint64_t* w, int tiled, size_t bh, size_t bw,
                            uint64_t* out) {
  return guard([&] {
    auto t = btnn::convert_activations(make_act(d, w), tiled != 0, btnn::FsbGeometry{bh, bw});
    std::memcpy(out, t.bits.data(), t.bits.n_words() * 8);
  });
}
int ref_bconv_pm1(const btnn_act_desc* in, const uint64_t* iw, const btnn_filter_desc* f, const uint64_t* fw,
                  const btnn_conv_geom* g, int threads, int32_t* out) {
  return guard([&] {
    auto r = btnn::bconv_pm1(make_act(in, iw), make_filter(f, fw), btnn::Conv2dGeometry{g->kh, g->kw, g->stride, g->pad},
                             threads);
    std::memcpy(out, r.v.data(), r.v.size() * 4);
  });
}
int ref_bconv_fused(const btnn_act_desc* in, const uint64_t* iw, const btnn_filter_desc* f, const uint64_t* fw,
                    const btnn_conv_geom* g, const btnn_conv_fused* fu, uint64_t* out) {
  return guard([&] {
    auto A = make_act(in, iw);
    auto F = make_filter(f, fw);
    btnn::Conv2dGeometry geo{g->kh, g->kw, g->stride, g->pad};
    std::vector<btnn::Threshold> thr = thresholds(fu->tau, fu->kind, fu->n_thresholds);
    btnn::BnParams bn;
    btnn::ConvFused cf;
    cf.threads = fu->threads;
    cf.thresholds = thr;
    if (fu->bn) { bn = bn_of(fu->bn); cf.bn = &bn; }
    btnn::RealTensorPQNO rin, rout;
    const size_t P = geo.out_h(in->height), Q = geo.out_w(in->width);
    if (fu->residual_in) {
      rin = btnn::RealTensorPQNO(P, Q, in->batch, f->out_channels);
      std::memcpy(rin.v.data(), fu->residual_in, rin.v.size() * 8);
      cf.residual_in = &rin;
    }
    if (fu->residual_out) cf.residual_out = &rout;
    auto r = btnn::bconv_fused(A, F, geo, cf);
    std::memcpy(out, r.bits.data(), r.bits.n_words() * 8);
    if (fu->residual_out) std::memcpy(fu->residual_out, rout.v.data(), rout.v.size() * 8);
  });
}
int ref_first_conv_bwn(const float* x, size_t n, size_t h, size_t w, size_t c, const float* wpm1, size_t nw,
                       size_t kh, size_t kw, size_t o, const btnn_conv_geom* g, int threads, double* out) {
  return guard([&] {
    btnn::RealTensorNHWC t(n, h, w, c);
    std::memcpy(t.v.data(), x, t.v.size() * 4);
    auto r = btnn::first_conv_bwn(t, std::span<const float>(wpm1, nw), kh, kw, o,
                                  btnn::Conv2dGeometry{g->kh, g->kw, g->stride, g->pad}, threads);
    std::memcpy(out, r.v.data(), r.v.size() * 8);
  });
}
int ref_or_pool(const btnn_act_desc* in, const uint64_t* iw, size_t window, size_t stride, int threads,
                uint64_t* out) {
  return guard([&] {
    auto r = btnn::or_pool(make_act(in, iw), window, stride, threads);
    std::memcpy(out, r.bits.data(), r.bits.n_words() * 8);
  });
}
void ref_fold_bn_sign(double gamma, double beta, double mean, double var, double eps, double* tau, uint8_t* kind) {
  auto t = btnn::fold_bn_sign(gamma, beta, mean, var, eps);
  *tau = t.tau;
  *kind = static_cast<uint8_t>(t.kind);
}
double ref_bn_apply(const btnn_bn* b, size_t ch, double x) { return bn_of(b).apply(ch, x); }

// run_inference (inference.hpp:67) on a model/store given as the C-ABI records — lets
// the tests run the reference on harness-built weights (same bits as the GPU path).
int ref_run_store(const btnn_model_spec* ms, const btnn_weight_store* wsp, const float* x, size_t batch,
                  double* logits, int32_t* labels) {
  return guard([&] {
    btnn::ModelSpec m;
    m.name = ms->name ? ms->name : "";
    m.in_h = ms->in_h; m.in_w = ms->in_w; m.in_c = ms->in_c; m.classes = ms->classes; m.epsilon = ms->epsilon;
    for (size_t i = 0; i < ms->n_layers; ++i) {
      const auto& s = ms->layers[i];
      btnn::LayerSpec l;
      l.kind = static_cast<btnn::LayerKind>(s.kind);
      l.kh = s.kh; l.kw = s.kw; l.out_channels = s.out_channels; l.stride = s.stride; l.pad = s.pad;
      l.window = s.window; l.pool_stride = s.pool_stride; l.units = s.units;
      l.in_h = s.in_h; l.in_w = s.in_w; l.in_channels = s.in_channels; l.out_h = s.out_h; l.out_w = s.out_w;
      l.residual_out = s.residual_out; l.residual_in = s.residual_in; l.shortcut_from = s.shortcut_from;
      m.layers.push_back(l);
    }
    btnn::WeightStore ws;
    ws.tiled = wsp->tiled != 0;
    ws.geo = btnn::FsbGeometry{wsp->bh ? wsp->bh : 8, wsp->bw ? wsp->bw : 128};
    ws.layers.resize(wsp->n_layers);
    for (size_t i = 0; i < wsp->n_layers; ++i) {
      const auto& r = wsp->layers[i];
      const auto& l = m.layers[i];
      auto& o = ws.layers[i];
      o.kind = l.kind;
      if (l.kind == btnn::LayerKind::FirstConvBWN || l.kind == btnn::LayerKind::BitConv) {
        o.filter = btnn::BitFilterKKOC(l.kh, l.kw, l.out_channels, l.in_channels, ws.tiled, ws.geo);
        if (r.filter_words) std::memcpy(o.filter.bits.data(), r.filter_words, o.filter.bits.n_words() * 8);
        if (r.conv_pm1) o.conv_pm1.assign(r.conv_pm1, r.conv_pm1 + r.conv_pm1_n);
      }
      if (l.kind == btnn::LayerKind::BitFc || l.kind == btnn::LayerKind::LastFc) {
        o.fc = btnn::BitMatrix(l.in_channels, l.units, ws.tiled ? btnn::Layout::FsbCol : btnn::Layout::ColPacked, ws.geo);
        std::memcpy(o.fc.data(), r.fc_words, o.fc.bits().n_words() * 8);
      }
      o.thresholds = thresholds(r.tau, r.tkind, r.n_thresholds);
      if (r.has_bn) { o.bn = bn_of(&r.bn); o.has_bn = true; }
    }
    btnn::RealTensorNHWC in(batch, m.in_h, m.in_w, m.in_c);
    std::memcpy(in.v.data(), x, in.v.size() * sizeof(float));
    auto res = btnn::run_inference(m, ws, in, {});
    std::memcpy(logits, res.logits.data(), res.logits.size() * sizeof(double));
    for (size_t i = 0; i < res.labels.size(); ++i) labels[i] = res.labels[i];
  });
}

}  // extern "C"
