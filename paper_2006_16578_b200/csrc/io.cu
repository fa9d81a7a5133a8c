// io.cu — weight and batch file ingestion for the device plan: the
// reference's BTNN bit-weight files (save_weights / load_weights, weights.hpp:298-445) and
// BTIN batch files (write_batch / read_batch, io.hpp:68-101), parsed on the host with the
// reference's checks and error classes, so `load weights -> read batch -> plan run` is the
// GPU counterpart of `btnn infer` (btnn_cli.cpp:69-110). Files are little-endian (io.hpp:20).
//
// The weight file keeps the writer's layout per layer (tag 0 plain, 1 tiled 8x128); the
// store handed to btnn_cuda_plan_create keeps that layout (the plan converts on upload), so a
// file must use one tag throughout — which save_weights guarantees (ws.tiled is global).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "api_internal.cuh"
#include "layout.cuh"

namespace {

using btnn_gpu::fail;
using btnn_gpu::require;

const char* kind_name(int k) {  // model.hpp:25-33
  switch (k) {
    case BTNN_FIRST_CONV_BWN: return "first_conv";
    case BTNN_BIT_CONV: return "bit_conv";
    case BTNN_OR_POOL: return "or_pool";
    case BTNN_BIT_FC: return "bit_fc";
    case BTNN_LAST_FC: return "last_fc";
    default: return "?";
  }
}

std::string layer_label(const btnn_model_spec& m, size_t i) {  // model.hpp:67-69
  return "layer " + std::to_string(i) + " (" + kind_name(m.layers[i].kind) + ")";
}

bool needs_bn_route(const btnn_layer_spec& l) {  // model.hpp:73-76
  return l.kind == BTNN_FIRST_CONV_BWN || l.kind == BTNN_LAST_FC || l.residual_in || l.residual_out;
}

// binio (io.hpp:19-66): exact-size reads, io_error on a short read.
struct Reader {
  std::ifstream is;
  explicit Reader(const std::string& path) : is(path, std::ios::binary) {
    require((bool)is, BTNN_IO_ERROR, "cannot open " + path);
  }
  void raw(void* p, size_t n) {
    if (!n) return;
    is.read(static_cast<char*>(p), static_cast<std::streamsize>(n));
    require(static_cast<size_t>(is.gcount()) == n, BTNN_IO_ERROR, "unexpected end of file");
  }
  template <class T>
  T pod() {
    T v;
    raw(&v, sizeof v);
    return v;
  }
  void magic(const char* m, const char* what) {
    char got[4];
    raw(got, 4);
    require(std::memcmp(got, m, 4) == 0, BTNN_IO_ERROR, std::string("bad magic, not a ") + what + " file");
  }
};

}  // namespace

// Host copy of a BTNN file in the btnn_weight_store view (all arrays owned here).
struct btnn_loaded_weights {
  std::vector<btnn_layer_weights> layers;
  std::vector<std::vector<uint64_t>> words;
  std::vector<std::vector<float>> pm1;
  std::vector<std::vector<double>> tau, bn;  // bn: gamma | beta | mean | var
  std::vector<std::vector<uint8_t>> tkind;
  btnn_weight_store view{};
};

extern "C" int btnn_cuda_load_weights(const char* path, const btnn_model_spec* m, btnn_loaded_weights** out) {
  return btnn_gpu::guard([&] {
    require(path && m && out, BTNN_INVALID_INPUT, "load_weights: null argument");
    const std::string p(path);
    Reader rd(p);
    rd.magic("BTNN", "bit weight");
    require(rd.pod<uint32_t>() == 1, BTNN_IO_ERROR, p + ": unknown version");
    const uint32_t count = rd.pod<uint32_t>();
    require(count == m->n_layers, BTNN_VALIDATION_ERROR,
            p + ": has " + std::to_string(count) + " layers, model '" + (m->name ? m->name : "") + "' has " +
                std::to_string(m->n_layers));
    auto* lw = new btnn_loaded_weights();
    std::unique_ptr<btnn_loaded_weights> guard_ptr(lw);
    lw->layers.resize(count);
    lw->words.resize(count);
    lw->pm1.resize(count);
    lw->tau.resize(count);
    lw->bn.resize(count);
    lw->tkind.resize(count);
    int tiled = -1;  // the file's layout tag, uniform across weighted layers
    for (size_t i = 0; i < count; ++i) {
      const btnn_layer_spec& l = m->layers[i];
      btnn_layer_weights& w = lw->layers[i];
      std::memset(&w, 0, sizeof w);
      w.kind = l.kind;
      const uint8_t kind = rd.pod<uint8_t>();
      require(kind == (uint8_t)l.kind, BTNN_VALIDATION_ERROR,
              layer_label(*m, i) + ": file record kind " + std::to_string(kind) + " does not match model");
      const bool is_conv = l.kind == BTNN_FIRST_CONV_BWN || l.kind == BTNN_BIT_CONV;
      const bool is_fc = l.kind == BTNN_BIT_FC || l.kind == BTNN_LAST_FC;
      uint32_t d[4] = {0, 0, 0, 0};
      const int nd = is_conv ? 4 : 2;
      for (int k = 0; k < nd; ++k) d[k] = rd.pod<uint32_t>();
      bool dims_ok;
      if (is_conv)
        dims_ok = d[0] == l.kh && d[1] == l.kw && d[2] == l.out_channels && d[3] == l.in_channels;
      else if (is_fc)
        dims_ok = d[0] == l.in_channels && d[1] == l.units;
      else
        dims_ok = d[0] == l.window && d[1] == l.pool_stride;
      require(dims_ok, BTNN_VALIDATION_ERROR, layer_label(*m, i) + ": file dims do not match model");
      const uint8_t stored_tiled = rd.pod<uint8_t>();
      require(stored_tiled <= 1, BTNN_IO_ERROR, p + ": unknown layout tag");
      const uint64_t words = rd.pod<uint64_t>();
      if (is_conv || is_fc) {
        if (tiled < 0) tiled = stored_tiled;
        require(tiled == stored_tiled, BTNN_UNSUPPORTED_SHAPE,
                layer_label(*m, i) + ": mixed plain/tiled layers in one weight file");
        const size_t want = is_conv ? btnn_gpu::filt_words(l.kh, l.kw, l.out_channels, l.in_channels, stored_tiled, 8, 128)
                                    : btnn_gpu::mat_words(l.in_channels, l.units,
                                                          stored_tiled ? BTNN_FSB_COL : BTNN_COL_PACKED, 8, 128);
        require(words == want, BTNN_VALIDATION_ERROR, layer_label(*m, i) + ": unexpected word count");
        lw->words[i].resize(words);
        rd.raw(lw->words[i].data(), words * 8);
        if (is_conv) {
          w.filter_words = lw->words[i].data();
          w.filter_n_words = words;
        } else {
          w.fc_words = lw->words[i].data();
          w.fc_n_words = words;
        }
        if (l.kind == BTNN_FIRST_CONV_BWN) {  // detail::unpack_first_conv (weights.hpp:231-240)
          std::vector<float>& pm = lw->pm1[i];
          pm.resize(l.kh * l.kw * l.out_channels * l.in_channels);
          size_t k = 0;
          for (size_t o = 0; o < l.out_channels; ++o)
            for (size_t r = 0; r < l.kh; ++r)
              for (size_t s = 0; s < l.kw; ++s)
                for (size_t c = 0; c < l.in_channels; ++c, ++k) {
                  const size_t b = btnn_gpu::filt_bit(l.kw, l.out_channels, l.in_channels, stored_tiled, 8, 128, r,
                                                      s, o, c);
                  pm[k] = btnn_gpu::bit_get(lw->words[i].data(), b) ? 1.0f : -1.0f;
                }
          w.conv_pm1 = pm.data();
          w.conv_pm1_n = pm.size();
        }
      } else {
        require(words == 0, BTNN_VALIDATION_ERROR, layer_label(*m, i) + ": pool layer carries weights");
      }
      const uint32_t thr = rd.pod<uint32_t>();
      const size_t out_ch = is_conv ? l.out_channels : (is_fc ? l.units : 0);
      const bool want_thr = !needs_bn_route(l) && l.kind != BTNN_OR_POOL;
      require(want_thr == (thr > 0) && (thr == 0 || thr == out_ch), BTNN_VALIDATION_ERROR,
              layer_label(*m, i) + ": threshold count does not match model");
      if (thr) {
        lw->tau[i].resize(thr);
        lw->tkind[i].resize(thr);
        rd.raw(lw->tau[i].data(), thr * 8);
        rd.raw(lw->tkind[i].data(), thr);
        for (uint8_t k : lw->tkind[i]) require(k <= 3, BTNN_IO_ERROR, p + ": unknown threshold direction");
        w.tau = lw->tau[i].data();
        w.tkind = lw->tkind[i].data();
        w.n_thresholds = thr;
      }
      if (needs_bn_route(l)) {  // gamma, beta, mean, var; BnParams::validate (layer_math.hpp:19-30)
        std::vector<double>& bn = lw->bn[i];
        bn.resize(4 * out_ch);
        rd.raw(bn.data(), bn.size() * 8);
        require(out_ch > 0, BTNN_INVALID_INPUT, "BnParams: channel arrays must be non-empty and equal length");
        require(m->epsilon > 0.0 && std::isfinite(m->epsilon), BTNN_INVALID_INPUT,
                "BnParams: eps must be positive and finite");
        for (size_t c = 0; c < out_ch; ++c) {
          const double g = bn[c], be = bn[out_ch + c], mu = bn[2 * out_ch + c], v = bn[3 * out_ch + c];
          require(std::isfinite(g) && std::isfinite(be) && std::isfinite(mu) && std::isfinite(v) && v >= 0.0,
                  BTNN_INVALID_INPUT, "BnParams: bad values at channel " + std::to_string(c));
        }
        w.has_bn = 1;
        w.bn.gamma = bn.data();
        w.bn.beta = bn.data() + out_ch;
        w.bn.mean = bn.data() + 2 * out_ch;
        w.bn.var = bn.data() + 3 * out_ch;
        w.bn.channels = out_ch;
        w.bn.eps = m->epsilon;
      }
    }
    lw->view.tiled = tiled > 0 ? 1 : 0;
    lw->view.bh = 8;
    lw->view.bw = 128;
    lw->view.layers = lw->layers.data();
    lw->view.n_layers = lw->layers.size();
    *out = guard_ptr.release();
  });
}

extern "C" int btnn_cuda_loaded_weights_store(const btnn_loaded_weights* h, btnn_weight_store* out) {
  return btnn_gpu::guard([&] {
    require(h && out, BTNN_INVALID_INPUT, "loaded_weights_store: null argument");
    *out = h->view;
  });
}

extern "C" int btnn_cuda_free_weights(btnn_loaded_weights* h) {
  delete h;
  return BTNN_OK;
}

// read_batch (io.hpp:83-101): header checks, whole samples only.
extern "C" int btnn_cuda_batch_dims(const char* path, size_t* n, size_t* h, size_t* w, size_t* c) {
  return btnn_gpu::guard([&] {
    require(path && n && h && w && c, BTNN_INVALID_INPUT, "batch_dims: null argument");
    const std::string p(path);
    Reader rd(p);
    rd.is.seekg(0, std::ios::end);
    const auto end = rd.is.tellg();
    require(end >= 0, BTNN_IO_ERROR, "cannot stat " + p);
    rd.is.seekg(0, std::ios::beg);
    const uint64_t fsize = (uint64_t)end;
    rd.magic("BTIN", "batch");
    const uint32_t hh = rd.pod<uint32_t>(), ww = rd.pod<uint32_t>(), cc = rd.pod<uint32_t>();
    require(hh && ww && cc, BTNN_IO_ERROR, p + ": zero dimension");
    require(fsize >= 16, BTNN_IO_ERROR, p + ": truncated header");
    const uint64_t payload = fsize - 16, sample = (uint64_t)hh * ww * cc * sizeof(float);
    require(payload != 0 && payload % sample == 0, BTNN_IO_ERROR, p + ": payload is not a whole number of samples");
    *n = (size_t)(payload / sample);
    *h = hh;
    *w = ww;
    *c = cc;
  });
}

extern "C" int btnn_cuda_read_batch(const char* path, float* out, size_t capacity) {
  return btnn_gpu::guard([&] {
    size_t n, h, w, c;
    const int st = btnn_cuda_batch_dims(path, &n, &h, &w, &c);
    require(st == BTNN_OK, st, btnn_cuda_last_error());
    require(out != nullptr && capacity >= n * h * w * c, BTNN_INVALID_INPUT, "read_batch: output buffer too small");
    Reader rd(path);
    rd.is.seekg(16, std::ios::beg);
    rd.raw(out, n * h * w * c * sizeof(float));
  });
}
