// test_adapter.cpp — GPU parity through the C++ drop-in adapter (include/btnn/cuda.hpp):
// for the reference's own test cases, btnn::cuda::f(args) must equal btnn::f(args)
// bit for bit (same value types, same layouts) and throw the same exception classes.
// Built against the unmodified reference headers by oracle/Makefile (target `adapter`)
// into build/test_adapter; run on the GPU box by tests/test_gpu_adapter.py.
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "btnn/bconv.hpp"
#include "btnn/bmm.hpp"
#include "btnn/cuda.hpp"
#include "btnn/inference.hpp"
#include "btnn/oracle.hpp"
#include "btnn/weights.hpp"

using namespace btnn;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond, what)                                              \
  do {                                                                 \
    if (cond) {                                                        \
      ++g_pass;                                                        \
    } else {                                                           \
      ++g_fail;                                                        \
      std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, what); \
    }                                                                  \
  } while (0)
template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static std::vector<float> randn(std::mt19937_64& rng, std::size_t n) {
  std::normal_distribution<float> d(0.0f, 1.0f);
  std::vector<float> v(n);
  for (auto& x : v) x = d(rng);
  return v;
}

static void test_bmm() {  // test_bmm.cpp:41-174
  std::mt19937_64 rng(101);
  const std::size_t shapes[][3] = {{1, 1, 1}, {3, 257, 5}, {8, 1024, 8}, {17, 384, 33}, {5, 100, 7}, {31, 130, 12},
                                   {64, 1024, 1024}, {200, 25088, 512}};
  for (const auto& s : shapes) {
    auto fa = randn(rng, s[0] * s[1]), fb = randn(rng, s[1] * s[2]);
    BitMatrix a = pack_matrix(fa, s[0], s[1], Layout::RowPacked), b = pack_matrix(fb, s[1], s[2], Layout::ColPacked);
    const std::string tag = std::to_string(s[0]) + "x" + std::to_string(s[1]) + "x" + std::to_string(s[2]);
    CHECK(cuda::bmm_pm1(a, b) == bmm_pm1(a, b), ("bmm_pm1 " + tag).c_str());
    if (s[1] % 128 == 0) CHECK(cuda::bmm_raw(a, b) == bmm_raw(a, b), ("bmm_raw " + tag).c_str());
    CHECK(cuda::bmm_pm1_bin(a, b).bits() == bmm_pm1_bin(a, b).bits(), ("bmm_pm1_bin " + tag).c_str());
    std::vector<Threshold> thr(s[2]);
    for (std::size_t j = 0; j < s[2]; ++j)
      thr[j] = {double(int(j % 7) - 3) + 0.5 * (j % 2), static_cast<ThresholdKind>(j % 4)};
    CHECK(cuda::bmm_pm1_bin(a, b, {}, thr).bits() == bmm_pm1_bin(a, b, {}, thr).bits(), ("bin thr " + tag).c_str());
    BitMatrix af = to_fsb(a), bf = to_fsb(b);
    CHECK(cuda::to_fsb(a).bits() == af.bits(), ("to_fsb " + tag).c_str());
    CHECK(cuda::from_fsb(bf).bits() == b.bits(), ("from_fsb " + tag).c_str());
    BmmOptions fsb{.variant = BmmVariant::Fsb};
    CHECK(cuda::bmm_pm1(af, bf, fsb) == bmm_pm1(af, bf, fsb), ("fsb pm1 " + tag).c_str());
    CHECK(cuda::bmm_pm1_bin(af, bf, fsb, thr).bits() == bmm_pm1_bin(af, bf, fsb, thr).bits(), ("fsb bin " + tag).c_str());
  }
  BitMatrix a = pack_matrix(randn(rng, 4 * 128), 4, 128, Layout::RowPacked);
  BitMatrix bshort = pack_matrix(randn(rng, 64 * 4), 64, 4, Layout::ColPacked);
  CHECK(throws<invalid_input>([&] { cuda::bmm_pm1(a, bshort); }), "bmm dim mismatch -> invalid_input");
  BitMatrix b = pack_matrix(randn(rng, 128 * 4), 128, 4, Layout::ColPacked);
  CHECK(throws<invalid_input>([&] { cuda::bmm_pm1(to_fsb(a), b, {.variant = BmmVariant::Fsb}); }), "fsb layout");
  CHECK(throws<unsupported_shape>([&] { cuda::bmm_pm1(to_fsb(a), to_fsb(b, {4, 64}), {.variant = BmmVariant::Fsb}); }),
        "tile geometry mismatch -> unsupported_shape");
  CHECK(throws<invalid_input>([&] { cuda::bmm_pm1(a, b, {.variant = BmmVariant::Blocked, .blocking = {8, 8, 100}}); }),
        "bad blocking -> invalid_input");
  BitMatrix a200 = pack_matrix(randn(rng, 4 * 200), 4, 200, Layout::RowPacked);
  BitMatrix b200 = pack_matrix(randn(rng, 200 * 4), 200, 4, Layout::ColPacked);
  CHECK(throws<unsupported_shape>([&] { cuda::bmm_raw(a200, b200); }), "bmm_raw K%128 -> unsupported_shape");
}

static void test_bconv() {  // test_bconv.cpp:59-283
  std::mt19937_64 rng(201);
  struct Case { std::size_t h, w, n, c, o, k, s, p; };
  const Case cases[] = {{8, 8, 3, 64, 32, 3, 1, 1},  {7, 9, 2, 130, 5, 3, 1, 1}, {8, 8, 1, 128, 128, 3, 2, 1},
                        {5, 5, 2, 16, 8, 5, 2, 2},   {4, 4, 2, 32, 16, 1, 1, 0}, {6, 6, 16, 128, 16, 3, 1, 0},
                        {9, 9, 2, 3, 4, 7, 4, 3},    {14, 14, 16, 256, 256, 3, 1, 1}, {28, 28, 8, 64, 128, 3, 2, 1}};
  for (const auto& cs : cases) {
    RealTensorNHWC x(cs.n, cs.h, cs.w, cs.c);
    x.v = randn(rng, x.v.size());
    auto wt = randn(rng, cs.k * cs.k * cs.o * cs.c);
    const Conv2dGeometry geo{cs.k, cs.k, cs.s, cs.p};
    BnParams bn;
    std::normal_distribution<double> nd(0.0, 1.0);
    for (std::size_t i = 0; i < cs.o; ++i) {
      bn.gamma.push_back(i % 7 == 0 ? 0.0 : nd(rng));
      bn.beta.push_back(nd(rng));
      bn.mean.push_back(nd(rng) * 10.0);
      bn.var.push_back(1.0 + 0.5 * nd(rng) * nd(rng));
      if (bn.var.back() < 0) bn.var.back() = -bn.var.back();
    }
    const auto thr = fold_bn_sign(bn);
    for (bool tiled : {false, true}) {
      const std::string tag = std::to_string(cs.h) + "x" + std::to_string(cs.c) + "->" + std::to_string(cs.o) +
                              (tiled ? " fsb" : " plain");
      BitTensorHWNC in = pack_nhwc(x, tiled);
      BitFilterKKOC f = pack_filter(wt, cs.k, cs.k, cs.o, cs.c, tiled);
      CHECK(cuda::pack_nhwc(x, tiled).bits == in.bits, ("pack_nhwc " + tag).c_str());
      CHECK(cuda::bconv_pm1(in, f, geo) == bconv_pm1(in, f, geo), ("bconv_pm1 " + tag).c_str());
      CHECK(cuda::bconv_fused(in, f, geo, {.thresholds = thr}).bits == bconv_fused(in, f, geo, {.thresholds = thr}).bits,
            ("fused thr " + tag).c_str());
      RealTensorPQNO t1, t2, u1, u2;
      auto b1 = bconv_fused(in, f, geo, {.bn = &bn, .residual_out = &t1});
      auto b2 = cuda::bconv_fused(in, f, geo, {.bn = &bn, .residual_out = &t2});
      CHECK(b1.bits == b2.bits && t1.v == t2.v, ("fused bn tap " + tag).c_str());
      auto c1 = bconv_fused(in, f, geo, {.bn = &bn, .residual_in = &t1, .residual_out = &u1});
      auto c2 = cuda::bconv_fused(in, f, geo, {.bn = &bn, .residual_in = &t1, .residual_out = &u2});
      CHECK(c1.bits == c2.bits && u1.v == u2.v, ("fused residual " + tag).c_str());
      if (cs.h % 2 == 0 && cs.w % 2 == 0)
        CHECK(cuda::or_pool(in, 2, 2).bits == or_pool(in, 2, 2).bits, ("or_pool " + tag).c_str());
      CHECK(cuda::flatten_to_matrix(in, tiled ? Layout::FsbRow : Layout::RowPacked).bits() ==
                flatten_to_matrix(in, tiled ? Layout::FsbRow : Layout::RowPacked).bits(),
            ("flatten " + tag).c_str());
    }
  }
  BitTensorHWNC in(4, 4, 1, 16);
  BitFilterKKOC f(3, 3, 8, 16), ft(3, 3, 8, 16, true);
  CHECK(throws<invalid_input>([&] { cuda::bconv_fused(in, f, {3, 3, 1, 1}, {}); }), "neither rule -> invalid_input");
  CHECK(throws<invalid_input>([&] { cuda::bconv_pm1(in, ft, {3, 3, 1, 1}); }), "mixed layouts -> invalid_input");
  CHECK(throws<invalid_input>([&] { cuda::bconv_pm1(in, f, {5, 5, 1, 1}); }), "kernel mismatch -> invalid_input");
  BitTensorHWNC tiny(1, 1, 1, 8);
  CHECK(throws<unsupported_shape>([&] { cuda::or_pool(tiny, 2, 2); }), "or_pool tiny -> unsupported_shape");
  // first conv (test_bconv.cpp:187-210) at the ResNet-18 and AlexNet geometries
  for (auto [k, s, p, o, hw] : {std::tuple<int, int, int, int, int>{7, 4, 3, 64, 60}, {11, 4, 5, 128, 60}, {5, 2, 2, 12, 9}}) {
    RealTensorNHWC x(3, hw, hw, 3);
    x.v = randn(rng, x.v.size());
    std::vector<float> w(std::size_t(k) * k * o * 3);
    for (auto& v : w) v = (rng() & 1) ? 1.0f : -1.0f;
    const Conv2dGeometry geo{std::size_t(k), std::size_t(k), std::size_t(s), std::size_t(p)};
    CHECK(cuda::first_conv_bwn(x, w, k, k, o, geo).v == first_conv_bwn(x, w, k, k, o, geo).v, "first_conv_bwn");
  }
}

static void test_models() {  // test_nn.cpp:266-364
  struct M { const char* name; const char* tok; std::size_t h, w, c, classes; std::vector<Shortcut> sc; std::uint64_t seed; std::size_t batch; };
  const M models[] = {
      {"cpf", "6C3-P2-12FC", 8, 8, 2, 4, {}, 101, 5},
      {"strided", "8C5/2-8C3-16FC", 16, 16, 3, 5, {}, 103, 4},
      {"mlp", "3x24FC", 4, 4, 1, 10, {}, 107, 9},
      {"headless", "6C3-P2", 8, 8, 2, 4, {}, 109, 6},
      {"res-a", "4C3-4C3-4C3-8FC", 8, 8, 2, 3, {{0, 2}}, 113, 5},
      {"res-b", "4C3-4C3-4C3-8C3/2-8C3-8C3", 8, 8, 2, 3, {{0, 2}, {2, 4}}, 127, 4},
      {"resnet18", "64C7/4-4x64C3-128C3/2-3x128C3-256C3/2-3x256C3-512C3/2-3x512C3-(2x512FC)", 224, 224, 3, 1000,
       {{0, 2}, {2, 4}, {4, 6}, {6, 8}, {8, 10}, {10, 12}, {12, 14}, {14, 16}}, 131, 4},
      {"alexnet", "(128C11/4)-P2-(256C5)-P2-(3x256C3)-P2-(3x4096FC)", 224, 224, 3, 1000, {}, 137, 2},
      {"cifar-vgg", "(2x128C3)-MP2-(2x256C3)-MP2-(2x512C3)-MP2-(3x1024FC)", 32, 32, 3, 10, {}, 139, 16},
      {"mnist-mlp", "1024FC-1024FC-1024FC-1024FC", 28, 28, 1, 10, {}, 149, 64},
  };
  for (const auto& d : models) {
    auto m = make_model(d.name, d.tok, d.h, d.w, d.c, d.classes, d.sc);
    const auto fw = random_weights(m, d.seed * 77 + 1);
    std::mt19937_64 rng(d.seed);
    RealTensorNHWC x(d.batch, d.h, d.w, d.c);
    x.v = randn(rng, x.v.size());
    for (bool tiled : {false, true}) {
      const auto ws = build_weights(m, fw, tiled);
      const auto want = run_inference(m, ws, x);
      const auto got = cuda::run_inference(m, ws, x);
      CHECK(got.logits == want.logits && got.labels == want.labels,
            (std::string("run_inference ") + d.name + (tiled ? " fsb" : " plain")).c_str());
      if (std::string(d.name) == "cpf" && !tiled) {
        cuda::Engine e(m, ws, 8, {0, 0});  // two shards on one device: batch split
        const auto r2 = e.run(x, {.breakdown = true});
        CHECK(r2.logits == want.logits && r2.timings.size() == m.layers.size(), "sharded engine + breakdown");
      }
    }
  }
  auto m = make_model("bad", "4C3-8FC", 8, 8, 2, 3);
  const auto ws = build_weights(m, random_weights(m, 67), false);
  RealTensorNHWC wrong(2, 4, 4, 2), nan_in(1, 8, 8, 2);
  nan_in.v[7] = std::nanf("");
  CHECK(throws<invalid_input>([&] { cuda::run_inference(m, ws, wrong); }), "wrong dims -> invalid_input");
  CHECK(throws<invalid_input>([&] { cuda::run_inference(m, ws, nan_in); }), "non-finite -> invalid_input");
}

int main(int argc, char** argv) {
  const std::string only = argc > 1 ? argv[1] : "";
  if (only.empty() || only == "bmm") test_bmm();
  if (only.empty() || only == "bconv") test_bconv();
  if (only.empty() || only == "models") test_models();
  std::printf("adapter parity: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
