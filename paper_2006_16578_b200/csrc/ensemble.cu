// ensemble.cu — BENN combine on the device (the
// paper's BTC-based BENN: K member BNNs classify the same batch and their outputs are
// merged by hard bagging, soft bagging or boosting, Zhu et al. 2019).
//
// Members' outputs sit in one device buffer, member-major (K x B x classes logits, K x B
// labels), as K plan_run_device calls leave them. One thread per (image, class) folds the
// members in member order, so the f64 sums are the left-to-right loop a CPU restatement
// runs (tests/test_ensemble.py) — bit-identical whatever the member count:
//   hard   votes[c]  = #{k : label_k == c}                         (exact, as f64)
//   soft   mean[c]   = ((l_0[c] + l_1[c]) + ... + l_{K-1}[c]) / K
//   boost  score[c]  = sum_k (label_k == c ? alpha_k : 0)           (weighted vote, SAMME)
//   boost_soft score[c] = sum_k alpha_k * l_k[c]                    (each product rounded)
// followed by the first-max label of each row (inference.hpp:177-184 tie rule).
#include <cuda_runtime.h>

#include <cstdint>

#include "api_internal.cuh"

namespace btnn_gpu {

constexpr int kMaxMembers = 64;

struct BennArgs {
  const double* logits;   // K x B x classes
  const int32_t* labels;  // K x B
  int K, B, classes, mode;
  double alpha[kMaxMembers];
  double* scores;   // B x classes
  int32_t* out;     // B
};

__global__ void benn_combine_kernel(const __grid_constant__ BennArgs a) {
  const size_t total = (size_t)a.B * a.classes, stride = (size_t)a.B * a.classes;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / a.classes), c = (int)(i - (size_t)b * a.classes);
    double s = 0.0;
    switch (a.mode) {
      case BTNN_BENN_HARD: {
        int v = 0;
        for (int k = 0; k < a.K; ++k) v += a.labels[(size_t)k * a.B + b] == c;
        s = (double)v;
        break;
      }
      case BTNN_BENN_SOFT:
        s = a.logits[i];
        for (int k = 1; k < a.K; ++k) s = __dadd_rn(s, a.logits[k * stride + i]);
        s = __ddiv_rn(s, (double)a.K);
        break;
      case BTNN_BENN_BOOST:
        for (int k = 0; k < a.K; ++k)
          if (a.labels[(size_t)k * a.B + b] == c) s = __dadd_rn(s, a.alpha[k]);
        break;
      default:  // BTNN_BENN_BOOST_SOFT
        s = __dmul_rn(a.alpha[0], a.logits[i]);
        for (int k = 1; k < a.K; ++k) s = __dadd_rn(s, __dmul_rn(a.alpha[k], a.logits[k * stride + i]));
        break;
    }
    a.scores[i] = s;
  }
}

// First-max label per row (inference.hpp:177-184: best = 0; v[j] > v[best] -> best = j), one
// thread per row so the scan order is the reference's.
__global__ void benn_argmax_kernel(const double* __restrict__ scores, int B, int classes, int32_t* out) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    const double* row = scores + (size_t)b * classes;
    int best = 0;
    double bv = row[0];
    for (int c = 1; c < classes; ++c) {
      const double v = row[c];
      if (v > bv) { bv = v; best = c; }
    }
    out[b] = best;
  }
}

}  // namespace btnn_gpu

using namespace btnn_gpu;

extern "C" int btnn_cuda_benn_combine(const double* d_logits, const int32_t* d_labels, size_t members, size_t batch,
                                      size_t classes, const double* alpha, int mode, double* d_scores,
                                      int32_t* d_out_labels, void* stream) {
  return guard([&] {
    require(members >= 1 && members <= (size_t)kMaxMembers, BTNN_INVALID_INPUT, "benn: 1..64 members");
    require(classes >= 1 && batch < (1u << 30) && classes < (1u << 20), BTNN_INVALID_INPUT, "benn: bad batch / classes");
    require(mode >= BTNN_BENN_HARD && mode <= BTNN_BENN_BOOST_SOFT, BTNN_INVALID_INPUT, "benn: unknown mode");
    const bool needs_logits = mode == BTNN_BENN_SOFT || mode == BTNN_BENN_BOOST_SOFT;
    const bool needs_labels = mode == BTNN_BENN_HARD || mode == BTNN_BENN_BOOST;
    require(!needs_logits || d_logits, BTNN_INVALID_INPUT, "benn: this mode combines logits");
    require(!needs_labels || d_labels, BTNN_INVALID_INPUT, "benn: this mode combines labels");
    require(alpha || mode == BTNN_BENN_HARD || mode == BTNN_BENN_SOFT, BTNN_INVALID_INPUT, "benn: boosting needs alpha");
    require(d_scores && d_out_labels, BTNN_INVALID_INPUT, "benn: null output");
    if (!batch) return;
    BennArgs a{};
    a.logits = d_logits;
    a.labels = d_labels;
    a.K = (int)members;
    a.B = (int)batch;
    a.classes = (int)classes;
    a.mode = mode;
    for (size_t k = 0; k < members; ++k) a.alpha[k] = alpha ? alpha[k] : 1.0;
    a.scores = d_scores;
    a.out = d_out_labels;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t total = batch * classes;
    const unsigned blocks = (unsigned)((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
    benn_combine_kernel<<<blocks, 256, 0, st>>>(a);
    BT_CUDA(cudaGetLastError());
    const unsigned rblocks = (unsigned)((batch + 127) / 128 < 148 * 4 ? (batch + 127) / 128 : 148 * 4);
    benn_argmax_kernel<<<rblocks, 128, 0, st>>>(d_scores, (int)batch, (int)classes, d_out_labels);
    BT_CUDA(cudaGetLastError());
  });
}
