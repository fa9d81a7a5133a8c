// dispatch.cu — engine selection for the implicit bit GEMM.
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "api_internal.cuh"

#include <atomic>

namespace btnn_gpu {

// Initial engine from BTNN_ENGINE=auto|popc|tc (btnn_cuda_set_engine overrides it).
static int engine_from_env() {
  const char* v = std::getenv("BTNN_ENGINE");
  if (v && !std::strcmp(v, "popc")) return BTNN_ENGINE_POPC;
  if (v && !std::strcmp(v, "tc")) return BTNN_ENGINE_TC;
  return BTNN_ENGINE_AUTO;
}
static std::atomic<int> g_engine{engine_from_env()};

int engine_override() { return g_engine.load(); }

static EngineHint resolve(EngineHint h) {
  if (h != EngineHint::Auto) return h;
  const int o = g_engine.load();
  return o == BTNN_ENGINE_POPC ? EngineHint::Popc : o == BTNN_ENGINE_TC ? EngineHint::TcI8 : EngineHint::Auto;
}

bool will_use_tc(const ConvShape& s, const Epi& e, EngineHint h, const TcFilter* tc) {
  h = resolve(h);
  return h != EngineHint::Popc && tc && tc->valid() && tc_supported(s, e);
}

const char* launch_bgemm(const ConvShape& s, const uint64_t* act, const uint64_t* filt, const Epi& e, cudaStream_t st,
                         EngineHint h, const TcFilter* tc, const TcChoice* ch) {
  h = resolve(h);
  const bool tc_ok = tc && tc->valid() && tc_supported(s, e);
  if (h == EngineHint::TcI8) require(tc_ok, BTNN_UNSUPPORTED_SHAPE, "tensor-core engine does not cover this shape");
  require(e.rout_half == nullptr || (tc_ok && h != EngineHint::Popc), BTNN_CUDA_ERROR,
          "halved tap output needs the tensor-core engine");
  if (tc_ok && h != EngineHint::Popc) {
    // fully-connected layers whose inner dimension fits it: the one-kernel packed BMM
    // (bmm_tc.cu) from the RowPacked activations and the ColPacked weights — threshold bits or
    // the last layer's bn logits
    const bool fc = s.P == 1 && s.Q == 1 && s.KH == 1 && s.KW == 1 && s.pad == 0 && !e.rin && !e.rout_half && !e.pool;
    if (fc && ((e.mode == EPI_BITS && !e.bn_mean && e.out_bits) || (e.mode == EPI_F64 && e.bn_mean && e.rout))) {
      if (const char* used = launch_bmm_fc(s.N, s.O, s.C, act, filt, e, st)) return used;
    }
    return launch_bgemm_tc(s, act, *tc, e, st, ch) ? "tc_i8_splitk" : "tc_i8";
  }
  launch_bgemm_popc(s, act, filt, e, st);
  return "popc";
}

}  // namespace btnn_gpu

extern "C" int btnn_cuda_set_engine(int engine) {
  return btnn_gpu::guard([&] {
    btnn_gpu::require(engine >= BTNN_ENGINE_AUTO && engine <= BTNN_ENGINE_TC, BTNN_INVALID_INPUT,
                      "set_engine: unknown engine");
    btnn_gpu::g_engine.store(engine);
  });
}
