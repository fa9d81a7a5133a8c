// dispatch.cu — engine selection for the implicit bit GEMM.
#include "api_internal.cuh"

namespace btnn_gpu {

const char* launch_bgemm(const ConvShape& s, const uint64_t* act, const uint64_t* filt, const Epi& e, cudaStream_t st,
                         EngineHint h, const TcFilter* tc) {
  const bool tc_ok = tc && tc->valid() && tc_supported(s, e);
  if (h == EngineHint::TcI8) require(tc_ok, BTNN_UNSUPPORTED_SHAPE, "tensor-core engine does not cover this shape");
  if (tc_ok && h != EngineHint::Popc) {
    launch_bgemm_tc(s, act, *tc, e, st);
    return "tc_i8";
  }
  launch_bgemm_popc(s, act, filt, e, st);
  return "popc";
}

}  // namespace btnn_gpu
