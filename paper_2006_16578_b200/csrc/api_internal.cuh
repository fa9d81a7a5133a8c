// api_internal.cuh — glue shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <new>
#include <string>
#include <vector>

#include "btnn_cuda.h"
#include "common.cuh"
#include "kernels.cuh"

namespace btnn_gpu {

void set_last_error(const std::string& m);

// Runs fn, mapping exceptions to the C-ABI status codes.
template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    set_last_error("");
    return BTNN_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return BTNN_CUDA_ERROR;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return BTNN_CUDA_ERROR;
  }
}

void check_matrix_desc(const btnn_matrix_desc* d);
void check_act_desc(const btnn_act_desc* d);
void check_filter_desc(const btnn_filter_desc* d);
void check_bn(const btnn_bn& bn);
size_t conv_out(size_t x, size_t k, size_t stride, size_t pad, bool height);
void thresholds_to_int(const double* tau, const uint8_t* kind, size_t n, std::vector<long long>& lo,
                       std::vector<long long>& hi);
void bn_to_device_arrays(const btnn_bn& bn, std::vector<double>& packed);
// Uploads the bn block (bnmath.cuh: mean | s | gamma | beta | reciprocal) and fills the
// reciprocal array on the device.
DevBuf upload_bn(const btnn_bn& bn, cudaStream_t st);
void launch_bn_recip(double* bn, int channels, cudaStream_t st);

// Engine selection for one implicit GEMM. Auto picks the tensor-core path when the shape
// and epilogue are covered by it and an expanded filter is available, else LOP3+POPC.
enum class EngineHint { Auto, Popc, TcI8 };
int engine_override();  // btnn_cuda_set_engine

// Tensor-core operand prepared once per filter (see kernels_tc.cu): +-1 int8 expansion
// of the filter in the UMMA canonical layout, plus per-(tap, o) logical weight sums.
struct TcFilter {
  DevBuf w8;        // int8 operand blocks
  DevBuf wsum;      // int32 [taps][O]
  int O = 0, O_pad = 0, taps = 0, kchunks = 0, n_tile = 0;
  bool valid() const { return w8.get() != nullptr; }
};

// Geometry of one tensor-core launch, chosen per layer shape by measurement (the plan's
// tuner, plan.cu): spt > 0 runs halo mode with that many output sites per tile, tmem_a = 1
// the TMEM-A path, groups the bn route's epilogue groups; {0, 0, 0} is the cost model's
// choice (kernels_tc.cu tc_geom).
struct TcChoice {
  int spt = 0, tmem_a = 0;
  int groups = 0;  // bn route: epilogue groups / TMEM accumulators (2 or 3; 0 = automatic)
};
// The distinct feasible geometries of (s, e), the cost model's own first; "halo/sptN" or
// "tmemA" names them.
std::vector<TcChoice> tc_choices(const ConvShape& s, const Epi& e);
std::string tc_choice_name(const ConvShape& s, const Epi& e, const TcChoice& c);

// Returns the engine name used ("tc_i8" / "popc").
const char* launch_bgemm(const ConvShape& s, const uint64_t* act, const uint64_t* filt, const Epi& e,
                         cudaStream_t st, EngineHint h, const TcFilter* tc = nullptr, const TcChoice* ch = nullptr);

// True when launch_bgemm would pick the tensor-core engine for (s, e).
bool will_use_tc(const ConvShape& s, const Epi& e, EngineHint h, const TcFilter* tc);

// Tensor-core support (kernels_tc.cu).
bool tc_supported(const ConvShape& s, const Epi& e);
void tc_prepare_filter(const ConvShape& s, const uint64_t* filt_plain, TcFilter& out, cudaStream_t st);
bool launch_bgemm_tc(const ConvShape& s, const uint64_t* act, const TcFilter& f, const Epi& e, cudaStream_t st,
                     const TcChoice* ch = nullptr);
// Records a tensor-core first-layer launch for btnn_cuda_last_tc_launch (kernels_first_tc.cu).
void note_first_conv_launch(int mode, int tiles, int grid);
void note_tc_launch(const char* variant, int units, int grid);
// Kernel-level BMM on packed operands in one tcgen05 kernel (bmm_tc.cu): RowPacked a (M x K),
// ColPacked b (N x K), K rounded up to 128 bits <= 1536; EPI_I32 (raw / pm1) or EPI_BITS.
bool bmm_tc_supported(int M, int N, int K);
void launch_bmm_tc(int M, int N, int K, const uint64_t* a, const uint64_t* b, const Epi& e, cudaStream_t st);
// K-pipelined packed BMM for any inner dimension (bmm_tc.cu, bmm_pipe_kernel): same operands
// and epilogues as launch_bmm_tc.
void launch_bmm_pipe(int M, int N, int K, const uint64_t* a, const uint64_t* b, const Epi& e, cudaStream_t st,
                     bool pre_b);
// Either of the two per btnn_cuda_set_bmm_kernel (auto: whole-K when it fits); returns the
// engine name ("tc_i8_bmm" / "tc_i8_bmm_pipe").
const char* launch_bmm_packed(int M, int N, int K, const uint64_t* a, const uint64_t* b, const Epi& e,
                              cudaStream_t st);
// Fully-connected plan layers: a packed kernel when it suits the shape, else nullptr.
const char* launch_bmm_fc(int M, int N, int K, const uint64_t* a, const uint64_t* b, const Epi& e, cudaStream_t st);

}  // namespace btnn_gpu
