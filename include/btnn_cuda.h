/*
 * btnn_cuda.h — C ABI of libbtnn_cuda.so, the B200 (sm_100a) implementation of the
 * btnn binarized-network hot path (arXiv 2006.16578, BTC-BNN).
 *
 * The reference (`/root/reference/proj/include/btnn`) is a header-only C++20 library
 * with no FFI; its public surface is the C++ layer/model API. Every entry point below
 * replaces exactly one of those functions, takes plain pointers and sizes in the
 * reference's own bit layouts (LSB-first uint64 words, plain/fsb, HWNC/KKOC/PQNO), and
 * returns a status code that mirrors the reference's exception taxonomy
 * (common.hpp:14-32). Host buffers in, host buffers out, synchronous — like the
 * reference calls. The C++ drop-in adapter `include/btnn/cuda.hpp` marshals the
 * reference value types onto these calls and re-throws the same exception types.
 *
 * Each function cites the reference interface it replaces (file:line, relative to
 * proj/include/btnn/).
 */
#ifndef BTNN_CUDA_H_
#define BTNN_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BTNN_CUDA_ABI_VERSION 1

/* Status codes: 0 ok; 1..4 = the reference's four exception types (common.hpp:14-32). */
enum {
  BTNN_OK = 0,
  BTNN_INVALID_INPUT = 1,     /* btnn::invalid_input      (common.hpp:14) */
  BTNN_UNSUPPORTED_SHAPE = 2, /* btnn::unsupported_shape  (common.hpp:19) */
  BTNN_IO_ERROR = 3,          /* btnn::io_error           (common.hpp:24) */
  BTNN_VALIDATION_ERROR = 4,  /* btnn::validation_error   (common.hpp:29) */
  BTNN_CUDA_ERROR = 5         /* device / driver failure (no reference analog) */
};

/* Matrix layouts (bit_matrix.hpp:21). */
enum { BTNN_ROW_PACKED = 0, BTNN_COL_PACKED = 1, BTNN_FSB_ROW = 2, BTNN_FSB_COL = 3 };
/* BMM variants (bmm.hpp:40). On the GPU the variant only selects operand validation. */
enum { BTNN_BMM_NAIVE = 0, BTNN_BMM_BLOCKED = 1, BTNN_BMM_FSB = 2 };
/* Threshold kinds (layer_math.hpp:38). */
enum { BTNN_GEQ = 0, BTNN_LEQ = 1, BTNN_CONST_PLUS = 2, BTNN_CONST_MINUS = 3 };
/* Layer kinds (model.hpp:17-23). */
enum { BTNN_FIRST_CONV_BWN = 0, BTNN_BIT_CONV = 1, BTNN_OR_POOL = 2, BTNN_BIT_FC = 3, BTNN_LAST_FC = 4 };

/* BitMatrix shape (bit_matrix.hpp:61-132). bh/bw: FsbGeometry (:36), ignored for packed layouts. */
typedef struct {
  size_t rows, cols;
  int layout;
  size_t bh, bw;
} btnn_matrix_desc;

/* BmmOptions (bmm.hpp:49-53) incl. BmmBlocking (:43-47). threads is accepted and ignored. */
typedef struct {
  int variant;
  size_t blk_rows, blk_cols, blk_k_bits;
  int threads;
} btnn_bmm_options;

/* BitTensorHWNC shape (tensors.hpp:71-114). */
typedef struct {
  size_t height, width, batch, channels;
  int tiled;
  size_t bh, bw;
} btnn_act_desc;

/* BitFilterKKOC shape (tensors.hpp:119-159). */
typedef struct {
  size_t kh, kw, out_channels, in_channels;
  int tiled;
  size_t bh, bw;
} btnn_filter_desc;

/* Conv2dGeometry (tensors.hpp:240-258). */
typedef struct {
  size_t kh, kw, stride, pad;
} btnn_conv_geom;

/* BnParams (layer_math.hpp:13-35): per-channel f64 arrays. */
typedef struct {
  const double *gamma, *beta, *mean, *var;
  size_t channels;
  double eps;
} btnn_bn;

/* ConvFused (bconv.hpp:152-158). Exactly one of (thresholds, bn). Residual tensors are
 * RealTensorPQNO values, p*q*batch*o doubles; residual_out is overwritten. */
typedef struct {
  const double* tau;        /* Threshold::tau, n_thresholds entries (or NULL) */
  const uint8_t* kind;      /* Threshold::kind */
  size_t n_thresholds;
  const btnn_bn* bn;        /* or NULL */
  const double* residual_in;
  double* residual_out;
  int threads;
} btnn_conv_fused;

/* ---- library ---------------------------------------------------------------------- */
int btnn_cuda_abi_version(void);
/* Message of the last failing call on this host thread ("" if none). */
const char* btnn_cuda_last_error(void);
int btnn_cuda_device_count(int* n);
/* Device used by the kernel-level calls issued from this host thread (default 0). */
int btnn_cuda_set_device(int device);
/* Bit-GEMM engine for subsequent BMM/BConv launches (process-wide): 0 = auto (tcgen05
 * kind::i8 tensor cores where the shape is covered, else CUDA-core LOP3+POPC),
 * 1 = force LOP3+POPC, 2 = force tensor cores (fails with BTNN_UNSUPPORTED_SHAPE when
 * a shape is not covered). Plans bind the engine when their graph is captured. */
enum { BTNN_ENGINE_AUTO = 0, BTNN_ENGINE_POPC = 1, BTNN_ENGINE_TC = 2 };
int btnn_cuda_set_engine(int engine);
/* Packed-operand BMM kernel for bmm_pm1 / bmm_raw / bmm_pm1_bin and fully-connected plan layers
 * (process-wide): 0 = auto (whole-K on-chip kernel when K <= 1536, else K-pipelined),
 * 1 = whole-K (fails with BTNN_UNSUPPORTED_SHAPE when K > 1536), 2 = K-pipelined, 3 = K-pipelined
 * with B always expanded inside the GEMM (the variant plan layers use; for tests). */
enum { BTNN_BMM_AUTO = 0, BTNN_BMM_WHOLE_K = 1, BTNN_BMM_PIPELINED = 2, BTNN_BMM_PIPELINED_NO_PRE = 3 };
int btnn_cuda_set_bmm_kernel(int which);

/* ---- storage sizes (words of uint64) --------------------------------------------- */
size_t btnn_cuda_matrix_words(const btnn_matrix_desc* d);     /* BitMatrix::storage_bits/64 */
size_t btnn_cuda_act_words(const btnn_act_desc* d);           /* BitTensorHWNC bits */
size_t btnn_cuda_filter_words(const btnn_filter_desc* d);     /* BitFilterKKOC bits */

/* ---- format stage ---------------------------------------------------------------- */
/* pack_matrix (bit_matrix.hpp:135-155): sign-binarize row-major floats (x >= 0 -> 1). */
int btnn_cuda_pack_matrix(const float* values, size_t n_values, const btnn_matrix_desc* out_desc,
                          uint64_t* out_words);
/* pack_nhwc (tensors.hpp:162-174): NHWC floats -> HWNC bits. */
int btnn_cuda_pack_nhwc(const float* x, size_t batch, size_t height, size_t width, size_t channels,
                        int tiled, size_t bh, size_t bw, uint64_t* out_words);
/* to_fsb / from_fsb (bit_matrix.hpp:224-253). out_desc gives the target geometry. */
int btnn_cuda_to_fsb(const btnn_matrix_desc* src, const uint64_t* src_words, size_t bh, size_t bw,
                     uint64_t* out_words);
int btnn_cuda_from_fsb(const btnn_matrix_desc* src, const uint64_t* src_words, uint64_t* out_words);
/* convert_activations (tensors.hpp:203-212). */
int btnn_cuda_convert_activations(const btnn_act_desc* src, const uint64_t* src_words, int tiled,
                                  size_t bh, size_t bw, uint64_t* out_words);
/* flatten_to_matrix (tensors.hpp:226-237). */
int btnn_cuda_flatten_to_matrix(const btnn_act_desc* src, const uint64_t* src_words,
                                const btnn_matrix_desc* out_desc, uint64_t* out_words);

/* ---- BMM (bmm.hpp:204-274) ------------------------------------------------------- */
/* bmm_raw (bmm.hpp:204-214): out = xor-popcount accumulators, a.rows x b.cols int32. */
int btnn_cuda_bmm_raw(const btnn_matrix_desc* a, const uint64_t* a_words, const btnn_matrix_desc* b,
                      const uint64_t* b_words, const btnn_bmm_options* opt, int32_t* out);
/* bmm_pm1 (bmm.hpp:219-228): out = n - 2*acc. */
int btnn_cuda_bmm_pm1(const btnn_matrix_desc* a, const uint64_t* a_words, const btnn_matrix_desc* b,
                      const uint64_t* b_words, const btnn_bmm_options* opt, int32_t* out);
/* bmm_pm1_bin (bmm.hpp:256-274): thresholded bits; output layout follows A's family
 * (RowPacked, or FsbRow with A's geometry). n_thresholds == 0 -> plain sign rule. */
int btnn_cuda_bmm_pm1_bin(const btnn_matrix_desc* a, const uint64_t* a_words,
                          const btnn_matrix_desc* b, const uint64_t* b_words,
                          const btnn_bmm_options* opt, const double* tau, const uint8_t* kind,
                          size_t n_thresholds, uint64_t* out_words);

/* ---- BConv (bconv.hpp:138-272) --------------------------------------------------- */
/* bconv_pm1 (bconv.hpp:138-146): IntTensorPQNO p*q*batch*o. */
int btnn_cuda_bconv_pm1(const btnn_act_desc* in, const uint64_t* in_words, const btnn_filter_desc* f,
                        const uint64_t* f_words, const btnn_conv_geom* geo, int32_t* out);
/* bconv_fused (bconv.hpp:160-194): packed HWNC bits in the input's layout. */
int btnn_cuda_bconv_fused(const btnn_act_desc* in, const uint64_t* in_words,
                          const btnn_filter_desc* f, const uint64_t* f_words,
                          const btnn_conv_geom* geo, const btnn_conv_fused* fused,
                          uint64_t* out_words);
/* first_conv_bwn (bconv.hpp:198-243): weights_pm1 is (o, r, s, c) ordered +-1 floats. */
int btnn_cuda_first_conv_bwn(const float* x, size_t batch, size_t height, size_t width,
                             size_t channels, const float* weights_pm1, size_t n_weights,
                             size_t kh, size_t kw, size_t out_channels, const btnn_conv_geom* geo,
                             double* out);
/* or_pool (bconv.hpp:247-272). */
int btnn_cuda_or_pool(const btnn_act_desc* in, const uint64_t* in_words, size_t window,
                      size_t stride, uint64_t* out_words);

/* Describes the last tensor-core kernel launched from this host thread (kernel-level
 * calls, or plans while their graph is captured): the kernel variant ("halo" or "tmemA",
 * then "/thr", "/bn", "/i32" or "/split", plus "/pg2", "/blocked", "/bres" when they apply;
 * "first_conv/stride4" or "first_conv/stride1" for the exact tensor-core first layer),
 * the number of (tile, K-split) work units and the persistent grid size. Tests use it to
 * prove which kernel path and how many tiles per CTA a case exercised. */
int btnn_cuda_last_tc_launch(char* variant, size_t n, int* units, int* grid);

/* Timing experiments only (builds with -DBTNN_TIMING=1): copies the per-K-step clock64
 * stamps recorded by CTA 0 of the last tensor-core GEMM launched with BTNN_TC_DBG & 16
 * (n <= 4096 entries). */
int btnn_cuda_debug_tc_timestamps(unsigned long long* out, size_t n);

/* Timing experiments only (BTNN_TIMING builds): per-tile clock64 stamps of CTA 0 of the last tensor-core first
 * layer launched with BTNN_FTC_DBG=1 (n <= 512 entries, 8 per tile). */
int btnn_cuda_debug_ftc_timestamps(unsigned long long* out, size_t n);

/* Self-test of the bn-route division (csrc/bnmath.cuh): fast[i] = a[i]/b[i] through the
 * per-channel-reciprocal path, ref[i] = __ddiv_rn(a[i], b[i]); host buffers of n doubles. */
int btnn_cuda_selftest_div(const double* a, const double* b, size_t n, double* fast, double* ref);

/* ---- benchmark suites (bench.hpp:129-299), device-timed ---------------------------- */
/* Optional readback of a suite run, for the reference-style precheck (bench.hpp:164-176,
 * 248-256): after timing, the device operands and the last result are copied to these host
 * buffers (any may be NULL). bmm: a = n x n RowPacked A words, b = ColPacked B words,
 * out = int32 n x n (bmm) or RowPacked bits (bmm-bin). bconv: a = packed HWNC input words,
 * b = plain KKOC filter words, out = int32 PQNO (bconv) or HWNC bits (bconv-bin).
 * kernel_ns (bmm only) receives the GEMM alone with B already expanded, and stream_ns the
 * whole call, each averaged over `reps` launches back to back between two events (the host
 * launch cost overlapped, as in a stream of calls); graph_ns the whole call with `reps` calls
 * captured in one CUDA graph and replayed (device time per call, no host launch in it). */
typedef struct {
  uint64_t* a_words;
  uint64_t* b_words;
  void* out;
  double* kernel_ns;
  double* stream_ns;
  double* graph_ns;
} btnn_bench_readback;
/* bench_bmm: n x n x n on random packed +-1 words (bench.hpp:76-87, 136-137); bin = 0 ->
 * "bmm" (bmm_pm1, int32 out), bin = 1 -> "bmm-bin" (bmm_pm1_bin sign rule, bit output).
 * Every repetition is the whole call from packed operands (B's tensor-core expansion
 * included). Median/min of `reps` CUDA-event-timed repetitions after `warmup`. `engine`
 * receives the engine name. Throughput = 2n^3 / median (bench.hpp:207-209). */
int btnn_cuda_bench_bmm(size_t n, int bin, int reps, int warmup, double* median_ns, double* min_ns, char* engine,
                        size_t engine_len, const btnn_bench_readback* rb);
/* bench_bconv: input_hw x input_hw x batch x c -> o, k x k kernel, stride 1, pad k/2;
 * bin = 0 -> "bconv" (binarize + bconv_pm1), bin = 1 -> "bconv-bin" (bconv_fused with sign
 * thresholds, bench.hpp:238). Throughput = 2*P*Q*N*C*O*K^2 / median (bench.hpp:290-292). */
int btnn_cuda_bench_bconv(size_t input_hw, size_t batch, size_t c, size_t o, size_t k, int bin, int reps, int warmup,
                          double* median_ns, double* min_ns, char* engine, size_t engine_len,
                          const btnn_bench_readback* rb);
/* The same suites on fsb-layout operands (8 x 128 tiles; the reference's "fsb" rows,
 * bench.hpp:140-156, 230-245): the tiled operands are converted on the device inside every
 * timed call (and a bit result back to tiles). Readback buffers receive the plain forms. */
int btnn_cuda_bench_bmm_fsb(size_t n, int bin, int reps, int warmup, double* median_ns, double* min_ns, char* engine,
                            size_t engine_len, const btnn_bench_readback* rb);
int btnn_cuda_bench_bconv_fsb(size_t input_hw, size_t batch, size_t c, size_t o, size_t k, int bin, int reps,
                              int warmup, double* median_ns, double* min_ns, char* engine, size_t engine_len,
                              const btnn_bench_readback* rb);

/* ---- model driver (inference.hpp:67-186) ----------------------------------------- */
/* LayerSpec (model.hpp:36-52), already resolved (resolve_model, model.hpp:190-296). */
typedef struct {
  int kind;
  size_t kh, kw, out_channels, stride, pad;
  size_t window, pool_stride;
  size_t units;
  size_t in_h, in_w, in_channels;
  size_t out_h, out_w;
  int residual_out, residual_in, shortcut_from;
} btnn_layer_spec;

/* ModelSpec (model.hpp:58-65). */
typedef struct {
  const char* name;
  size_t in_h, in_w, in_c, classes;
  double epsilon;
  const btnn_layer_spec* layers;
  size_t n_layers;
} btnn_model_spec;

/* LayerWeights (weights.hpp:213-221), in the store's layout. */
typedef struct {
  int kind;
  const uint64_t* filter_words; size_t filter_n_words;   /* conv kinds: BitFilterKKOC bits */
  const float* conv_pm1; size_t conv_pm1_n;              /* first conv: (o,r,s,c) +-1 floats */
  const uint64_t* fc_words; size_t fc_n_words;           /* fc kinds: BitMatrix in x out, ColPacked/FsbCol */
  const double* tau; const uint8_t* tkind; size_t n_thresholds;
  int has_bn;
  btnn_bn bn;
} btnn_layer_weights;

/* WeightStore (weights.hpp:223-227). */
typedef struct {
  int tiled;
  size_t bh, bw;
  const btnn_layer_weights* layers;
  size_t n_layers;
} btnn_weight_store;

typedef struct btnn_plan btnn_plan;

/* ---- file ingestion -------------------------------------------- */
/* load_weights (weights.hpp:354-445): a BTNN bit-weight file for `model`, with the
 * reference's checks (magic/version/tags -> BTNN_IO_ERROR; layer count, kinds, dims, word
 * and threshold counts -> BTNN_VALIDATION_ERROR; BnParams::validate -> BTNN_INVALID_INPUT).
 * The store keeps the file's layout (plain, or tiled 8x128); the first conv's +-1 floats
 * are unpacked from its filter bits (detail::unpack_first_conv, weights.hpp:231-240). */
typedef struct btnn_loaded_weights btnn_loaded_weights;
int btnn_cuda_load_weights(const char* path, const btnn_model_spec* model, btnn_loaded_weights** out);
/* View for btnn_cuda_plan_create; valid until btnn_cuda_free_weights. */
int btnn_cuda_loaded_weights_store(const btnn_loaded_weights* w, btnn_weight_store* out);
int btnn_cuda_free_weights(btnn_loaded_weights* w);
/* read_batch (io.hpp:83-101): BTIN header -> n, h, w, c (whole samples only), then the
 * f32 NHWC payload into out (capacity in floats). BTNN_IO_ERROR on a malformed file. */
int btnn_cuda_batch_dims(const char* path, size_t* n, size_t* h, size_t* w, size_t* c);
int btnn_cuda_read_batch(const char* path, float* out, size_t capacity);

/* Build a device plan: validate model/weights like run_inference (inference.hpp:69-75),
 * convert weights to the device formats and upload them once to every listed device.
 * max_batch bounds the per-call batch; the batch is sharded across the devices in
 * contiguous chunks (one CUDA stream and one host thread per device). */
int btnn_cuda_plan_create(const btnn_model_spec* model, const btnn_weight_store* ws, size_t max_batch,
                          const int* devices, int n_devices, btnn_plan** out);
/* run_inference (inference.hpp:67-186) on host buffers: x is NHWC f32 batch*H*W*C; logits
 * batch*classes f64 and labels (first argmax) are written back. Synchronous. */
int btnn_cuda_plan_run(btnn_plan* plan, const float* x, size_t batch, double* logits, int32_t* labels);
/* Device-resident variant for shard `shard` (its own device): pointers are device
 * pointers on that device; stream is a cudaStream_t (NULL = the plan's stream). Async. */
int btnn_cuda_plan_run_device(btnn_plan* plan, int shard, const float* d_x, size_t batch,
                              double* d_logits, int32_t* d_labels, void* stream);
/* After a plan_run_device has completed (the caller synchronized its stream): 1 when that
 * run's input held a non-finite value — the condition under which run_inference throws
 * invalid_input (inference.hpp:69-75); the device run's logits are then not the reference's. */
int btnn_cuda_plan_input_status(btnn_plan* plan, int shard, int* nonfinite);
/* End-to-end input pipelining of btnn_cuda_plan_run (the host-buffer run_inference): the chunk
 * sizes shard `shard` uses for `batch` images (n_sizes of them, the first `cap` written) and its
 * measured model: model[0] = 1 once calibrated (on the shard's first host run), [1] host->device
 * copy us per image, [2] graph latency t0 us, [3] graph us per image, [4] the modelled step us. */
int btnn_cuda_plan_e2e_schedule(btnn_plan* plan, int shard, size_t batch, double* model, size_t* sizes, size_t cap,
                                size_t* n_sizes);
/* Per-layer device time of the last plan_run on shard 0, ms (RunOptions::breakdown,
 * inference.hpp:169-174). n_layers entries. */
int btnn_cuda_plan_layer_ms(btnn_plan* plan, double* ms, size_t n_layers);
/* Enable/disable per-layer timing (adds events; off by default). */
int btnn_cuda_plan_set_breakdown(btnn_plan* plan, int enabled);
/* Kernel launches per plan_run on one shard (for the bench's gpu_launches). */
int btnn_cuda_plan_launches(btnn_plan* plan, size_t batch, size_t* launches);
/* Inspection: copy the f64 residual tap (RealTensorPQNO) that layer i stored during the
 * last run on shard 0, dims[0]*dims[1]*batch*dims[3] doubles with dims from
 * btnn_cuda_plan_tap_dims. BTNN_INVALID_INPUT if the layer has no residual_out port. */
int btnn_cuda_plan_read_tap(btnn_plan* plan, size_t i, size_t batch, double* out);
/* Shape of the stored tap of layer i: dims = {h, w, averaged, channels}. A layer whose
 * only consumer halves the shortcut (adapt_shortcut, inference.hpp:43-63) stores the
 * 2x2-averaged tap directly (averaged = 1, h = out_h/2, w = out_w/2); otherwise the full
 * tap (averaged = 0). */
int btnn_cuda_plan_tap_dims(btnn_plan* plan, size_t i, size_t* dims);
/* Plan tuner (on by default; BTNN_AUTOTUNE=0 or btnn_cuda_set_autotune(0) turns it off for
 * plans created afterwards): at plan_create every tensor-core conv layer times each
 * geometry its shape allows (the cost model's pick, halo mode at each feasible sites-per-tile,
 * the TMEM-A path) in eager forwards at the plan's max batch and keeps the fastest. All
 * geometries compute the same exact sums. */
int btnn_cuda_set_autotune(int enabled);
/* Layer i's candidates as "name,name,..." with the pick starred ("*halo/spt2,halo/spt4,tmemA"),
 * and their measured ms (n_ms entries at most); "" for layers without candidates. */
int btnn_cuda_plan_layer_choice(btnn_plan* plan, size_t i, char* buf, size_t n, double* ms, size_t n_ms);
/* Run candidate k (btnn_cuda_plan_layer_choice order) for layer i from now on. */
int btnn_cuda_plan_set_layer_choice(btnn_plan* plan, size_t i, size_t k);
/* Name of the engine chosen for layer i ("tc_i8", "popc", "fp64", "orpool", ...). */
const char* btnn_cuda_plan_layer_engine(btnn_plan* plan, size_t i);
int btnn_cuda_plan_destroy(btnn_plan* plan);

/* ---- BENN ensembles ---------------------------- */
/* Combine K member outputs on the device. d_logits: K x batch x classes f64 (member-major,
 * as K plan_run_device calls leave them), d_labels: K x batch. Members fold in member order:
 *   HARD        votes[c] = #{k : label_k == c} (as f64)
 *   SOFT        mean[c] = (((l_0 + l_1) + ...) + l_{K-1}) / K
 *   BOOST       score[c] = sum_k (label_k == c ? alpha_k : 0)  (weighted vote)
 *   BOOST_SOFT  score[c] = sum_k fl(alpha_k * l_k[c])
 * then the first-max label per row (inference.hpp:177-184). alpha: host array of K member
 * weights (boosting modes). Outputs are device pointers; async on `stream` (NULL = legacy). */
enum { BTNN_BENN_HARD = 0, BTNN_BENN_SOFT = 1, BTNN_BENN_BOOST = 2, BTNN_BENN_BOOST_SOFT = 3 };
int btnn_cuda_benn_combine(const double* d_logits, const int32_t* d_labels, size_t members, size_t batch,
                           size_t classes, const double* alpha, int mode, double* d_scores, int32_t* d_out_labels,
                           void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BTNN_CUDA_H_ */
