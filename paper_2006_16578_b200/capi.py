"""ctypes mirror of include/btnn_cuda.h and the loader for libbtnn_cuda.so.

The product is the C ABI (and the C++ adapter include/btnn/cuda.hpp above it); this
module is the Python harness the tests and bench.py use to call it. Loading fails
loudly when the built library is missing — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# BTNN_LIB selects another build of the library (the timing-experiment build, Makefile)
LIB_PATH = os.environ.get("BTNN_LIB") or os.path.join(_HERE, "libbtnn_cuda.so")

BTNN_OK, BTNN_INVALID_INPUT, BTNN_UNSUPPORTED_SHAPE, BTNN_IO_ERROR, BTNN_VALIDATION_ERROR, BTNN_CUDA_ERROR = range(6)
ROW_PACKED, COL_PACKED, FSB_ROW, FSB_COL = range(4)
BMM_NAIVE, BMM_BLOCKED, BMM_FSB = range(3)
GEQ, LEQ, CONST_PLUS, CONST_MINUS = range(4)
FIRST_CONV_BWN, BIT_CONV, OR_POOL, BIT_FC, LAST_FC = range(5)
ENGINE_AUTO, ENGINE_POPC, ENGINE_TC = range(3)

sz = C.c_size_t


class MatrixDesc(C.Structure):
    _fields_ = [("rows", sz), ("cols", sz), ("layout", C.c_int), ("bh", sz), ("bw", sz)]


class BmmOptions(C.Structure):
    _fields_ = [("variant", C.c_int), ("blk_rows", sz), ("blk_cols", sz), ("blk_k_bits", sz), ("threads", C.c_int)]


class ActDesc(C.Structure):
    _fields_ = [("height", sz), ("width", sz), ("batch", sz), ("channels", sz), ("tiled", C.c_int), ("bh", sz), ("bw", sz)]


class FilterDesc(C.Structure):
    _fields_ = [("kh", sz), ("kw", sz), ("out_channels", sz), ("in_channels", sz), ("tiled", C.c_int), ("bh", sz), ("bw", sz)]


class ConvGeom(C.Structure):
    _fields_ = [("kh", sz), ("kw", sz), ("stride", sz), ("pad", sz)]


class Bn(C.Structure):
    _fields_ = [("gamma", C.POINTER(C.c_double)), ("beta", C.POINTER(C.c_double)), ("mean", C.POINTER(C.c_double)),
                ("var", C.POINTER(C.c_double)), ("channels", sz), ("eps", C.c_double)]


class ConvFused(C.Structure):
    _fields_ = [("tau", C.POINTER(C.c_double)), ("kind", C.POINTER(C.c_uint8)), ("n_thresholds", sz),
                ("bn", C.POINTER(Bn)), ("residual_in", C.POINTER(C.c_double)), ("residual_out", C.POINTER(C.c_double)),
                ("threads", C.c_int)]


class BenchReadback(C.Structure):
    _fields_ = [("a_words", C.POINTER(C.c_uint64)), ("b_words", C.POINTER(C.c_uint64)), ("out", C.c_void_p),
                ("kernel_ns", C.POINTER(C.c_double)), ("stream_ns", C.POINTER(C.c_double)),
                ("graph_ns", C.POINTER(C.c_double))]


class LayerSpec(C.Structure):
    _fields_ = [("kind", C.c_int), ("kh", sz), ("kw", sz), ("out_channels", sz), ("stride", sz), ("pad", sz),
                ("window", sz), ("pool_stride", sz), ("units", sz), ("in_h", sz), ("in_w", sz), ("in_channels", sz),
                ("out_h", sz), ("out_w", sz), ("residual_out", C.c_int), ("residual_in", C.c_int),
                ("shortcut_from", C.c_int)]


class ModelSpec(C.Structure):
    _fields_ = [("name", C.c_char_p), ("in_h", sz), ("in_w", sz), ("in_c", sz), ("classes", sz), ("epsilon", C.c_double),
                ("layers", C.POINTER(LayerSpec)), ("n_layers", sz)]


class LayerWeights(C.Structure):
    _fields_ = [("kind", C.c_int), ("filter_words", C.POINTER(C.c_uint64)), ("filter_n_words", sz),
                ("conv_pm1", C.POINTER(C.c_float)), ("conv_pm1_n", sz), ("fc_words", C.POINTER(C.c_uint64)),
                ("fc_n_words", sz), ("tau", C.POINTER(C.c_double)), ("tkind", C.POINTER(C.c_uint8)),
                ("n_thresholds", sz), ("has_bn", C.c_int), ("bn", Bn)]


class WeightStore(C.Structure):
    _fields_ = [("tiled", C.c_int), ("bh", sz), ("bw", sz), ("layers", C.POINTER(LayerWeights)), ("n_layers", sz)]


class BtnnError(RuntimeError):
    """A non-zero status from the C ABI; .code mirrors the reference exception class."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib = None

P = C.POINTER
u64p, i32p, f32p, f64p, u8p = P(C.c_uint64), P(C.c_int32), P(C.c_float), P(C.c_double), P(C.c_uint8)

_PROTOS = {
    "btnn_cuda_abi_version": (C.c_int, []),
    "btnn_cuda_last_error": (C.c_char_p, []),
    "btnn_cuda_device_count": (C.c_int, [P(C.c_int)]),
    "btnn_cuda_set_device": (C.c_int, [C.c_int]),
    "btnn_cuda_set_engine": (C.c_int, [C.c_int]),
    "btnn_cuda_set_bmm_kernel": (C.c_int, [C.c_int]),
    "btnn_cuda_matrix_words": (sz, [P(MatrixDesc)]),
    "btnn_cuda_act_words": (sz, [P(ActDesc)]),
    "btnn_cuda_filter_words": (sz, [P(FilterDesc)]),
    "btnn_cuda_pack_matrix": (C.c_int, [f32p, sz, P(MatrixDesc), u64p]),
    "btnn_cuda_pack_nhwc": (C.c_int, [f32p, sz, sz, sz, sz, C.c_int, sz, sz, u64p]),
    "btnn_cuda_to_fsb": (C.c_int, [P(MatrixDesc), u64p, sz, sz, u64p]),
    "btnn_cuda_from_fsb": (C.c_int, [P(MatrixDesc), u64p, u64p]),
    "btnn_cuda_convert_activations": (C.c_int, [P(ActDesc), u64p, C.c_int, sz, sz, u64p]),
    "btnn_cuda_flatten_to_matrix": (C.c_int, [P(ActDesc), u64p, P(MatrixDesc), u64p]),
    "btnn_cuda_bmm_raw": (C.c_int, [P(MatrixDesc), u64p, P(MatrixDesc), u64p, P(BmmOptions), i32p]),
    "btnn_cuda_bmm_pm1": (C.c_int, [P(MatrixDesc), u64p, P(MatrixDesc), u64p, P(BmmOptions), i32p]),
    "btnn_cuda_bmm_pm1_bin": (C.c_int, [P(MatrixDesc), u64p, P(MatrixDesc), u64p, P(BmmOptions), f64p, u8p, sz, u64p]),
    "btnn_cuda_bconv_pm1": (C.c_int, [P(ActDesc), u64p, P(FilterDesc), u64p, P(ConvGeom), i32p]),
    "btnn_cuda_bconv_fused": (C.c_int, [P(ActDesc), u64p, P(FilterDesc), u64p, P(ConvGeom), P(ConvFused), u64p]),
    "btnn_cuda_first_conv_bwn": (C.c_int, [f32p, sz, sz, sz, sz, f32p, sz, sz, sz, sz, P(ConvGeom), f64p]),
    "btnn_cuda_or_pool": (C.c_int, [P(ActDesc), u64p, sz, sz, u64p]),
    "btnn_cuda_bench_bmm": (C.c_int, [sz, C.c_int, C.c_int, C.c_int, f64p, f64p, C.c_char_p, sz, P(BenchReadback)]),
    "btnn_cuda_bench_bmm_fsb": (C.c_int, [sz, C.c_int, C.c_int, C.c_int, f64p, f64p, C.c_char_p, sz, P(BenchReadback)]),
    "btnn_cuda_bench_bconv": (C.c_int, [sz, sz, sz, sz, sz, C.c_int, C.c_int, C.c_int, f64p, f64p, C.c_char_p, sz,
                                        P(BenchReadback)]),
    "btnn_cuda_bench_bconv_fsb": (C.c_int, [sz, sz, sz, sz, sz, C.c_int, C.c_int, C.c_int, f64p, f64p, C.c_char_p, sz,
                                        P(BenchReadback)]),
    "btnn_cuda_plan_create": (C.c_int, [P(ModelSpec), P(WeightStore), sz, P(C.c_int), C.c_int, P(C.c_void_p)]),
    "btnn_cuda_plan_run": (C.c_int, [C.c_void_p, f32p, sz, f64p, i32p]),
    "btnn_cuda_plan_run_device": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, sz, C.c_void_p, C.c_void_p, C.c_void_p]),
    "btnn_cuda_plan_layer_ms": (C.c_int, [C.c_void_p, f64p, sz]),
    "btnn_cuda_plan_set_breakdown": (C.c_int, [C.c_void_p, C.c_int]),
    "btnn_cuda_plan_launches": (C.c_int, [C.c_void_p, sz, P(sz)]),
    "btnn_cuda_plan_read_tap": (C.c_int, [C.c_void_p, sz, sz, f64p]),
    "btnn_cuda_plan_tap_dims": (C.c_int, [C.c_void_p, sz, P(sz)]),
    "btnn_cuda_selftest_div": (C.c_int, [f64p, f64p, sz, f64p, f64p]),
    "btnn_cuda_debug_tc_timestamps": (C.c_int, [P(C.c_uint64), sz]),
    "btnn_cuda_last_tc_launch": (C.c_int, [C.c_char_p, sz, P(C.c_int), P(C.c_int)]),
    "btnn_cuda_debug_ftc_timestamps": (C.c_int, [P(C.c_uint64), sz]),
    "btnn_cuda_plan_layer_engine": (C.c_char_p, [C.c_void_p, sz]),
    "btnn_cuda_plan_destroy": (C.c_int, [C.c_void_p]),
    "btnn_cuda_set_autotune": (C.c_int, [C.c_int]),
    "btnn_cuda_plan_input_status": (C.c_int, [C.c_void_p, C.c_int, P(C.c_int)]),
    "btnn_cuda_plan_e2e_schedule": (C.c_int, [C.c_void_p, C.c_int, sz, P(C.c_double), P(sz), sz, P(sz)]),
    "btnn_cuda_plan_set_layer_choice": (C.c_int, [C.c_void_p, sz, sz]),
    "btnn_cuda_plan_layer_choice": (C.c_int, [C.c_void_p, sz, C.c_char_p, sz, P(C.c_double), sz]),
    "btnn_cuda_benn_combine": (C.c_int, [C.c_void_p, C.c_void_p, sz, sz, sz, C.POINTER(C.c_double), C.c_int,
                                         C.c_void_p, C.c_void_p, C.c_void_p]),
    "btnn_cuda_load_weights": (C.c_int, [C.c_char_p, P(ModelSpec), P(C.c_void_p)]),
    "btnn_cuda_loaded_weights_store": (C.c_int, [C.c_void_p, P(WeightStore)]),
    "btnn_cuda_free_weights": (C.c_int, [C.c_void_p]),
    "btnn_cuda_batch_dims": (C.c_int, [C.c_char_p, P(sz), P(sz), P(sz), P(sz)]),
    "btnn_cuda_read_batch": (C.c_int, [C.c_char_p, f32p, sz]),
}

EXPORTS = tuple(_PROTOS)


def lib() -> C.CDLL:
    """Load libbtnn_cuda.so (built by __graft_entry__.build()). Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        _lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _PROTOS.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def check(status: int) -> None:
    if status != BTNN_OK:
        raise BtnnError(status, lib().btnn_cuda_last_error().decode())


def last_tc_launch():
    """(variant, work units, grid) of the last tensor-core GEMM launched on this thread."""
    buf = C.create_string_buffer(64)
    units, grid = C.c_int(), C.c_int()
    check(lib().btnn_cuda_last_tc_launch(buf, 64, C.byref(units), C.byref(grid)))
    return buf.value.decode(), units.value, grid.value


def set_engine(engine: int) -> None:
    """btnn_cuda_set_engine: 0 auto, 1 LOP3+POPC, 2 tcgen05 tensor cores."""
    check(lib().btnn_cuda_set_engine(engine))


BMM_AUTO, BMM_WHOLE_K, BMM_PIPELINED, BMM_PIPELINED_NO_PRE = range(4)


def set_bmm_kernel(which: int) -> None:
    """btnn_cuda_set_bmm_kernel: 0 auto, 1 whole-K on-chip kernel (K <= 1536), 2 K-pipelined,
    3 K-pipelined with B expanded inside the GEMM."""
    check(lib().btnn_cuda_set_bmm_kernel(which))
