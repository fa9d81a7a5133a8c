"""ctypes loaders for the CPU checkers (TEST INFRASTRUCTURE).

- oracle(): oracle/liboracle.so, the C restatement of the reference hot path.
- ref():    oracle/_ref/libbtnn_ref_v{3,4}.so, the reference's own headers compiled
            behind oracle/ref_shim.cpp (None when not built).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use these.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2006_16578_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")

P = C.POINTER
sz = C.c_size_t
u64p, i32p, f32p, f64p, u8p = P(C.c_uint64), P(C.c_int32), P(C.c_float), P(C.c_double), P(C.c_uint8)
MD, AD, FD, CG, CF, BN = (P(capi.MatrixDesc), P(capi.ActDesc), P(capi.FilterDesc), P(capi.ConvGeom), P(capi.ConvFused),
                          P(capi.Bn))

_ORACLE = {
    "bo_pack_signs_f32": (C.c_int, [f32p, sz, u64p]),
    "bo_dot_pm1": (C.c_int64, [u64p, u64p, sz]),
    "bo_matrix_words": (sz, [sz, sz, C.c_int, sz, sz]),
    "bo_bit_index": (sz, [sz, sz, C.c_int, sz, sz, sz, sz]),
    "bo_pack_matrix": (C.c_int, [f32p, sz, sz, C.c_int, sz, sz, u64p]),
    "bo_convert_matrix": (None, [sz, sz, C.c_int, sz, sz, u64p, C.c_int, sz, sz, u64p]),
    "bo_act_words": (sz, [sz, sz, sz, sz, C.c_int, sz, sz]),
    "bo_filter_words": (sz, [sz, sz, sz, sz, C.c_int, sz, sz]),
    "bo_pack_nhwc": (C.c_int, [f32p, sz, sz, sz, sz, C.c_int, sz, sz, u64p]),
    "bo_pack_filter": (C.c_int, [f32p, sz, sz, sz, sz, C.c_int, sz, sz, u64p]),
    "bo_flatten": (None, [sz, sz, sz, sz, C.c_int, sz, sz, u64p, C.c_int, sz, sz, u64p]),
    "bo_bn_apply": (C.c_double, [BN, sz, C.c_double]),
    "bo_fire": (C.c_int, [C.c_double, C.c_uint8, C.c_double]),
    "bo_fold_bn_sign": (None, [C.c_double] * 5 + [f64p, u8p]),
    "bo_bmm_raw": (C.c_int, [MD, u64p, MD, u64p, C.c_int, i32p]),
    "bo_bmm_pm1": (C.c_int, [MD, u64p, MD, u64p, C.c_int, i32p]),
    "bo_bmm_pm1_bin": (C.c_int, [MD, u64p, MD, u64p, C.c_int, f64p, u8p, sz, u64p]),
    "bo_bconv_pm1": (C.c_int, [AD, u64p, FD, u64p, CG, i32p]),
    "bo_bconv_fused": (C.c_int, [AD, u64p, FD, u64p, CG, CF, u64p]),
    "bo_first_conv_bwn": (C.c_int, [f32p, sz, sz, sz, sz, f32p, sz, sz, sz, CG, f64p]),
    "bo_or_pool": (C.c_int, [AD, u64p, sz, sz, u64p]),
    "bo_run_inference": (C.c_int, [P(capi.ModelSpec), P(capi.WeightStore), f32p, sz, f64p, i32p]),
    "bo_ref_matmul": (None, [f64p, f64p, sz, sz, sz, f64p]),
    "bo_ref_conv_zero_pad": (C.c_int, [f64p, sz, sz, sz, sz, f64p, sz, sz, sz, sz, sz, f64p]),
    "bo_ref_max_pool": (C.c_int, [f64p, sz, sz, sz, sz, sz, sz, f64p]),
    "bo_ref_fc": (None, [f64p, sz, sz, f64p, sz, f64p]),
    "bo_ref_htanh": (C.c_double, [C.c_double]),
}

_REF = {
    "ref_last_error": (C.c_char_p, []),
    "ref_model_parse_json": (C.c_void_p, [C.c_char_p, P(C.c_int)]),
    "ref_make_model": (C.c_void_p, [C.c_char_p, C.c_char_p, sz, sz, sz, sz, P(sz), P(sz), sz, C.c_double, P(C.c_int)]),
    "ref_model_view": (P(capi.ModelSpec), [C.c_void_p]),
    "ref_model_free": (None, [C.c_void_p]),
    "ref_random_weights": (C.c_void_p, [C.c_void_p, C.c_uint64]),
    "ref_float_weights_new": (C.c_void_p, [sz]),
    "ref_float_weights_set": (None, [C.c_void_p, sz, f32p, sz, f64p, f64p, f64p, f64p, sz, C.c_double]),
    "ref_float_weights_get": (None, [C.c_void_p, sz, P(f32p), P(sz), P(f64p), P(f64p), P(f64p), P(f64p), P(sz)]),
    "ref_float_weights_free": (None, [C.c_void_p]),
    "ref_build_weights": (C.c_void_p, [C.c_void_p, C.c_void_p, C.c_int, sz, sz, P(C.c_int)]),
    "ref_store_view": (P(capi.WeightStore), [C.c_void_p]),
    "ref_store_free": (None, [C.c_void_p]),
    "ref_normal_floats": (None, [C.c_uint64, f32p, sz]),
    "ref_mt19937_64": (None, [C.c_uint64, u64p, sz]),
    "ref_run_inference": (C.c_int, [C.c_void_p, C.c_void_p, f32p, sz, C.c_int, f64p, i32p, f64p]),
    "ref_pipeline": (C.c_int, [C.c_void_p, C.c_void_p, f32p, sz, f64p, i32p]),
    "ref_matrix_words": (sz, [MD]),
    "ref_pack_matrix": (C.c_int, [f32p, sz, MD, u64p]),
    "ref_to_fsb": (C.c_int, [MD, u64p, sz, sz, u64p]),
    "ref_from_fsb": (C.c_int, [MD, u64p, u64p]),
    "ref_bmm": (C.c_int, [C.c_int, MD, u64p, MD, u64p, C.c_int, C.c_int, f64p, u8p, sz, C.c_void_p]),
    "ref_pack_nhwc": (C.c_int, [f32p, sz, sz, sz, sz, C.c_int, sz, sz, u64p]),
    "ref_pack_filter": (C.c_int, [f32p, sz, sz, sz, sz, C.c_int, sz, sz, u64p]),
    "ref_flatten": (C.c_int, [AD, u64p, C.c_int, sz, sz, u64p]),
    "ref_convert_activations": (C.c_int, [AD, u64p, C.c_int, sz, sz, u64p]),
    "ref_bconv_pm1": (C.c_int, [AD, u64p, FD, u64p, CG, C.c_int, i32p]),
    "ref_bconv_fused": (C.c_int, [AD, u64p, FD, u64p, CG, CF, u64p]),
    "ref_first_conv_bwn": (C.c_int, [f32p, sz, sz, sz, sz, f32p, sz, sz, sz, sz, CG, C.c_int, f64p]),
    "ref_or_pool": (C.c_int, [AD, u64p, sz, sz, C.c_int, u64p]),
    "ref_fold_bn_sign": (None, [C.c_double] * 5 + [f64p, u8p]),
    "ref_bn_apply": (C.c_double, [BN, sz, C.c_double]),
    "ref_run_store": (C.c_int, [P(capi.ModelSpec), P(capi.WeightStore), f32p, sz, f64p, i32p]),
    "ref_save_weights": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p]),
    "ref_write_batch": (C.c_int, [f32p, sz, sz, sz, sz, C.c_char_p]),
    "ref_infer_files": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.c_char_p, sz, f64p, i32p, P(sz)]),
}

_oracle = None
_ref = False


def _bind(lib, protos):
    for name, (res, args) in protos.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def oracle():
    global _oracle
    if _oracle is None:
        path = os.path.join(ORACLE_DIR, "liboracle.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: build with `make -C oracle`")
        _oracle = _bind(C.CDLL(path), _ORACLE)
    return _oracle


def _host_has_v4() -> bool:
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    need = ["avx512f", "avx512bw", "avx512dq", "avx512vl", "avx512cd", "avx512_vpopcntdq"]
    return all(f" {f}" in flags for f in need)


def ref_variant() -> str:
    return "v4" if _host_has_v4() else "v3"


def ref():
    """The compiled reference (oracle/_ref), or None if it was not built."""
    global _ref
    if _ref is False:
        path = os.path.join(ORACLE_DIR, "_ref", f"libbtnn_ref_{ref_variant()}.so")
        _ref = _bind(C.CDLL(path), _REF) if os.path.exists(path) else None
    return _ref


def ptr(a, t):
    return a.ctypes.data_as(P(t))


# ---- reference model/weights helpers -------------------------------------------------
class RefModel:
    """A model resolved by the reference (model.hpp) plus helpers to mirror it."""

    def __init__(self, handle):
        self.h = handle
        self.view = ref().ref_model_view(handle).contents

    @classmethod
    def make(cls, name, tokens, in_h, in_w, in_c, classes, shortcuts=(), epsilon=1e-5):
        fr = (sz * max(len(shortcuts), 1))(*[s[0] for s in shortcuts])
        to = (sz * max(len(shortcuts), 1))(*[s[1] for s in shortcuts])
        st = C.c_int()
        h = ref().ref_make_model(name.encode(), tokens.encode(), in_h, in_w, in_c, classes, fr, to, len(shortcuts),
                                 epsilon, C.byref(st))
        if st.value:
            raise ValueError(f"[{st.value}] {ref().ref_last_error().decode()}")
        return cls(h)

    @classmethod
    def parse(cls, text: str):
        st = C.c_int()
        h = ref().ref_model_parse_json(text.encode(), C.byref(st))
        if st.value:
            raise ValueError(f"[{st.value}] {ref().ref_last_error().decode()}")
        return cls(h)

    def layers(self):
        return [self.view.layers[i] for i in range(self.view.n_layers)]

    def __del__(self):
        try:
            ref().ref_model_free(self.h)
        except Exception:
            pass


class RefWeights:
    """FloatWeights + WeightStore built by the reference (weights.hpp:34-73, 255-296)."""

    def __init__(self, model: RefModel, seed: int, tiled=False, bh=8, bw=128):
        self.model = model
        self.fw = ref().ref_random_weights(model.h, seed)
        st = C.c_int()
        self.ws = ref().ref_build_weights(model.h, self.fw, int(tiled), bh, bw, C.byref(st))
        if st.value:
            raise ValueError(ref().ref_last_error().decode())
        self.store = ref().ref_store_view(self.ws).contents

    def run_inference(self, x: np.ndarray, threads=0):
        b = x.shape[0]
        c = self.model.view.classes
        lg = np.zeros(b * c, dtype=np.float64)
        lb = np.zeros(b, dtype=np.int32)
        xx = np.ascontiguousarray(x, dtype=np.float32)
        st = ref().ref_run_inference(self.model.h, self.ws, ptr(xx, C.c_float), b, threads, ptr(lg, C.c_double),
                                     ptr(lb, C.c_int32), None)
        if st:
            raise ValueError(f"[{st}] {ref().ref_last_error().decode()}")
        return lg.reshape(b, c), lb

    def pipeline(self, x: np.ndarray):
        b = x.shape[0]
        c = self.model.view.classes
        lg = np.zeros(b * c, dtype=np.float64)
        lb = np.zeros(b, dtype=np.int32)
        xx = np.ascontiguousarray(x, dtype=np.float32)
        st = ref().ref_pipeline(self.model.h, self.fw, ptr(xx, C.c_float), b, ptr(lg, C.c_double), ptr(lb, C.c_int32))
        if st:
            raise ValueError(ref().ref_last_error().decode())
        return lg.reshape(b, c), lb

    def __del__(self):
        try:
            ref().ref_store_free(self.ws)
            ref().ref_float_weights_free(self.fw)
        except Exception:
            pass


def normal_floats(seed: int, n: int) -> np.ndarray:
    """std::normal_distribution<float>(0,1) over mt19937_64(seed), as the CLI draws inputs."""
    out = np.zeros(n, dtype=np.float32)
    ref().ref_normal_floats(seed, ptr(out, C.c_float), n)
    return out


def oracle_run_inference(spec: capi.ModelSpec, store: capi.WeightStore, x: np.ndarray):
    b = x.shape[0]
    lg = np.zeros(b * spec.classes, dtype=np.float64)
    lb = np.zeros(b, dtype=np.int32)
    xx = np.ascontiguousarray(x, dtype=np.float32)
    st = oracle().bo_run_inference(C.byref(spec), C.byref(store), ptr(xx, C.c_float), b, ptr(lg, C.c_double),
                                   ptr(lb, C.c_int32))
    if st:
        raise ValueError(f"oracle status {st}")
    return lg.reshape(b, spec.classes), lb
