"""Python face of libbtnn_cuda: the reference's layer/model API names over the C ABI.

Each function mirrors one reference function (same name, same argument meaning, same
error class via BtnnError.code) and calls the sm_100a implementation through
include/btnn_cuda.h. Arrays are numpy; bit tensors are uint64 word arrays in the
reference layouts.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from .capi import check, lib
from .model import Model
from .weights import WeightStoreHost


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def matrix_words(rows, cols, layout, bh=8, bw=128) -> int:
    return lib().btnn_cuda_matrix_words(C.byref(capi.MatrixDesc(rows, cols, layout, bh, bw)))


def _opts(variant=capi.BMM_BLOCKED, blocking=(8, 8, 1024)):
    return capi.BmmOptions(variant, blocking[0], blocking[1], blocking[2], 0)


# ---- BMM (bmm.hpp:204-274) ------------------------------------------------------------
def bmm_raw(a: capi.MatrixDesc, aw, b: capi.MatrixDesc, bw, variant=capi.BMM_BLOCKED, blocking=(8, 8, 1024)):
    out = np.zeros(a.rows * b.cols, dtype=np.int32)
    aw, bw = _u64(aw), _u64(bw)
    check(lib().btnn_cuda_bmm_raw(C.byref(a), _p(aw, C.c_uint64), C.byref(b), _p(bw, C.c_uint64),
                                  C.byref(_opts(variant, blocking)), _p(out, C.c_int32)))
    return out.reshape(a.rows, b.cols)


def bmm_pm1(a, aw, b, bw, variant=capi.BMM_BLOCKED, blocking=(8, 8, 1024)):
    out = np.zeros(a.rows * b.cols, dtype=np.int32)
    aw, bw = _u64(aw), _u64(bw)
    check(lib().btnn_cuda_bmm_pm1(C.byref(a), _p(aw, C.c_uint64), C.byref(b), _p(bw, C.c_uint64),
                                  C.byref(_opts(variant, blocking)), _p(out, C.c_int32)))
    return out.reshape(a.rows, b.cols)


def bmm_pm1_bin(a, aw, b, bw, variant=capi.BMM_BLOCKED, tau=None, kind=None, blocking=(8, 8, 1024)):
    out_layout = capi.FSB_ROW if a.layout == capi.FSB_ROW else capi.ROW_PACKED
    out = np.zeros(matrix_words(a.rows, b.cols, out_layout, a.bh, a.bw), dtype=np.uint64)
    aw, bw = _u64(aw), _u64(bw)
    n = 0 if tau is None else len(tau)
    tau = np.ascontiguousarray(tau if tau is not None else np.zeros(1), dtype=np.float64)
    kind = np.ascontiguousarray(kind if kind is not None else np.zeros(1), dtype=np.uint8)
    check(lib().btnn_cuda_bmm_pm1_bin(C.byref(a), _p(aw, C.c_uint64), C.byref(b), _p(bw, C.c_uint64),
                                      C.byref(_opts(variant, blocking)), _p(tau, C.c_double), _p(kind, C.c_uint8), n,
                                      _p(out, C.c_uint64)))
    return out


# ---- BConv (bconv.hpp:138-272) --------------------------------------------------------
def _act(h, w, n, c, tiled=False, bh=8, bw=128):
    return capi.ActDesc(h, w, n, c, int(tiled), bh, bw)


def _out_dim(x, k, s, p):
    return (x + 2 * p - k) // s + 1


def bconv_pm1(ind: capi.ActDesc, iw, fd: capi.FilterDesc, fw, geo: capi.ConvGeom):
    P, Q = _out_dim(ind.height, geo.kh, geo.stride, geo.pad), _out_dim(ind.width, geo.kw, geo.stride, geo.pad)
    out = np.zeros(max(P, 0) * max(Q, 0) * ind.batch * fd.out_channels, dtype=np.int32)
    iw, fw = _u64(iw), _u64(fw)
    check(lib().btnn_cuda_bconv_pm1(C.byref(ind), _p(iw, C.c_uint64), C.byref(fd), _p(fw, C.c_uint64), C.byref(geo),
                                    _p(out, C.c_int32)))
    return out


def bconv_fused(ind, iw, fd, fw, geo, tau=None, kind=None, bn=None, eps=1e-5, residual_in=None, want_residual_out=False):
    """bconv_fused (bconv.hpp:160-194). bn = (gamma, beta, mean, var). Returns (bits, residual_out|None)."""
    P, Q = _out_dim(ind.height, geo.kh, geo.stride, geo.pad), _out_dim(ind.width, geo.kw, geo.stride, geo.pad)
    O = fd.out_channels
    out = np.zeros(max(lib().btnn_cuda_act_words(C.byref(_act(max(P, 1), max(Q, 1), ind.batch, O, ind.tiled, ind.bh, ind.bw))), 1),
                   dtype=np.uint64)
    f = capi.ConvFused()
    keep = []
    if tau is not None and len(tau):
        t = np.ascontiguousarray(tau, dtype=np.float64)
        k = np.ascontiguousarray(kind, dtype=np.uint8)
        keep += [t, k]
        f.tau, f.kind, f.n_thresholds = _p(t, C.c_double), _p(k, C.c_uint8), len(t)
    bnc = None
    if bn is not None:
        arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in bn]
        keep += arrs
        bnc = capi.Bn(*(_p(a, C.c_double) for a in arrs), len(arrs[0]), eps)
        f.bn = C.pointer(bnc)
    if residual_in is not None:
        r = np.ascontiguousarray(residual_in, dtype=np.float64)
        keep.append(r)
        f.residual_in = _p(r, C.c_double)
    rout = None
    if want_residual_out:
        rout = np.zeros(max(P, 1) * max(Q, 1) * ind.batch * O, dtype=np.float64)
        f.residual_out = _p(rout, C.c_double)
    iw, fw = _u64(iw), _u64(fw)
    check(lib().btnn_cuda_bconv_fused(C.byref(ind), _p(iw, C.c_uint64), C.byref(fd), _p(fw, C.c_uint64), C.byref(geo),
                                      C.byref(f), _p(out, C.c_uint64)))
    return out, rout


def first_conv_bwn(x: np.ndarray, w_pm1: np.ndarray, kh, kw, o, geo: capi.ConvGeom):
    """first_conv_bwn (bconv.hpp:198-243); x NHWC f32, w_pm1 (o, r, s, c)."""
    n, h, w, c = x.shape
    P, Q = _out_dim(h, geo.kh, geo.stride, geo.pad), _out_dim(w, geo.kw, geo.stride, geo.pad)
    out = np.zeros(max(P, 0) * max(Q, 0) * n * o, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float32)
    wp = np.ascontiguousarray(w_pm1, dtype=np.float32).reshape(-1)
    check(lib().btnn_cuda_first_conv_bwn(_p(x, C.c_float), n, h, w, c, _p(wp, C.c_float), wp.size, kh, kw, o,
                                         C.byref(geo), _p(out, C.c_double)))
    return out


def or_pool(ind: capi.ActDesc, iw, window, stride):
    oh = (ind.height - window) // stride + 1 if ind.height >= window and stride else 1
    ow = (ind.width - window) // stride + 1 if ind.width >= window and stride else 1
    out = np.zeros(max(lib().btnn_cuda_act_words(C.byref(_act(oh, ow, ind.batch, ind.channels, ind.tiled, ind.bh, ind.bw))), 1),
                   dtype=np.uint64)
    iw = _u64(iw)
    check(lib().btnn_cuda_or_pool(C.byref(ind), _p(iw, C.c_uint64), window, stride, _p(out, C.c_uint64)))
    return out


# ---- format stage ------------------------------------------------------------------
def pack_matrix(values: np.ndarray, rows, cols, layout, bh=8, bw=128):
    v = np.ascontiguousarray(values, dtype=np.float32).reshape(-1)
    d = capi.MatrixDesc(rows, cols, layout, bh, bw)
    out = np.zeros(max(matrix_words(rows, cols, layout, bh, bw), 1), dtype=np.uint64)
    check(lib().btnn_cuda_pack_matrix(_p(v, C.c_float), v.size, C.byref(d), _p(out, C.c_uint64)))
    return out


def pack_nhwc(x: np.ndarray, tiled=False, bh=8, bw=128):
    n, h, w, c = x.shape
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.zeros(lib().btnn_cuda_act_words(C.byref(_act(h, w, n, c, tiled, bh, bw))), dtype=np.uint64)
    check(lib().btnn_cuda_pack_nhwc(_p(x, C.c_float), n, h, w, c, int(tiled), bh, bw, _p(out, C.c_uint64)))
    return out


def to_fsb(d: capi.MatrixDesc, words, bh=8, bw=128):
    tgt = capi.FSB_ROW if d.layout == capi.ROW_PACKED else capi.FSB_COL
    out = np.zeros(max(matrix_words(d.rows, d.cols, tgt, bh, bw), 1), dtype=np.uint64)
    words = _u64(words)
    check(lib().btnn_cuda_to_fsb(C.byref(d), _p(words, C.c_uint64), bh, bw, _p(out, C.c_uint64)))
    return out


def from_fsb(d: capi.MatrixDesc, words):
    tgt = capi.ROW_PACKED if d.layout == capi.FSB_ROW else capi.COL_PACKED
    out = np.zeros(max(matrix_words(d.rows, d.cols, tgt), 1), dtype=np.uint64)
    words = _u64(words)
    check(lib().btnn_cuda_from_fsb(C.byref(d), _p(words, C.c_uint64), _p(out, C.c_uint64)))
    return out


def flatten_to_matrix(d: capi.ActDesc, words, layout, bh=8, bw=128):
    feats = d.height * d.width * d.channels
    out = np.zeros(matrix_words(d.batch, feats, layout, bh, bw), dtype=np.uint64)
    words = _u64(words)
    md = capi.MatrixDesc(d.batch, feats, layout, bh, bw)
    check(lib().btnn_cuda_flatten_to_matrix(C.byref(d), _p(words, C.c_uint64), C.byref(md), _p(out, C.c_uint64)))
    return out


def convert_activations(d: capi.ActDesc, words, tiled, bh=8, bw=128):
    out = np.zeros(lib().btnn_cuda_act_words(C.byref(_act(d.height, d.width, d.batch, d.channels, tiled, bh, bw))),
                   dtype=np.uint64)
    words = _u64(words)
    check(lib().btnn_cuda_convert_activations(C.byref(d), _p(words, C.c_uint64), int(tiled), bh, bw, _p(out, C.c_uint64)))
    return out


# ---- model driver (inference.hpp:67-186) ---------------------------------------------
class LoadedWeights:
    """load_weights (weights.hpp:354-445) of a BTNN bit-weight file, parsed by the library
    (btnn_cuda_load_weights) with the reference's checks; pass it to Plan like a store."""

    def __init__(self, path: str, m):
        self._spec = m.c_spec() if isinstance(m, Model) else m
        h = C.c_void_p()
        check(lib().btnn_cuda_load_weights(str(path).encode(), C.byref(self._spec), C.byref(h)))
        self.h = h

    def c_store(self):
        st = capi.WeightStore()
        check(lib().btnn_cuda_loaded_weights_store(self.h, C.byref(st)))
        return st

    def __del__(self):
        try:
            if self.h:
                lib().btnn_cuda_free_weights(self.h)
                self.h = None
        except Exception:
            pass


def read_batch(path: str) -> np.ndarray:
    """read_batch (io.hpp:83-101): a BTIN file as an (n, h, w, c) float32 array."""
    n, h, w, c = C.c_size_t(), C.c_size_t(), C.c_size_t(), C.c_size_t()
    p = str(path).encode()
    check(lib().btnn_cuda_batch_dims(p, C.byref(n), C.byref(h), C.byref(w), C.byref(c)))
    x = np.empty((n.value, h.value, w.value, c.value), dtype=np.float32)
    check(lib().btnn_cuda_read_batch(p, _p(x, C.c_float), x.size))
    return x


class Plan:
    """A device plan for (model, weight store); run() is run_inference on host arrays."""

    def __init__(self, m: Model, ws, max_batch: int, devices=(0,)):
        self.model = m
        self._spec = m.c_spec() if isinstance(m, Model) else m
        self._store = ws.c_store() if hasattr(ws, "c_store") else ws
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        check(lib().btnn_cuda_plan_create(C.byref(self._spec), C.byref(self._store), max_batch, devs, len(devices),
                                          C.byref(h)))
        self.h = h
        self.classes = self._spec.classes
        self.n_layers = self._spec.n_layers
        self.in_dims = (self._spec.in_h, self._spec.in_w, self._spec.in_c)
        self.devices = tuple(devices)
        self.device = devices[0] if len(devices) == 1 else -1  # -1: sharded over devices

    def run(self, x: np.ndarray):
        x = np.ascontiguousarray(x, dtype=np.float32)
        # btnn_cuda_plan_run reads batch * in_h * in_w * in_c floats: the shape is checked
        # here, as run_inference does (inference.hpp:69-75)
        if x.ndim != 4 or tuple(x.shape[1:]) != self.in_dims:
            raise capi.BtnnError(capi.BTNN_INVALID_INPUT, "run_inference: input dims do not match model")
        b = x.shape[0]
        logits = np.zeros(b * self.classes, dtype=np.float64)
        labels = np.zeros(b, dtype=np.int32)
        check(lib().btnn_cuda_plan_run(self.h, _p(x, C.c_float), b, _p(logits, C.c_double), _p(labels, C.c_int32)))
        return logits.reshape(b, self.classes), labels

    def run_device(self, d_x: int, batch: int, d_logits: int = 0, d_labels: int = 0, stream: int = 0, shard: int = 0):
        check(lib().btnn_cuda_plan_run_device(self.h, shard, C.c_void_p(d_x), batch, C.c_void_p(d_logits or None),
                                              C.c_void_p(d_labels or None), C.c_void_p(stream or None)))

    def input_status(self, shard: int = 0) -> bool:
        """True when the last completed run_device on `shard` saw a non-finite input value
        (run_inference's invalid_input condition)."""
        f = C.c_int()
        check(lib().btnn_cuda_plan_input_status(self.h, shard, C.byref(f)))
        return bool(f.value)

    def e2e_schedule(self, batch: int, shard: int = 0):
        """The input pipelining run() uses for `batch` images on `shard`: chunk sizes and the
        measured model behind them (None before the shard's first host run calibrated it)."""
        model = (C.c_double * 5)()
        sizes = (C.c_size_t * 32)()
        n = C.c_size_t()
        check(lib().btnn_cuda_plan_e2e_schedule(self.h, shard, batch, model, sizes, 32, C.byref(n)))
        if not model[0]:
            return None
        return {"chunks": [int(sizes[i]) for i in range(min(n.value, 32))], "copy_us_per_image": model[1],
                "graph_t0_us": model[2], "graph_us_per_image": model[3], "modelled_step_us": model[4]}

    def set_breakdown(self, on: bool):
        check(lib().btnn_cuda_plan_set_breakdown(self.h, int(on)))

    def layer_ms(self):
        out = np.zeros(self.n_layers, dtype=np.float64)
        check(lib().btnn_cuda_plan_layer_ms(self.h, _p(out, C.c_double), self.n_layers))
        return out

    def launches(self, batch: int) -> int:
        n = C.c_size_t()
        check(lib().btnn_cuda_plan_launches(self.h, batch, C.byref(n)))
        return n.value

    def tap_dims(self, i: int):
        """(h, w, averaged, channels) of the tap layer i stored in the last run."""
        d = (C.c_size_t * 4)()
        check(lib().btnn_cuda_plan_tap_dims(self.h, i, d))
        return tuple(int(v) for v in d)

    def read_tap(self, i: int, batch: int):
        """The f64 residual tap layer i stored in the last run (shard 0), PQNO flat: the
        full tap, or the 2x2-averaged one when tap_dims(i)[2] == 1."""
        h, w, _, c = self.tap_dims(i)
        out = np.zeros(h * w * batch * c, dtype=np.float64)
        check(lib().btnn_cuda_plan_read_tap(self.h, i, batch, _p(out, C.c_double)))
        return out

    def layer_choice(self, i: int):
        """(candidate names, index of the pick, measured ms per candidate) of layer i's tuned
        tensor-core geometry (empty for layers without candidates)."""
        buf = C.create_string_buffer(256)
        ms = (C.c_double * 16)()
        check(lib().btnn_cuda_plan_layer_choice(self.h, i, buf, 256, ms, 16))
        names = [n for n in buf.value.decode().split(",") if n]
        pick = next((k for k, n in enumerate(names) if n.startswith("*")), -1)
        return [n.lstrip("*") for n in names], pick, list(ms[:len(names)])

    def set_layer_choice(self, i: int, k: int):
        """Run candidate k of layer_choice(i) for layer i from now on."""
        check(lib().btnn_cuda_plan_set_layer_choice(self.h, i, k))

    def engines(self):
        return [lib().btnn_cuda_plan_layer_engine(self.h, i).decode() for i in range(self.n_layers)]

    def close(self):
        if getattr(self, "h", None):
            lib().btnn_cuda_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_inference(m: Model, ws, x: np.ndarray, devices=(0,)):
    """One-shot run_inference (inference.hpp:67): plan, run, release."""
    p = Plan(m, ws, max(x.shape[0], 1), devices)
    try:
        return p.run(x)
    finally:
        p.close()
