"""Weights for the harness: float weights, binarization into the reference bit layouts,
bn+sign folding, and the C-ABI WeightStore view.

Mirrors weights.hpp: random_weights (:34-73; same distributions, drawn with numpy's
generator rather than libstdc++'s, so values differ from the reference for a given
seed), pack_filter (tensors.hpp:177-193), pack_fc (weights.hpp:231-240),
unpack_first_conv (:224-229), build_weights (:255-296), fold_bn_sign
(layer_math.hpp:61-67). For bit-identical parity with the reference's own
random_weights, tests import the reference-built store instead (tests/refshim.py).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from .model import Model, needs_bn_route


def ru(v: int, m: int) -> int:
    return (v + m - 1) // m * m


def bits_to_words(bits: np.ndarray) -> np.ndarray:
    """Flat bool array (length multiple of 64) -> LSB-first uint64 words."""
    b = np.packbits(bits.astype(np.uint8).reshape(-1), bitorder="little")
    return b.view("<u8").copy()


def words_to_bits(words: np.ndarray, n: int | None = None) -> np.ndarray:
    b = np.unpackbits(np.ascontiguousarray(words, dtype="<u8").view(np.uint8), bitorder="little").astype(bool)
    return b if n is None else b[:n]


# ---- index math (bit_matrix.hpp:36-114, tensors.hpp:79-147) ----------------------
def mat_padded(rows, cols, layout, bh=8, bw=128):
    pr = {capi.ROW_PACKED: rows, capi.COL_PACKED: ru(rows, 128), capi.FSB_ROW: ru(rows, bh), capi.FSB_COL: ru(rows, bw)}[layout]
    pc = {capi.ROW_PACKED: ru(cols, 128), capi.COL_PACKED: cols, capi.FSB_ROW: ru(cols, bw), capi.FSB_COL: ru(cols, bh)}[layout]
    return pr, pc


def mat_bit_index(rows, cols, layout, r, c, bh=8, bw=128):
    pr, pc = mat_padded(rows, cols, layout, bh, bw)
    if layout == capi.ROW_PACKED:
        return r * pc + c
    if layout == capi.COL_PACKED:
        return c * pr + r
    if layout == capi.FSB_ROW:
        return ((r // bh) * (pc // bw) + c // bw) * (bh * bw) + (r % bh) * bw + (c % bw)
    return ((c // bh) * (pr // bw) + r // bw) * (bh * bw) + (c % bh) * bw + (r % bw)


def mat_words(rows, cols, layout, bh=8, bw=128):
    pr, pc = mat_padded(rows, cols, layout, bh, bw)
    return pr * pc // 64


def pack_matrix(values: np.ndarray, rows: int, cols: int, layout: int, bh=8, bw=128) -> np.ndarray:
    """pack_matrix (bit_matrix.hpp:135-155) for a rows x cols float array."""
    v = np.asarray(values).reshape(rows, cols)
    if not np.all(np.isfinite(v)):
        raise ValueError("pack_matrix: non-finite value")
    bits = np.zeros(mat_words(rows, cols, layout, bh, bw) * 64, dtype=bool)
    r, c = np.nonzero(v >= 0)
    bits[mat_bit_index(rows, cols, layout, r, c, bh, bw)] = True
    return bits_to_words(bits)


def act_words(h, w, n, c, tiled=False, bh=8, bw=128):
    return h * w * ru(n, bh if tiled else 8) * ru(c, bw if tiled else 128) // 64


def act_bit_index(w, n, c, tiled, hh, ww, nn, cc, bh=8, bw=128):
    np_, cp = ru(n, bh if tiled else 8), ru(c, bw if tiled else 128)
    base = (hh * w + ww) * np_ * cp
    if not tiled:
        return base + nn * cp + cc
    return base + ((nn // bh) * (cp // bw) + cc // bw) * (bh * bw) + (nn % bh) * bw + (cc % bw)


def pack_nhwc(x: np.ndarray, tiled=False, bh=8, bw=128) -> np.ndarray:
    """pack_nhwc (tensors.hpp:162-174); x is (N, H, W, C)."""
    n, h, w, c = x.shape
    bits = np.zeros(act_words(h, w, n, c, tiled, bh, bw) * 64, dtype=bool)
    nn, hh, ww, cc = np.nonzero(x >= 0)
    bits[act_bit_index(w, n, c, tiled, hh, ww, nn, cc, bh, bw)] = True
    return bits_to_words(bits)


def unpack_act(words, h, w, n, c, tiled=False, bh=8, bw=128) -> np.ndarray:
    """Bits of an HWNC tensor as a bool (H, W, N, C) array."""
    bits = words_to_bits(words)
    hh, ww, nn, cc = np.meshgrid(np.arange(h), np.arange(w), np.arange(n), np.arange(c), indexing="ij")
    return bits[act_bit_index(w, n, c, tiled, hh, ww, nn, cc, bh, bw)]


def filter_words(kh, kw, o, c, tiled=False, bh=8, bw=128):
    return kh * kw * ru(o, bh if tiled else 8) * ru(c, bw if tiled else 128) // 64


def pack_filter(wt: np.ndarray, kh, kw, o, c, tiled=False, bh=8, bw=128) -> np.ndarray:
    """pack_filter (tensors.hpp:177-193): flat (r, s, o, c) floats."""
    w = np.asarray(wt).reshape(kh, kw, o, c)
    op, cp = ru(o, bh if tiled else 8), ru(c, bw if tiled else 128)
    bits = np.zeros(kh * kw * op * cp, dtype=bool)
    r, s, oo, cc = np.nonzero(w >= 0)
    base = (r * kw + s) * op * cp
    if tiled:
        idx = base + ((oo // bh) * (cp // bw) + cc // bw) * (bh * bw) + (oo % bh) * bw + (cc % bw)
    else:
        idx = base + oo * cp + cc
    bits[idx] = True
    return bits_to_words(bits)


def pack_fc(w: np.ndarray, n_in: int, n_out: int, tiled=False, bh=8, bw=128) -> np.ndarray:
    """pack_fc (weights.hpp:231-240): BitMatrix(in, out) column j = weights row j."""
    layout = capi.FSB_COL if tiled else capi.COL_PACKED
    wm = np.asarray(w).reshape(n_out, n_in)
    bits = np.zeros(mat_words(n_in, n_out, layout, bh, bw) * 64, dtype=bool)
    j, d = np.nonzero(wm >= 0)
    bits[mat_bit_index(n_in, n_out, layout, d, j, bh, bw)] = True
    return bits_to_words(bits)


def fold_bn_sign(gamma, beta, mean, var, eps):
    """layer_math.hpp:61-67, element-wise in IEEE f64 with the reference's op order."""
    gamma, beta, mean, var = (np.asarray(a, dtype=np.float64) for a in (gamma, beta, mean, var))
    s = np.sqrt(var + eps)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        tau_nz = mean - beta * s / gamma
    tau = np.where(gamma != 0.0, tau_nz, 0.0)
    kind = np.where(gamma > 0.0, capi.GEQ, np.where(gamma < 0.0, capi.LEQ,
                                                     np.where(beta >= 0.0, capi.CONST_PLUS, capi.CONST_MINUS)))
    return tau.astype(np.float64), kind.astype(np.uint8)


def bn_apply(v, gamma, beta, mean, var, eps):
    """BnParams::apply (layer_math.hpp:32-34), vectorized over channels (last axis)."""
    return (np.asarray(v, dtype=np.float64) - mean) / np.sqrt(var + eps) * gamma + beta


class FloatWeights:
    """FloatWeights (weights.hpp:20-31): per layer float weights + bn arrays."""

    def __init__(self, layers):
        self.layers = layers  # list of dict(weights=f32 array, gamma, beta, mean, var) or None for pools


def random_weights(m: Model, seed: int) -> FloatWeights:
    """random_weights (weights.hpp:34-73) with numpy's PCG64 generator."""
    rng = np.random.default_rng(seed)
    out = []
    for l in m.layers:
        if l.kind == capi.OR_POOL:
            out.append(None)
            continue
        if l.kind in (capi.FIRST_CONV_BWN, capi.BIT_CONV):
            nw, ch, fan = l.kh * l.kw * l.out_channels * l.in_channels, l.out_channels, l.kh * l.kw * l.in_channels
        else:
            nw, ch, fan = l.units * l.in_channels, l.units, l.in_channels
        w = rng.standard_normal(nw, dtype=np.float32)
        spread = np.sqrt(float(fan)) * 0.5
        out.append(dict(weights=w, gamma=rng.standard_normal(ch), beta=rng.standard_normal(ch),
                        mean=rng.standard_normal(ch) * spread, var=rng.uniform(0.25, 2.0, ch)))
    return FloatWeights(out)


class WeightStoreHost:
    """WeightStore (weights.hpp:223-227) held as numpy arrays, with a C-ABI view."""

    def __init__(self, m: Model, layers, tiled=False, bh=8, bw=128):
        self.model, self.layers, self.tiled, self.bh, self.bw = m, layers, tiled, bh, bw

    def c_store(self) -> capi.WeightStore:
        arr = (capi.LayerWeights * len(self.layers))()
        keep = []

        def ptr(a, t):
            if a is None:
                return C.POINTER(t)()
            a = np.ascontiguousarray(a)
            keep.append(a)
            return a.ctypes.data_as(C.POINTER(t))

        for i, (l, lw) in enumerate(zip(self.model.layers, self.layers)):
            rec = capi.LayerWeights()
            rec.kind = l.kind
            if lw.get("filter") is not None:
                rec.filter_words, rec.filter_n_words = ptr(lw["filter"], C.c_uint64), lw["filter"].size
            if lw.get("conv_pm1") is not None:
                rec.conv_pm1, rec.conv_pm1_n = ptr(lw["conv_pm1"], C.c_float), lw["conv_pm1"].size
            if lw.get("fc") is not None:
                rec.fc_words, rec.fc_n_words = ptr(lw["fc"], C.c_uint64), lw["fc"].size
            if lw.get("tau") is not None:
                rec.tau, rec.tkind, rec.n_thresholds = ptr(lw["tau"], C.c_double), ptr(lw["kind"], C.c_uint8), lw["tau"].size
            if lw.get("bn") is not None:
                g, b, mu, v = (np.ascontiguousarray(x, dtype=np.float64) for x in lw["bn"])
                rec.has_bn = 1
                rec.bn = capi.Bn(ptr(g, C.c_double), ptr(b, C.c_double), ptr(mu, C.c_double), ptr(v, C.c_double),
                                 g.size, self.model.epsilon)
            arr[i] = rec
        self._keep = (arr, keep)
        return capi.WeightStore(int(self.tiled), self.bh, self.bw, arr, len(self.layers))


def build_weights(m: Model, fw: FloatWeights, tiled=False, bh=8, bw=128) -> WeightStoreHost:
    """build_weights (weights.hpp:255-296)."""
    layers = []
    for l, lw in zip(m.layers, fw.layers):
        rec = {}
        if l.kind == capi.OR_POOL:
            layers.append(rec)
            continue
        w = np.asarray(lw["weights"], dtype=np.float32)
        if l.kind in (capi.FIRST_CONV_BWN, capi.BIT_CONV):
            rec["filter"] = pack_filter(w, l.kh, l.kw, l.out_channels, l.in_channels, tiled, bh, bw)
            if l.kind == capi.FIRST_CONV_BWN:
                # unpack_first_conv (weights.hpp:224-229): (o, r, s, c) +-1 floats
                pm = np.where(w.reshape(l.kh, l.kw, l.out_channels, l.in_channels) >= 0, 1.0, -1.0).astype(np.float32)
                rec["conv_pm1"] = np.ascontiguousarray(pm.transpose(2, 0, 1, 3)).reshape(-1)
        else:
            rec["fc"] = pack_fc(w, l.in_channels, l.units, tiled, bh, bw)
        bn = tuple(np.asarray(lw[k], dtype=np.float64) for k in ("gamma", "beta", "mean", "var"))
        if needs_bn_route(l):
            rec["bn"] = bn
        else:
            rec["tau"], rec["kind"] = fold_bn_sign(*bn, m.epsilon)
        layers.append(rec)
    return WeightStoreHost(m, layers, tiled, bh, bw)
