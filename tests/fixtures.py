"""Golden-fixture loading helpers (tests/golden/*.npz, made by make_golden.py)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2006_16578_b200 import capi

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SPEC_FIELDS = ["kind", "kh", "kw", "out_channels", "stride", "pad", "window", "pool_stride", "units", "in_h", "in_w",
               "in_channels", "out_h", "out_w", "residual_out", "residual_in", "shortcut_from"]

_cache = {}


def load(name: str):
    if name not in _cache:
        _cache[name] = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    return _cache[name]


def indices(d: dict, prefix: str, suffix: str):
    """Sorted case indices i for keys f'{prefix}{i}_{suffix}'."""
    out = set()
    for k in d:
        if k.startswith(prefix) and k.endswith("_" + suffix):
            mid = k[len(prefix):-len(suffix) - 1]
            if mid.isdigit():
                out.add(int(mid))
    return sorted(out)


class FixtureModel:
    """A reference-built (model, weight store, input, logits) case as C-ABI structs."""

    def __init__(self, d: dict, prefix: str):
        self.keep = []
        hdr = d[prefix + "hdr"]
        self.in_h, self.in_w, self.in_c, self.classes, n = (int(v) for v in hdr)
        specs = d[prefix + "specs"]
        arr = (capi.LayerSpec * n)()
        for i in range(n):
            arr[i] = capi.LayerSpec(*[int(v) for v in specs[i]])
        self.name = prefix.encode()
        self.spec = capi.ModelSpec(self.name, self.in_h, self.in_w, self.in_c, self.classes, float(d[prefix + "eps"][0]),
                                   arr, n)
        self.keep.append(arr)
        tiled, bh, bw = (int(v) for v in d[prefix + "store"])
        larr = (capi.LayerWeights * n)()
        for i in range(n):
            q = f"{prefix}L{i}_"
            rec = capi.LayerWeights()
            rec.kind = int(specs[i][0])
            if q + "filter" in d:
                a = np.ascontiguousarray(d[q + "filter"], dtype=np.uint64)
                self.keep.append(a)
                rec.filter_words, rec.filter_n_words = a.ctypes.data_as(C.POINTER(C.c_uint64)), a.size
            if q + "conv_pm1" in d:
                a = np.ascontiguousarray(d[q + "conv_pm1"], dtype=np.float32)
                self.keep.append(a)
                rec.conv_pm1, rec.conv_pm1_n = a.ctypes.data_as(C.POINTER(C.c_float)), a.size
            if q + "fc" in d:
                a = np.ascontiguousarray(d[q + "fc"], dtype=np.uint64)
                self.keep.append(a)
                rec.fc_words, rec.fc_n_words = a.ctypes.data_as(C.POINTER(C.c_uint64)), a.size
            if q + "tau" in d:
                t = np.ascontiguousarray(d[q + "tau"], dtype=np.float64)
                k = np.ascontiguousarray(d[q + "tkind"], dtype=np.uint8)
                self.keep += [t, k]
                rec.tau, rec.tkind, rec.n_thresholds = (t.ctypes.data_as(C.POINTER(C.c_double)),
                                                        k.ctypes.data_as(C.POINTER(C.c_uint8)), t.size)
            if q + "bn" in d:
                bn = [np.ascontiguousarray(x, dtype=np.float64) for x in d[q + "bn"]]
                self.keep += bn
                rec.has_bn = 1
                rec.bn = capi.Bn(*(x.ctypes.data_as(C.POINTER(C.c_double)) for x in bn), bn[0].size,
                                 float(d[prefix + "eps"][0]))
            larr[i] = rec
        self.keep.append(larr)
        self.store = capi.WeightStore(tiled, bh, bw, larr, n)
        self.x = d[prefix + "x"]
        self.logits = d[prefix + "logits"]
        self.labels = d[prefix + "labels"]


def fixture_models():
    d = load("models")
    out = []
    for k in sorted(d):
        if k.endswith("_hdr"):
            p = k[:-3]
            out.append((p, FixtureModel(d, p)))
    return out
