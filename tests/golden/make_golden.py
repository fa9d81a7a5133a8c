"""Generate the golden fixtures under tests/golden/ by running the REFERENCE itself.

Run in the build container (needs oracle/_ref built from /root/reference):
    python tests/golden/make_golden.py
Every output here comes from the reference's own functions, compiled from its
unmodified headers behind oracle/ref_shim.cpp; inputs are the same seeded draws the
reference tests use (std::mt19937_64 + std::normal_distribution<float>). The fixtures
travel with the repo so the GPU box (no reference tree) can check against them.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from paper_2006_16578_b200 import capi  # noqa: E402
from oracle_lib import RefModel, RefWeights, normal_floats, ptr, ref  # noqa: E402

sz = C.c_size_t


def _st(st):
    if st:
        raise RuntimeError(f"[{st}] {ref().ref_last_error().decode()}")


def ref_pack_matrix(v, rows, cols, layout, bh=8, bw=128):
    d = capi.MatrixDesc(rows, cols, layout, bh, bw)
    out = np.zeros(ref().ref_matrix_words(C.byref(d)), dtype=np.uint64)
    vv = np.ascontiguousarray(v, dtype=np.float32)
    _st(ref().ref_pack_matrix(ptr(vv, C.c_float), vv.size, C.byref(d), ptr(out, C.c_uint64)))
    return out


def ref_to_fsb(d, w, bh=8, bw=128):
    tgt = capi.FSB_ROW if d.layout == capi.ROW_PACKED else capi.FSB_COL
    od = capi.MatrixDesc(d.rows, d.cols, tgt, bh, bw)
    out = np.zeros(ref().ref_matrix_words(C.byref(od)), dtype=np.uint64)
    _st(ref().ref_to_fsb(C.byref(d), ptr(w, C.c_uint64), bh, bw, ptr(out, C.c_uint64)))
    return out, od


def ref_bmm(which, a, aw, b, bw, variant, tau=None, kind=None):
    if which < 2:
        out = np.zeros(a.rows * b.cols, dtype=np.int32)
    else:
        lay = capi.FSB_ROW if a.layout == capi.FSB_ROW else capi.ROW_PACKED
        out = np.zeros(ref().ref_matrix_words(C.byref(capi.MatrixDesc(a.rows, b.cols, lay, a.bh, a.bw))), dtype=np.uint64)
    n = 0 if tau is None else len(tau)
    t = np.ascontiguousarray(tau if tau is not None else [0.0], dtype=np.float64)
    k = np.ascontiguousarray(kind if kind is not None else [0], dtype=np.uint8)
    _st(ref().ref_bmm(which, C.byref(a), ptr(aw, C.c_uint64), C.byref(b), ptr(bw, C.c_uint64), variant, 0,
                      ptr(t, C.c_double), ptr(k, C.c_uint8), n, out.ctypes.data_as(C.c_void_p)))
    return out


def gen_bmm():
    """test_bmm.cpp:41-137 shapes and cases."""
    out = {}
    shapes = [(1, 1, 1), (3, 257, 5), (8, 1024, 8), (17, 384, 33), (5, 100, 7), (31, 130, 12), (9, 301, 14),
              (7, 150, 4), (6, 256, 9), (64, 1024, 96)]
    for idx, (m, n, k) in enumerate(shapes):
        fa = normal_floats(1000 + idx, m * n)
        fb = normal_floats(2000 + idx, n * k)
        A = ref_pack_matrix(fa, m, n, capi.ROW_PACKED)
        B = ref_pack_matrix(fb.reshape(n, k), n, k, capi.COL_PACKED)
        da, db = capi.MatrixDesc(m, n, capi.ROW_PACKED, 8, 128), capi.MatrixDesc(n, k, capi.COL_PACKED, 8, 128)
        p = f"s{idx}_"
        out[p + "shape"] = np.array([m, n, k])
        out[p + "fa"], out[p + "fb"], out[p + "A"], out[p + "B"] = fa, fb, A, B
        out[p + "pm1"] = ref_bmm(1, da, A, db, B, capi.BMM_BLOCKED)
        if n % 128 == 0:
            out[p + "raw"] = ref_bmm(0, da, A, db, B, capi.BMM_NAIVE)
        out[p + "bin"] = ref_bmm(2, da, A, db, B, capi.BMM_BLOCKED)
        # per-column thresholds cycling through the four kinds (test_bmm.cpp:120-137)
        tau = np.array([(3.0, -2.0, 0.0, 0.0)[j % 4] + (j // 4) for j in range(k)], dtype=np.float64)
        kind = np.array([j % 4 for j in range(k)], dtype=np.uint8)
        out[p + "tau"], out[p + "kind"] = tau, kind
        out[p + "bin_thr"] = ref_bmm(2, da, A, db, B, capi.BMM_BLOCKED, tau, kind)
        Af, dfa = ref_to_fsb(da, A)
        Bf, dfb = ref_to_fsb(db, B)
        out[p + "Afsb"], out[p + "Bfsb"] = Af, Bf
        out[p + "bin_fsb"] = ref_bmm(2, dfa, Af, dfb, Bf, capi.BMM_FSB, tau, kind)
    np.savez_compressed(os.path.join(HERE, "bmm.npz"), **out)


def _act(h, w, n, c, tiled):
    return capi.ActDesc(h, w, n, c, int(tiled), 8, 128)


def gen_bconv():
    """test_bconv.cpp:59-152 cases: pm1, fused threshold/bn, residual tap and injection."""
    out = {}
    cases = [(8, 8, 3, 64, 32, 3, 1, 1), (7, 9, 2, 130, 5, 3, 1, 1), (8, 8, 1, 128, 128, 3, 2, 1),
             (5, 5, 2, 16, 8, 5, 2, 2), (4, 4, 2, 32, 16, 1, 1, 0), (6, 6, 16, 128, 16, 3, 1, 0),
             (9, 9, 2, 3, 4, 7, 4, 3), (6, 6, 3, 64, 24, 3, 1, 1), (4, 4, 2, 32, 32, 3, 1, 1),
             (14, 14, 5, 256, 72, 3, 2, 1)]
    for idx, (h, w, n, c, o, k, s, pd) in enumerate(cases):
        x = normal_floats(3000 + idx, n * h * w * c)
        wt = normal_floats(4000 + idx, k * k * o * c)
        p = f"c{idx}_"
        out[p + "case"] = np.array([h, w, n, c, o, k, s, pd])
        out[p + "x"], out[p + "wt"] = x, wt
        geo = capi.ConvGeom(k, k, s, pd)
        P, Q = (h + 2 * pd - k) // s + 1, (w + 2 * pd - k) // s + 1
        for tiled in (0, 1):
            t = "t" if tiled else "p"
            ad = _act(h, w, n, c, tiled)
            fd = capi.FilterDesc(k, k, o, c, tiled, 8, 128)
            aw = np.zeros(sum([0]) or 1, dtype=np.uint64)
            from paper_2006_16578_b200.weights import act_words, filter_words
            aw = np.zeros(act_words(h, w, n, c, tiled), dtype=np.uint64)
            fw = np.zeros(filter_words(k, k, o, c, tiled), dtype=np.uint64)
            _st(ref().ref_pack_nhwc(ptr(x, C.c_float), n, h, w, c, tiled, 8, 128, ptr(aw, C.c_uint64)))
            _st(ref().ref_pack_filter(ptr(wt, C.c_float), k, k, o, c, tiled, 8, 128, ptr(fw, C.c_uint64)))
            out[p + t + "_act"], out[p + t + "_filt"] = aw, fw
            if not tiled:
                v = np.zeros(P * Q * n * o, dtype=np.int32)
                _st(ref().ref_bconv_pm1(C.byref(ad), ptr(aw, C.c_uint64), C.byref(fd), ptr(fw, C.c_uint64), C.byref(geo),
                                        0, ptr(v, C.c_int32)))
                out[p + "pm1"] = v
            # bn params like test_bconv.cpp:88-117 (gamma = 0 on every 7th channel)
            rng = np.random.default_rng(5000 + idx)
            gamma = np.where(np.arange(o) % 7 == 0, 0.0, rng.standard_normal(o))
            beta, mean, var = rng.standard_normal(o), rng.standard_normal(o) * 10.0, rng.uniform(0.0, 2.0, o)
            out[p + "bn"] = np.stack([gamma, beta, mean, var])
            tau = np.zeros(o)
            kind = np.zeros(o, dtype=np.uint8)
            for j in range(o):
                tt, kk = C.c_double(), C.c_uint8()
                ref().ref_fold_bn_sign(gamma[j], beta[j], mean[j], var[j], 1e-5, C.byref(tt), C.byref(kk))
                tau[j], kind[j] = tt.value, kk.value
            out[p + "tau"], out[p + "kind"] = tau, kind
            words = act_words(P, Q, n, o, tiled)
            bits_thr = np.zeros(words, dtype=np.uint64)
            f = capi.ConvFused()
            f.tau, f.kind, f.n_thresholds = ptr(tau, C.c_double), ptr(kind, C.c_uint8), o
            _st(ref().ref_bconv_fused(C.byref(ad), ptr(aw, C.c_uint64), C.byref(fd), ptr(fw, C.c_uint64), C.byref(geo),
                                      C.byref(f), ptr(bits_thr, C.c_uint64)))
            out[p + t + "_bits_thr"] = bits_thr
            g, b, mu, vv = (np.ascontiguousarray(a) for a in (gamma, beta, mean, var))
            bn = capi.Bn(ptr(g, C.c_double), ptr(b, C.c_double), ptr(mu, C.c_double), ptr(vv, C.c_double), o, 1e-5)
            rin = normal_floats(6000 + idx, P * Q * n * o).astype(np.float64) * 3.0
            out[p + "rin"] = rin
            rout = np.zeros(P * Q * n * o)
            bits_bn = np.zeros(words, dtype=np.uint64)
            f2 = capi.ConvFused()
            f2.bn = C.pointer(bn)
            f2.residual_in = ptr(rin, C.c_double)
            f2.residual_out = ptr(rout, C.c_double)
            _st(ref().ref_bconv_fused(C.byref(ad), ptr(aw, C.c_uint64), C.byref(fd), ptr(fw, C.c_uint64), C.byref(geo),
                                      C.byref(f2), ptr(bits_bn, C.c_uint64)))
            out[p + t + "_bits_bn"], out[p + t + "_rout"] = bits_bn, rout
    np.savez_compressed(os.path.join(HERE, "bconv.npz"), **out)


def gen_first_conv_pool():
    out = {}
    cases = [(2, 9, 9, 3, 12, 5, 2, 2), (2, 30, 30, 3, 64, 7, 4, 3), (1, 23, 23, 3, 32, 11, 4, 5), (3, 8, 8, 2, 6, 3, 1, 1)]
    for idx, (n, h, w, c, o, k, s, pd) in enumerate(cases):
        x = normal_floats(7000 + idx, n * h * w * c)
        wpm = np.where(normal_floats(7100 + idx, o * k * k * c) >= 0, 1.0, -1.0).astype(np.float32)
        P, Q = (h + 2 * pd - k) // s + 1, (w + 2 * pd - k) // s + 1
        y = np.zeros(P * Q * n * o)
        geo = capi.ConvGeom(k, k, s, pd)
        _st(ref().ref_first_conv_bwn(ptr(x, C.c_float), n, h, w, c, ptr(wpm, C.c_float), wpm.size, k, k, o, C.byref(geo),
                                     0, ptr(y, C.c_double)))
        p = f"f{idx}_"
        out[p + "case"], out[p + "x"], out[p + "w"], out[p + "y"] = np.array([n, h, w, c, o, k, s, pd]), x, wpm, y
    # or_pool (test_bconv.cpp:212-247)
    from paper_2006_16578_b200.weights import act_words
    for idx, (h, w, n, c, win, st, tiled) in enumerate([(6, 6, 3, 130, 2, 2, 0), (6, 6, 3, 130, 2, 2, 1),
                                                       (7, 7, 2, 64, 3, 2, 0), (8, 8, 9, 256, 2, 2, 0)]):
        words = np.zeros(act_words(h, w, n, c, tiled), dtype=np.uint64)
        x = normal_floats(8000 + idx, n * h * w * c)
        _st(ref().ref_pack_nhwc(ptr(x, C.c_float), n, h, w, c, tiled, 8, 128, ptr(words, C.c_uint64)))
        oh, ow = (h - win) // st + 1, (w - win) // st + 1
        o = np.zeros(act_words(oh, ow, n, c, tiled), dtype=np.uint64)
        _st(ref().ref_or_pool(C.byref(_act(h, w, n, c, tiled)), ptr(words, C.c_uint64), win, st, 0, ptr(o, C.c_uint64)))
        p = f"p{idx}_"
        out[p + "case"], out[p + "in"], out[p + "out"] = np.array([h, w, n, c, win, st, tiled]), words, o
    np.savez_compressed(os.path.join(HERE, "first_conv_pool.npz"), **out)


SPEC_FIELDS = ["kind", "kh", "kw", "out_channels", "stride", "pad", "window", "pool_stride", "units", "in_h", "in_w",
               "in_channels", "out_h", "out_w", "residual_out", "residual_in", "shortcut_from"]


def dump_model(prefix, rm: RefModel, rw: RefWeights, out: dict):
    v = rm.view
    out[prefix + "hdr"] = np.array([v.in_h, v.in_w, v.in_c, v.classes, v.n_layers])
    out[prefix + "eps"] = np.array([v.epsilon])
    out[prefix + "specs"] = np.array([[getattr(v.layers[i], f) for f in SPEC_FIELDS] for i in range(v.n_layers)],
                                     dtype=np.int64)
    s = rw.store
    out[prefix + "store"] = np.array([s.tiled, s.bh, s.bw])
    for i in range(s.n_layers):
        L = s.layers[i]
        q = f"{prefix}L{i}_"
        if L.filter_n_words:
            out[q + "filter"] = np.ctypeslib.as_array(L.filter_words, (L.filter_n_words,)).copy()
        if L.conv_pm1_n:
            out[q + "conv_pm1"] = np.ctypeslib.as_array(L.conv_pm1, (L.conv_pm1_n,)).copy()
        if L.fc_n_words:
            out[q + "fc"] = np.ctypeslib.as_array(L.fc_words, (L.fc_n_words,)).copy()
        if L.n_thresholds:
            out[q + "tau"] = np.ctypeslib.as_array(L.tau, (L.n_thresholds,)).copy()
            out[q + "tkind"] = np.ctypeslib.as_array(L.tkind, (L.n_thresholds,)).copy()
        if L.has_bn:
            ch = L.bn.channels
            out[q + "bn"] = np.stack([np.ctypeslib.as_array(getattr(L.bn, f), (ch,)).copy()
                                      for f in ("gamma", "beta", "mean", "var")])


MODELS = [  # test_nn.cpp:280-307, plus a ResNet-style and the stock shapes at small size
    ("cpf", "6C3-P2-12FC", 8, 8, 2, 4, [], 101, 5),
    ("strided", "8C5/2-8C3-16FC", 16, 16, 3, 5, [], 103, 4),
    ("mlp", "3x24FC", 4, 4, 1, 10, [], 107, 9),
    ("headless", "6C3-P2", 8, 8, 2, 4, [], 109, 6),
    ("res-a", "4C3-4C3-4C3-8FC", 8, 8, 2, 3, [(0, 2)], 113, 5),
    ("res-b", "4C3-4C3-4C3-8C3/2-8C3-8C3", 8, 8, 2, 3, [(0, 2), (2, 4)], 127, 4),
    ("res18-32", "64C7/4-4x64C3-128C3/2-3x128C3-256C3/2-3x256C3-512C3/2-3x512C3-(2x512FC)", 64, 64, 3, 1000,
     [(a, a + 2) for a in range(0, 16, 2)], 131, 3),
    ("mlp-mnist", "1024FC-1024FC-1024FC-1024FC", 28, 28, 1, 10, [], 137, 16),
]


def gen_models():
    out = {}
    for mi, (name, tokens, h, w, c, classes, sc, seed, batch) in enumerate(MODELS):
        rm = RefModel.make(name, tokens, h, w, c, classes, sc)
        for tiled in (0, 1):
            rw = RefWeights(rm, seed * 77 + 1, tiled=bool(tiled))
            p = f"m{mi}{'t' if tiled else 'p'}_"
            dump_model(p, rm, rw, out)
            x = normal_floats(seed, batch * h * w * c).reshape(batch, h, w, c)
            lg, lb = rw.run_inference(x)
            lg2, lb2 = rw.pipeline(x)
            assert np.array_equal(lg, lg2) and np.array_equal(lb, lb2), name
            out[p + "x"], out[p + "logits"], out[p + "labels"] = x, lg, lb
        out[f"m{mi}_name"] = np.array(name)
    np.savez_compressed(os.path.join(HERE, "models.npz"), **out)


if __name__ == "__main__":
    assert ref() is not None, "oracle/_ref not built (make -C oracle)"
    gen_bmm()
    gen_bconv()
    gen_first_conv_pool()
    gen_models()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
