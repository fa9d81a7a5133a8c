"""Pins the C oracle (oracle/btnn_oracle.c) before it is trusted as the GPU checker:
(1) the reference's own known-answer tests, restated; (2) the golden fixtures produced
by the reference itself (tests/golden/make_golden.py); (3) live comparison against the
compiled reference (oracle/_ref) on fresh random cases when it is present.
"""
import ctypes as C
import math

import numpy as np
import pytest

from fixtures import fixture_models, indices, load
from oracle_lib import RefModel, RefWeights, normal_floats, oracle, oracle_run_inference, ptr, ref
from paper_2006_16578_b200 import capi

O = oracle


def u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


# ---------------------------------------------------------------- known answers
def test_pack_signs_mixed():  # test_bitcore.cpp:28-33
    out = np.zeros(1, dtype=np.uint64)
    v = np.array([1.0, -2.0, 3.5, -0.25], dtype=np.float32)
    assert O().bo_pack_signs_f32(ptr(v, C.c_float), 4, ptr(out, C.c_uint64)) == 0
    assert out[0] == 0x5


def test_pack_signs_zero_and_nonfinite():  # test_bitcore.cpp:35-53
    out = np.zeros(1, dtype=np.uint64)
    v = np.array([0.0, -0.0], dtype=np.float32)
    O().bo_pack_signs_f32(ptr(v, C.c_float), 2, ptr(out, C.c_uint64))
    assert out[0] == 0x3
    for bad in (np.array([1.0, np.nan], dtype=np.float32), np.array([np.inf], dtype=np.float32)):
        assert O().bo_pack_signs_f32(ptr(bad, C.c_float), bad.size, ptr(out, C.c_uint64)) == capi.BTNN_INVALID_INPUT
    neg = np.full(200, -1.0, dtype=np.float32)
    o4 = np.zeros(4, dtype=np.uint64)
    O().bo_pack_signs_f32(ptr(neg, C.c_float), 200, ptr(o4, C.c_uint64))
    assert not o4.any()


def test_dot_pm1_identical_opposite():  # test_bitcore.cpp:65-70
    rng = np.random.default_rng(7)
    a = rng.integers(0, 2**63, 2, dtype=np.uint64)
    inv = ~a
    assert O().bo_dot_pm1(ptr(a, C.c_uint64), ptr(a, C.c_uint64), 128) == 128
    assert O().bo_dot_pm1(ptr(a, C.c_uint64), ptr(inv, C.c_uint64), 128) == -128


def test_fsb_known_index():  # test_bitcore.cpp:107-114
    assert O().bo_bit_index(4, 8, capi.FSB_ROW, 2, 4, 0, 0) == 0
    assert O().bo_bit_index(4, 8, capi.FSB_ROW, 2, 4, 2, 5) == 25
    assert O().bo_bit_index(8, 4, capi.FSB_COL, 2, 4, 5, 2) == 25


def test_padded_dims():  # test_bitcore.cpp:123-136
    assert O().bo_matrix_words(10, 200, capi.ROW_PACKED, 8, 128) * 64 == 10 * 256
    assert O().bo_matrix_words(200, 10, capi.COL_PACKED, 8, 128) * 64 == 256 * 10
    assert O().bo_matrix_words(10, 200, capi.FSB_ROW, 8, 128) * 64 == 16 * 256
    assert O().bo_matrix_words(200, 10, capi.FSB_COL, 8, 128) * 64 == 256 * 16


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def test_ref_matmul_hand():  # test_oracle.cpp:25-37
    a, b = _f64([1, 2, 3, 4, 5, 6]), _f64([7, 8, 9, 10, 11, 12])
    out = np.zeros(4)
    O().bo_ref_matmul(ptr(a, C.c_double), ptr(b, C.c_double), 2, 3, 2, ptr(out, C.c_double))
    assert out.tolist() == [58, 64, 139, 154]
    a2, idm = _f64([1, -1, 1, 1, 1, -1]), _f64(np.eye(3).reshape(-1))
    out2 = np.zeros(6)
    O().bo_ref_matmul(ptr(a2, C.c_double), ptr(idm, C.c_double), 2, 3, 3, ptr(out2, C.c_double))
    assert out2.tolist() == a2.tolist()


def test_ref_conv_hand():  # test_oracle.cpp:44-61
    x, w = _f64(np.ones(9)), _f64(np.ones(9))
    out = np.zeros(9)
    assert O().bo_ref_conv_zero_pad(ptr(x, C.c_double), 1, 3, 3, 1, ptr(w, C.c_double), 1, 3, 3, 1, 1,
                                    ptr(out, C.c_double)) == 0
    assert out.tolist() == [4, 6, 4, 6, 9, 6, 4, 6, 4]
    x2, w2 = _f64([1, 2, 3, 4]), _f64([1, 1])
    out2 = np.zeros(2)
    O().bo_ref_conv_zero_pad(ptr(x2, C.c_double), 1, 1, 4, 1, ptr(w2, C.c_double), 1, 1, 2, 2, 0, ptr(out2, C.c_double))
    assert out2.tolist() == [3, 7]
    x3, w3 = _f64(np.ones(4)), _f64(np.ones(9))
    assert O().bo_ref_conv_zero_pad(ptr(x3, C.c_double), 1, 2, 2, 1, ptr(w3, C.c_double), 1, 3, 3, 1, 0,
                                    ptr(out, C.c_double)) == capi.BTNN_INVALID_INPUT


def test_ref_pool_fc_htanh():  # test_oracle.cpp:70-101
    x = _f64([-1, 1, -1, -1])
    out = np.zeros(1)
    O().bo_ref_max_pool(ptr(x, C.c_double), 2, 2, 1, 1, 2, 2, ptr(out, C.c_double))
    assert out[0] == 1.0
    x9 = _f64(np.ones(9))
    assert O().bo_ref_max_pool(ptr(x9, C.c_double), 3, 3, 1, 1, 2, 2, ptr(out, C.c_double)) == capi.BTNN_INVALID_INPUT
    xf, wf = _f64([1, -1, 1, -1, -1, 1]), _f64([1, 1, 1, -1, 1, -1])
    of = np.zeros(4)
    O().bo_ref_fc(ptr(xf, C.c_double), 2, 3, ptr(wf, C.c_double), 2, ptr(of, C.c_double))
    assert of.tolist() == [1, -3, -1, -1]
    assert O().bo_ref_htanh(3.5) == 1.0 and O().bo_ref_htanh(-3.5) == -1.0 and O().bo_ref_htanh(0.25) == 0.25


def test_corner_excludes():  # test_bconv.cpp:74-86
    c = 96
    from paper_2006_16578_b200.weights import act_words, filter_words, pack_filter, pack_nhwc
    aw = pack_nhwc(np.ones((1, 6, 6, c), dtype=np.float32))
    fw = pack_filter(np.ones(3 * 3 * 2 * c, dtype=np.float32), 3, 3, 2, c)
    assert aw.size == act_words(6, 6, 1, c) and fw.size == filter_words(3, 3, 2, c)
    out = np.zeros(6 * 6 * 1 * 2, dtype=np.int32)
    ad, fd, g = capi.ActDesc(6, 6, 1, c, 0, 8, 128), capi.FilterDesc(3, 3, 2, c, 0, 8, 128), capi.ConvGeom(3, 3, 1, 1)
    assert O().bo_bconv_pm1(C.byref(ad), ptr(aw, C.c_uint64), C.byref(fd), ptr(fw, C.c_uint64), C.byref(g),
                            ptr(out, C.c_int32)) == 0
    v = out.reshape(6, 6, 1, 2)
    assert v[0, 0, 0, 0] == 4 * c and v[0, 1, 0, 0] == 6 * c and v[1, 1, 0, 0] == 9 * c


def test_fold_direction_and_zero_gamma():  # test_nn.cpp:53-79
    t, k = C.c_double(), C.c_uint8()
    O().bo_fold_bn_sign(2.0, 1.0, 10.0, 1.0, 1e-5, C.byref(t), C.byref(k))
    assert k.value == capi.GEQ and O().bo_fire(t.value, k.value, 100.0) and not O().bo_fire(t.value, k.value, -100.0)
    O().bo_fold_bn_sign(-2.0, 1.0, 10.0, 1.0, 1e-5, C.byref(t), C.byref(k))
    assert k.value == capi.LEQ and not O().bo_fire(t.value, k.value, 100.0) and O().bo_fire(t.value, k.value, -100.0)
    O().bo_fold_bn_sign(0.0, 0.5, 0.0, 1.0, 1e-5, C.byref(t), C.byref(k))
    assert k.value == capi.CONST_PLUS and O().bo_fire(t.value, k.value, -1e9)
    O().bo_fold_bn_sign(0.0, -0.5, 0.0, 1.0, 1e-5, C.byref(t), C.byref(k))
    assert k.value == capi.CONST_MINUS and not O().bo_fire(t.value, k.value, 1e9)


def test_fold_matches_bn_sign_on_integers():  # test_nn.cpp:37-51
    rng = np.random.default_rng(31)
    g = rng.standard_normal(400)
    g[rng.random(400) < 0.1] = 0.0
    b, mu, var = rng.standard_normal(400), rng.standard_normal(400) * 8, rng.uniform(0.25, 2.0, 400)
    t, k = C.c_double(), C.c_uint8()
    for ch in range(400):
        O().bo_fold_bn_sign(g[ch], b[ch], mu[ch], var[ch], 1e-5, C.byref(t), C.byref(k))
        gg, bb, mm, vv = (_f64([x]) for x in (g[ch], b[ch], mu[ch], var[ch]))
        bn = capi.Bn(ptr(gg, C.c_double), ptr(bb, C.c_double), ptr(mm, C.c_double), ptr(vv, C.c_double), 1, 1e-5)
        for v in rng.integers(-4096, 4097, 50):
            assert O().bo_fire(t.value, k.value, float(v)) == (O().bo_bn_apply(C.byref(bn), 0, float(v)) >= 0.0)


# ---------------------------------------------------------------- golden fixtures
def _md(r, c, lay):
    return capi.MatrixDesc(int(r), int(c), lay, 8, 128)


@pytest.mark.parametrize("i", indices(load("bmm"), "s", "shape"))
def test_oracle_bmm_golden(i):
    d = load("bmm")
    m, n, k = (int(v) for v in d[f"s{i}_shape"])
    A, B = u64(d[f"s{i}_A"]), u64(d[f"s{i}_B"])
    da, db = _md(m, n, capi.ROW_PACKED), _md(n, k, capi.COL_PACKED)
    out = np.zeros(m * k, dtype=np.int32)
    assert O().bo_bmm_pm1(C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(B, C.c_uint64), capi.BMM_BLOCKED,
                          ptr(out, C.c_int32)) == 0
    assert np.array_equal(out, d[f"s{i}_pm1"])
    if f"s{i}_raw" in d:
        O().bo_bmm_raw(C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(B, C.c_uint64), capi.BMM_NAIVE, ptr(out, C.c_int32))
        assert np.array_equal(out, d[f"s{i}_raw"])
    bits = np.zeros(d[f"s{i}_bin"].size, dtype=np.uint64)
    tau, kind = _f64(d[f"s{i}_tau"]), np.ascontiguousarray(d[f"s{i}_kind"], dtype=np.uint8)
    O().bo_bmm_pm1_bin(C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(B, C.c_uint64), capi.BMM_BLOCKED, None, None, 0,
                       ptr(bits, C.c_uint64))
    assert np.array_equal(bits, d[f"s{i}_bin"])
    O().bo_bmm_pm1_bin(C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(B, C.c_uint64), capi.BMM_BLOCKED,
                       ptr(tau, C.c_double), ptr(kind, C.c_uint8), k, ptr(bits, C.c_uint64))
    assert np.array_equal(bits, d[f"s{i}_bin_thr"])
    Af, Bf = u64(d[f"s{i}_Afsb"]), u64(d[f"s{i}_Bfsb"])
    fb = np.zeros(d[f"s{i}_bin_fsb"].size, dtype=np.uint64)
    O().bo_bmm_pm1_bin(C.byref(_md(m, n, capi.FSB_ROW)), ptr(Af, C.c_uint64), C.byref(_md(n, k, capi.FSB_COL)),
                       ptr(Bf, C.c_uint64), capi.BMM_FSB, ptr(tau, C.c_double), ptr(kind, C.c_uint8), k, ptr(fb, C.c_uint64))
    assert np.array_equal(fb, d[f"s{i}_bin_fsb"])


@pytest.mark.parametrize("i", indices(load("bconv"), "c", "case"))
def test_oracle_bconv_golden(i):
    d = load("bconv")
    h, w, n, c, o, k, s, pd = (int(v) for v in d[f"c{i}_case"])
    P, Q = (h + 2 * pd - k) // s + 1, (w + 2 * pd - k) // s + 1
    g = capi.ConvGeom(k, k, s, pd)
    for tiled, t in ((0, "p"), (1, "t")):
        ad, fd = capi.ActDesc(h, w, n, c, tiled, 8, 128), capi.FilterDesc(k, k, o, c, tiled, 8, 128)
        aw, fw = u64(d[f"c{i}_{t}_act"]), u64(d[f"c{i}_{t}_filt"])
        v = np.zeros(P * Q * n * o, dtype=np.int32)
        assert O().bo_bconv_pm1(C.byref(ad), ptr(aw, C.c_uint64), C.byref(fd), ptr(fw, C.c_uint64), C.byref(g),
                                ptr(v, C.c_int32)) == 0
        assert np.array_equal(v, d[f"c{i}_pm1"]), t
        tau, kind = _f64(d[f"c{i}_tau"]), np.ascontiguousarray(d[f"c{i}_kind"], dtype=np.uint8)
        f = capi.ConvFused()
        f.tau, f.kind, f.n_thresholds = ptr(tau, C.c_double), ptr(kind, C.c_uint8), o
        bits = np.zeros(d[f"c{i}_{t}_bits_thr"].size, dtype=np.uint64)
        assert O().bo_bconv_fused(C.byref(ad), ptr(aw, C.c_uint64), C.byref(fd), ptr(fw, C.c_uint64), C.byref(g),
                                  C.byref(f), ptr(bits, C.c_uint64)) == 0
        assert np.array_equal(bits, d[f"c{i}_{t}_bits_thr"])
        bnp = [_f64(x) for x in d[f"c{i}_bn"]]
        bn = capi.Bn(*(ptr(x, C.c_double) for x in bnp), o, 1e-5)
        rin, rout = _f64(d[f"c{i}_rin"]), np.zeros(P * Q * n * o)
        f2 = capi.ConvFused()
        f2.bn, f2.residual_in, f2.residual_out = C.pointer(bn), ptr(rin, C.c_double), ptr(rout, C.c_double)
        O().bo_bconv_fused(C.byref(ad), ptr(aw, C.c_uint64), C.byref(fd), ptr(fw, C.c_uint64), C.byref(g), C.byref(f2),
                           ptr(bits, C.c_uint64))
        assert np.array_equal(bits, d[f"c{i}_{t}_bits_bn"])
        assert np.array_equal(rout.view(np.uint64), d[f"c{i}_{t}_rout"].view(np.uint64))


def test_oracle_first_conv_and_pool_golden():
    d = load("first_conv_pool")
    for i in indices(d, "f", "case"):
        n, h, w, c, o, k, s, pd = (int(v) for v in d[f"f{i}_case"])
        x, wp = np.ascontiguousarray(d[f"f{i}_x"], dtype=np.float32), np.ascontiguousarray(d[f"f{i}_w"], dtype=np.float32)
        y = np.zeros(d[f"f{i}_y"].size)
        g = capi.ConvGeom(k, k, s, pd)
        assert O().bo_first_conv_bwn(ptr(x, C.c_float), n, h, w, c, ptr(wp, C.c_float), k, k, o, C.byref(g),
                                     ptr(y, C.c_double)) == 0
        assert np.array_equal(y.view(np.uint64), d[f"f{i}_y"].view(np.uint64))
    for i in indices(d, "p", "case"):
        h, w, n, c, win, st, tiled = (int(v) for v in d[f"p{i}_case"])
        inp = u64(d[f"p{i}_in"])
        out = np.zeros(d[f"p{i}_out"].size, dtype=np.uint64)
        assert O().bo_or_pool(C.byref(capi.ActDesc(h, w, n, c, tiled, 8, 128)), ptr(inp, C.c_uint64), win, st,
                              ptr(out, C.c_uint64)) == 0
        assert np.array_equal(out, d[f"p{i}_out"])


@pytest.mark.parametrize("prefix,fm", fixture_models(), ids=lambda v: v if isinstance(v, str) else "")
def test_oracle_run_inference_golden(prefix, fm):
    if fm.in_h * fm.in_w >= 64 * 64 and "t_" in prefix:
        pytest.skip("large tiled case covered in plain layout (oracle is bit-serial)")
    lg, lb = oracle_run_inference(fm.spec, fm.store, fm.x)
    assert np.array_equal(lg.view(np.uint64), fm.logits.view(np.uint64))
    assert np.array_equal(lb, fm.labels)


# ---------------------------------------------------------------- live reference
needs_ref = pytest.mark.skipif(ref() is None, reason="oracle/_ref not built")


@needs_ref
def test_oracle_vs_reference_random_bmm():  # acceptance.cpp:56-99 in miniature
    rng = np.random.default_rng(99)
    for case in range(40):
        m, n, k = (int(v) for v in rng.integers(1, 200, 3))
        fa, fb = rng.standard_normal(m * n, dtype=np.float32), rng.standard_normal(n * k, dtype=np.float32)
        from paper_2006_16578_b200.weights import pack_matrix
        A, B = pack_matrix(fa, m, n, capi.ROW_PACKED), pack_matrix(fb, n, k, capi.COL_PACKED)
        da, db = _md(m, n, capi.ROW_PACKED), _md(n, k, capi.COL_PACKED)
        want = np.zeros(m * k, dtype=np.int32)
        got = np.zeros(m * k, dtype=np.int32)
        assert ref().ref_bmm(1, C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(B, C.c_uint64), capi.BMM_NAIVE, 1,
                             None, None, 0, want.ctypes.data_as(C.c_void_p)) == 0
        O().bo_bmm_pm1(C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(B, C.c_uint64), capi.BMM_NAIVE, ptr(got, C.c_int32))
        assert np.array_equal(want, got)
        dense = (np.where(fa >= 0, 1.0, -1.0).reshape(m, n) @ np.where(fb >= 0, 1.0, -1.0).reshape(n, k)).astype(np.int32)
        assert np.array_equal(dense.reshape(-1), got)


@needs_ref
def test_oracle_vs_reference_error_classes():  # test_bmm.cpp:156-174
    from paper_2006_16578_b200.weights import pack_matrix
    A = pack_matrix(np.ones(4 * 128, np.float32), 4, 128, capi.ROW_PACKED)
    Bs = pack_matrix(np.ones(64 * 4, np.float32), 64, 4, capi.COL_PACKED)
    out = np.zeros(64, dtype=np.int32)
    da, db = _md(4, 128, capi.ROW_PACKED), _md(64, 4, capi.COL_PACKED)
    r = ref().ref_bmm(1, C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(Bs, C.c_uint64), capi.BMM_BLOCKED, 1, None, None,
                      0, out.ctypes.data_as(C.c_void_p))
    o = O().bo_bmm_pm1(C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(Bs, C.c_uint64), capi.BMM_BLOCKED, ptr(out, C.c_int32))
    assert r == o == capi.BTNN_INVALID_INPUT


@needs_ref
def test_oracle_vs_reference_resnet_small():
    """The full stock ResNet-18 structure at 32x32: oracle == reference run_inference."""
    rm = RefModel.parse(open_model("resnet18", 32))
    rw = RefWeights(rm, 5)
    x = normal_floats(9, 2 * 32 * 32 * 3).reshape(2, 32, 32, 3)
    want, wl = rw.run_inference(x)
    got, gl = oracle_run_inference(rm.view, rw.store, x)
    assert np.array_equal(want.view(np.uint64), got.view(np.uint64)) and np.array_equal(wl, gl)


def open_model(name, hw):
    import json
    from paper_2006_16578_b200.model import STOCK
    doc = json.loads(json.dumps(STOCK[name]))
    doc["input"]["height"] = doc["input"]["width"] = hw
    return json.dumps(doc)
