"""GPU parity of the kernel-level C ABI: every output bit-exact against the reference's
golden fixtures and the C oracle, plus random sweeps in the style of acceptance.cpp
criteria 1, 2 and 6, and the reference's error classes."""
import ctypes as C

import numpy as np
import pytest

from fixtures import indices, load
from oracle_lib import oracle, ptr
from paper_2006_16578_b200 import btnn as B
from paper_2006_16578_b200 import capi
from paper_2006_16578_b200 import weights as Wt

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("engine")]


def md(r, c, lay, bh=8, bw=128):
    return capi.MatrixDesc(int(r), int(c), lay, bh, bw)


@pytest.mark.parametrize("i", indices(load("bmm"), "s", "shape"))
def test_bmm_golden(i):
    d = load("bmm")
    m, n, k = (int(v) for v in d[f"s{i}_shape"])
    da, db = md(m, n, capi.ROW_PACKED), md(n, k, capi.COL_PACKED)
    A, Bw = d[f"s{i}_A"], d[f"s{i}_B"]
    for variant in (capi.BMM_NAIVE, capi.BMM_BLOCKED):
        assert np.array_equal(B.bmm_pm1(da, A, db, Bw, variant).reshape(-1), d[f"s{i}_pm1"])
    if f"s{i}_raw" in d:
        assert np.array_equal(B.bmm_raw(da, A, db, Bw).reshape(-1), d[f"s{i}_raw"])
    assert np.array_equal(B.bmm_pm1_bin(da, A, db, Bw), d[f"s{i}_bin"])
    assert np.array_equal(B.bmm_pm1_bin(da, A, db, Bw, tau=d[f"s{i}_tau"], kind=d[f"s{i}_kind"]), d[f"s{i}_bin_thr"])
    got = B.bmm_pm1_bin(md(m, n, capi.FSB_ROW), d[f"s{i}_Afsb"], md(n, k, capi.FSB_COL), d[f"s{i}_Bfsb"], capi.BMM_FSB,
                        tau=d[f"s{i}_tau"], kind=d[f"s{i}_kind"])
    assert np.array_equal(got, d[f"s{i}_bin_fsb"])


def test_bmm_random_sweep_vs_oracle():  # acceptance.cpp criterion 1 (600 cases) in reduced form
    rng = np.random.default_rng(101)
    for case in range(120):
        m, n, k = (int(v) for v in rng.integers(1, 300, 3))
        if case % 10 == 0:
            n = int(rng.integers(1, 8)) * 128
        fa, fb = rng.standard_normal(m * n, dtype=np.float32), rng.standard_normal(n * k, dtype=np.float32)
        A, Bw = Wt.pack_matrix(fa, m, n, capi.ROW_PACKED), Wt.pack_matrix(fb, n, k, capi.COL_PACKED)
        da, db = md(m, n, capi.ROW_PACKED), md(n, k, capi.COL_PACKED)
        want = np.zeros(m * k, dtype=np.int32)
        oracle().bo_bmm_pm1(C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(Bw, C.c_uint64), capi.BMM_NAIVE,
                            ptr(want, C.c_int32))
        got = B.bmm_pm1(da, A, db, Bw).reshape(-1)
        assert np.array_equal(got, want), (m, n, k)
        dense = np.where(fa >= 0, 1, -1).reshape(m, n) @ np.where(fb >= 0, 1, -1).reshape(n, k)
        assert np.array_equal(got, dense.reshape(-1).astype(np.int32))


def test_bmm_1024_cube():
    """The BASELINE config: 1024^3 on random packed words (bench.hpp:76-87), vs the oracle."""
    rng = np.random.default_rng(1)
    A = rng.integers(0, 2**64, 1024 * 16, dtype=np.uint64)
    Bw = rng.integers(0, 2**64, 1024 * 16, dtype=np.uint64)
    da, db = md(1024, 1024, capi.ROW_PACKED), md(1024, 1024, capi.COL_PACKED)
    want = np.zeros(1024 * 1024, dtype=np.int32)
    oracle().bo_bmm_pm1(C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(Bw, C.c_uint64), capi.BMM_NAIVE,
                        ptr(want, C.c_int32))
    assert np.array_equal(B.bmm_pm1(da, A, db, Bw).reshape(-1), want)
    raw = B.bmm_raw(da, A, db, Bw).reshape(-1)
    assert np.array_equal(1024 - 2 * raw, want)


@pytest.mark.parametrize("m,n,k", [(300, 700, 1536), (1000, 65, 1200), (129, 1, 33), (1, 129, 1408), (130, 131, 1537)])
def test_bmm_packed_kernel_shapes(m, n, k, engine):
    """The whole-K packed BMM (bmm_tc.cu) over tile edges in M and N, inner dimensions up to
    its 1536-bit limit (partial last words, odd chunk counts), and past it (the K-pipelined
    kernel): pm1, raw and thresholded bits vs the C oracle."""
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    fa, fb = rng.standard_normal(m * k, dtype=np.float32), rng.standard_normal(k * n, dtype=np.float32)
    A, Bw = Wt.pack_matrix(fa, m, k, capi.ROW_PACKED), Wt.pack_matrix(fb, k, n, capi.COL_PACKED)
    da, db = md(m, k, capi.ROW_PACKED), md(k, n, capi.COL_PACKED)
    want = np.zeros(m * n, dtype=np.int32)
    oracle().bo_bmm_pm1(C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(Bw, C.c_uint64), capi.BMM_NAIVE,
                        ptr(want, C.c_int32))
    assert np.array_equal(B.bmm_pm1(da, A, db, Bw).reshape(-1), want), (m, n, k)
    if engine == "tc":
        assert capi.last_tc_launch()[0] == ("bmm_packed/i32" if k <= 1536 else "bmm_pipe/i32"), capi.last_tc_launch()
    if k % 128 == 0:
        assert np.array_equal(k - 2 * B.bmm_raw(da, A, db, Bw).reshape(-1), want)
    bits = B.bmm_pm1_bin(da, A, db, Bw)
    dense = (want.reshape(m, n) >= 0)
    words = np.zeros((m, (n + 127) // 128 * 2), dtype=np.uint64)
    for j in range(n):
        words[:, j // 64] |= dense[:, j].astype(np.uint64) << np.uint64(j % 64)
    assert np.array_equal(np.asarray(bits).reshape(-1), words.reshape(-1))


@pytest.fixture(params=["pre", "in-kernel"])
def pipelined(request):
    """The K-pipelined packed BMM, with B pre-expanded for 128 x 256 tiles or always in-kernel."""
    capi.set_bmm_kernel(capi.BMM_PIPELINED if request.param == "pre" else capi.BMM_PIPELINED_NO_PRE)
    yield
    capi.set_bmm_kernel(capi.BMM_AUTO)


@pytest.mark.parametrize("i", indices(load("bmm"), "s", "shape"))
def test_bmm_golden_pipelined(i, pipelined, engine):
    """The reference's BMM golden cases (plain and fsb, four threshold kinds) on the K-pipelined kernel."""
    test_bmm_golden(i)
    if engine == "tc":
        assert capi.last_tc_launch()[0].startswith("bmm_pipe/"), capi.last_tc_launch()


def test_bmm_random_sweep_pipelined(pipelined):
    test_bmm_random_sweep_vs_oracle()


@pytest.mark.parametrize("m,n,k", [(300, 700, 1536), (129, 1, 33), (1, 129, 1408), (130, 131, 1537), (257, 300, 4160),
                                   (1024, 1100, 9216), (512, 512, 25088), (96, 2000, 4097), (8192, 1200, 300), (8192, 2304, 1100)])
def test_bmm_pipelined_shapes(m, n, k, pipelined, engine):
    """K-pipelined packed BMM: tile edges in M and N (128 x 64 and 128 x 128 tiles), K-step
    counts below and above the ring and prefetch depths, partial last words; pm1, raw and
    thresholded bits (random tau, all four kinds) vs the C oracle."""
    rng = np.random.default_rng(m * 5 + n * 11 + k)
    wpr = (k + 127) // 128 * 2  # words per packed row / column; bits past K are zero

    def packed(rows):
        w = rng.integers(0, 2**64, (rows, wpr), dtype=np.uint64)
        bit = np.arange(wpr * 64).reshape(wpr, 64)
        keep = (np.uint64(1) << np.arange(64, dtype=np.uint64))[None, :] * (bit < k)
        w &= np.bitwise_or.reduce(keep.astype(np.uint64), axis=1)[None, :]
        return w.reshape(-1)

    A, Bw = packed(m), packed(n)
    da, db = md(m, k, capi.ROW_PACKED), md(k, n, capi.COL_PACKED)
    want = np.zeros(m * n, dtype=np.int32)
    assert oracle().bo_bmm_pm1(C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(Bw, C.c_uint64), capi.BMM_NAIVE,
                               ptr(want, C.c_int32)) == 0
    assert np.array_equal(B.bmm_pm1(da, A, db, Bw).reshape(-1), want), (m, n, k)
    if engine == "tc":
        assert capi.last_tc_launch()[0].startswith("bmm_pipe") and capi.last_tc_launch()[0].endswith("/i32")
    if k % 128 == 0:  # (bmm_raw: the reference requires whole 128-bit words)
        assert np.array_equal(B.bmm_raw(da, A, db, Bw).reshape(-1), (k - want) // 2)
    tau = rng.standard_normal(n) * 30
    kind = rng.integers(0, 4, n).astype(np.uint8)
    bits = B.bmm_pm1_bin(da, A, db, Bw, tau=tau, kind=kind)
    wbits = np.zeros_like(bits)
    assert oracle().bo_bmm_pm1_bin(C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(Bw, C.c_uint64), capi.BMM_NAIVE,
                                   ptr(np.ascontiguousarray(tau), C.c_double), ptr(kind, C.c_uint8), n,
                                   ptr(wbits, C.c_uint64)) == 0
    assert np.array_equal(bits, wbits)


@pytest.mark.parametrize("i", indices(load("bconv"), "c", "case"))
def test_bconv_golden(i):
    d = load("bconv")
    h, w, n, c, o, k, s, pd = (int(v) for v in d[f"c{i}_case"])
    g = capi.ConvGeom(k, k, s, pd)
    bn = tuple(d[f"c{i}_bn"])
    for tiled, t in ((0, "p"), (1, "t")):
        ad, fd = capi.ActDesc(h, w, n, c, tiled, 8, 128), capi.FilterDesc(k, k, o, c, tiled, 8, 128)
        aw, fw = d[f"c{i}_{t}_act"], d[f"c{i}_{t}_filt"]
        assert np.array_equal(B.bconv_pm1(ad, aw, fd, fw, g), d[f"c{i}_pm1"]), t
        bits, _ = B.bconv_fused(ad, aw, fd, fw, g, tau=d[f"c{i}_tau"], kind=d[f"c{i}_kind"])
        assert np.array_equal(bits, d[f"c{i}_{t}_bits_thr"]), t
        bits, rout = B.bconv_fused(ad, aw, fd, fw, g, bn=bn, residual_in=d[f"c{i}_rin"], want_residual_out=True)
        assert np.array_equal(bits, d[f"c{i}_{t}_bits_bn"]), t
        assert np.array_equal(rout.view(np.uint64), d[f"c{i}_{t}_rout"].view(np.uint64)), t


def test_bconv_random_sweep_vs_oracle():  # acceptance.cpp criterion 2 (K, stride, pad sweep)
    rng = np.random.default_rng(202)
    for case in range(60):
        k = int(rng.choice([1, 3, 5, 7, 11]))
        s = int(rng.choice([1, 2, 4]))
        pd = int(rng.choice([0, 1, 2, 5]))
        h = int(rng.integers(max(1, k - 2 * pd), 16))
        w = int(rng.integers(max(1, k - 2 * pd), 16))
        n, c, o = int(rng.integers(1, 6)), int(rng.integers(1, 200)), int(rng.integers(1, 80))
        x = rng.standard_normal((n, h, w, c), dtype=np.float32)
        wt = rng.standard_normal(k * k * o * c, dtype=np.float32)
        aw, fw = Wt.pack_nhwc(x), Wt.pack_filter(wt, k, k, o, c)
        ad, fd, g = capi.ActDesc(h, w, n, c, 0, 8, 128), capi.FilterDesc(k, k, o, c, 0, 8, 128), capi.ConvGeom(k, k, s, pd)
        P, Q = (h + 2 * pd - k) // s + 1, (w + 2 * pd - k) // s + 1
        want = np.zeros(P * Q * n * o, dtype=np.int32)
        assert oracle().bo_bconv_pm1(C.byref(ad), ptr(aw, C.c_uint64), C.byref(fd), ptr(fw, C.c_uint64), C.byref(g),
                                     ptr(want, C.c_int32)) == 0
        assert np.array_equal(B.bconv_pm1(ad, aw, fd, fw, g), want), (h, w, n, c, o, k, s, pd)


def test_bconv_corner_excludes():  # test_bconv.cpp:74-86
    c = 96
    aw = Wt.pack_nhwc(np.ones((1, 6, 6, c), np.float32))
    fw = Wt.pack_filter(np.ones(3 * 3 * 2 * c, np.float32), 3, 3, 2, c)
    v = B.bconv_pm1(capi.ActDesc(6, 6, 1, c, 0, 8, 128), aw, capi.FilterDesc(3, 3, 2, c, 0, 8, 128),
                    fw, capi.ConvGeom(3, 3, 1, 1)).reshape(6, 6, 1, 2)
    assert v[0, 0, 0, 0] == 4 * c and v[0, 1, 0, 0] == 6 * c and v[1, 1, 0, 0] == 9 * c


def test_first_conv_and_pool_golden():
    d = load("first_conv_pool")
    for i in indices(d, "f", "case"):
        n, h, w, c, o, k, s, pd = (int(v) for v in d[f"f{i}_case"])
        y = B.first_conv_bwn(d[f"f{i}_x"].reshape(n, h, w, c), d[f"f{i}_w"], k, k, o, capi.ConvGeom(k, k, s, pd))
        assert np.array_equal(y.view(np.uint64), d[f"f{i}_y"].view(np.uint64)), i
    for i in indices(d, "p", "case"):
        h, w, n, c, win, st, tiled = (int(v) for v in d[f"p{i}_case"])
        out = B.or_pool(capi.ActDesc(h, w, n, c, tiled, 8, 128), d[f"p{i}_in"], win, st)
        assert np.array_equal(out, d[f"p{i}_out"]), i


def test_format_stage_vs_harness_packers():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((3, 5, 7, 130), dtype=np.float32)
    x[0, 0, 0, :4] = [0.0, -0.0, 1.0, -1.0]
    for tiled in (False, True):
        assert np.array_equal(B.pack_nhwc(x, tiled), Wt.pack_nhwc(x, tiled))
    v = rng.standard_normal(17 * 300, dtype=np.float32)
    for lay in range(4):
        assert np.array_equal(B.pack_matrix(v, 17, 300, lay), Wt.pack_matrix(v, 17, 300, lay)), lay
    A = Wt.pack_matrix(v, 17, 300, capi.ROW_PACKED)
    # test_bitcore.cpp:168-183 round trips; widths 32 / 96 take the bit-by-bit conversion
    # path, multiples of 64 the whole-word one
    for geo in ((8, 128), (4, 64), (2, 256), (16, 128), (4, 32), (2, 96)):
        f = B.to_fsb(md(17, 300, capi.ROW_PACKED), A, *geo)
        assert np.array_equal(f, Wt.pack_matrix(v, 17, 300, capi.FSB_ROW, *geo))
        assert np.array_equal(B.from_fsb(md(17, 300, capi.FSB_ROW, *geo), f), A)
    ad = capi.ActDesc(5, 7, 3, 130, 0, 8, 128)
    aw = Wt.pack_nhwc(x)
    assert np.array_equal(B.convert_activations(ad, aw, True), Wt.pack_nhwc(x, True))
    for geo in ((8, 128), (4, 64), (2, 32)):  # tiled -> plain and back, word and bit paths
        t = B.convert_activations(ad, aw, True, *geo)
        assert np.array_equal(t, Wt.pack_nhwc(x, True, *geo)), geo
        assert np.array_equal(B.convert_activations(capi.ActDesc(5, 7, 3, 130, 1, *geo), t, False), aw), geo
    # column layouts: ColPacked <-> fsb_col
    Bc = Wt.pack_matrix(v, 17, 300, capi.COL_PACKED)
    for geo in ((8, 128), (2, 64), (4, 32)):
        f = B.to_fsb(md(17, 300, capi.COL_PACKED), Bc, *geo)
        assert np.array_equal(f, Wt.pack_matrix(v, 17, 300, capi.FSB_COL, *geo)), geo
        assert np.array_equal(B.from_fsb(md(17, 300, capi.FSB_COL, *geo), f), Bc), geo
    flat = x.reshape(3, -1)
    assert np.array_equal(B.flatten_to_matrix(ad, aw, capi.ROW_PACKED), Wt.pack_matrix(flat, 3, flat.shape[1], capi.ROW_PACKED))
    bad = x.copy()
    bad[1, 2, 3, 4] = np.nan
    with pytest.raises(capi.BtnnError) as e:
        B.pack_nhwc(bad)
    assert e.value.code == capi.BTNN_INVALID_INPUT


def test_fused_equals_unfused():  # acceptance.cpp criterion 6 in reduced form
    rng = np.random.default_rng(66)
    for case in range(20):
        h = w = int(rng.integers(3, 12))
        n, c, o = int(rng.integers(1, 9)), int(rng.integers(1, 300)), int(rng.integers(1, 130))
        k, s = int(rng.choice([1, 3, 5])), int(rng.choice([1, 2]))
        pd = k // 2
        x = rng.standard_normal((n, h, w, c), dtype=np.float32)
        wt = rng.standard_normal(k * k * o * c, dtype=np.float32)
        ad, fd, g = capi.ActDesc(h, w, n, c, 0, 8, 128), capi.FilterDesc(k, k, o, c, 0, 8, 128), capi.ConvGeom(k, k, s, pd)
        aw, fw = Wt.pack_nhwc(x), Wt.pack_filter(wt, k, k, o, c)
        P, Q = (h + 2 * pd - k) // s + 1, (w + 2 * pd - k) // s + 1
        v = B.bconv_pm1(ad, aw, fd, fw, g).reshape(P, Q, n, o)
        gamma, beta = rng.standard_normal(o), rng.standard_normal(o)
        mean, var = rng.standard_normal(o) * 5, rng.uniform(0.25, 2.0, o)
        tau, kind = Wt.fold_bn_sign(gamma, beta, mean, var, 1e-5)
        bits, _ = B.bconv_fused(ad, aw, fd, fw, g, tau=tau, kind=kind)
        want = Wt.bn_apply(v, gamma, beta, mean, var, 1e-5) >= 0
        got = Wt.unpack_act(bits, P, Q, n, o)
        assert np.array_equal(got.transpose(0, 1, 2, 3), want)
        rin = rng.standard_normal(P * Q * n * o)
        bits2, rout = B.bconv_fused(ad, aw, fd, fw, g, bn=(gamma, beta, mean, var), residual_in=rin, want_residual_out=True)
        y = Wt.bn_apply(v, gamma, beta, mean, var, 1e-5).reshape(-1) + rin
        assert np.array_equal(rout.view(np.uint64), y.view(np.uint64))
        assert np.array_equal(Wt.unpack_act(bits2, P, Q, n, o).reshape(-1), (y >= 0))


def test_error_classes_match_reference():  # test_bmm.cpp:156-174, test_bconv.cpp:330-361
    a = md(4, 128, capi.ROW_PACKED)
    A = np.zeros(8, np.uint64)
    with pytest.raises(capi.BtnnError) as e:
        B.bmm_pm1_bin(a, A, md(128, 4, capi.COL_PACKED), A, tau=np.zeros(3), kind=np.zeros(3))
    assert e.value.code == capi.BTNN_INVALID_INPUT
    with pytest.raises(capi.BtnnError) as e:
        B.bmm_pm1(md(4, 128, capi.FSB_ROW), np.zeros(16, np.uint64), md(128, 4, capi.COL_PACKED), A, capi.BMM_FSB)
    assert e.value.code == capi.BTNN_INVALID_INPUT
    ad, g = capi.ActDesc(4, 4, 1, 16, 0, 8, 128), capi.ConvGeom(3, 3, 1, 1)
    fd = capi.FilterDesc(3, 3, 8, 16, 0, 8, 128)
    with pytest.raises(capi.BtnnError) as e:
        B.bconv_fused(ad, np.zeros(64, np.uint64), fd, np.zeros(144, np.uint64), g, tau=np.zeros(8), kind=np.zeros(8),
                      want_residual_out=True)
    assert e.value.code == capi.BTNN_INVALID_INPUT
    with pytest.raises(capi.BtnnError) as e:
        B.bconv_pm1(ad, np.zeros(64, np.uint64), capi.FilterDesc(3, 3, 8, 32, 0, 8, 128), np.zeros(144, np.uint64), g)
    assert e.value.code == capi.BTNN_INVALID_INPUT
    with pytest.raises(capi.BtnnError) as e:
        B.bconv_pm1(ad, np.zeros(64, np.uint64), fd, np.zeros(144, np.uint64), capi.ConvGeom(5, 5, 1, 1))
    assert e.value.code == capi.BTNN_INVALID_INPUT
    with pytest.raises(capi.BtnnError) as e:
        B.bconv_pm1(capi.ActDesc(2, 2, 1, 16, 0, 8, 128), np.zeros(16, np.uint64), fd, np.zeros(144, np.uint64),
                    capi.ConvGeom(3, 3, 1, 0))
    assert e.value.code == capi.BTNN_UNSUPPORTED_SHAPE


def test_bn_division_matches_ddiv_rn():
    """bnmath.cuh: the per-channel-reciprocal division equals __ddiv_rn and IEEE a/b
    bit for bit — bn-route operands (integer v - mean over s = sqrt(var + eps)), random
    doubles over a wide exponent range, and the range edges where __ddiv_rn leaves its
    fast path (zeros, tiny and huge quotients)."""
    rng = np.random.default_rng(5)
    n = 1 << 20
    s = np.sqrt(rng.uniform(0.25, 2.0, n) + 1e-5)
    v = rng.integers(-4608, 4609, n).astype(np.float64)
    mean = rng.standard_normal(n) * np.sqrt(4608) / 2
    a1, b1 = v - mean, s
    a2 = rng.standard_normal(n) * np.exp2(rng.integers(-1000, 1000, n).astype(np.float64))
    b2 = np.abs(rng.standard_normal(n)) * np.exp2(rng.integers(-60, 60, n).astype(np.float64)) + 1e-300
    edge = np.array([0.0, -0.0, 5e-324, -5e-324, 2.0**-1022, 2.0**-900, 2.0**-899, 1.0, -1.0, 1e300, -1e300, 2.0**1000])
    a3 = np.repeat(edge, 8)
    b3 = np.tile(np.array([1.0, 3.0, 1e-3, 0.7, 2.0**-60, 2.0**60, 1e-300, 1e300]), edge.size)
    a, b = np.concatenate([a1, a2, a3]), np.concatenate([b1, b2, b3])
    fast, ref = np.zeros_like(a), np.zeros_like(a)
    capi.check(capi.lib().btnn_cuda_selftest_div(ptr(a, C.c_double), ptr(b, C.c_double), a.size,
                                                 ptr(fast, C.c_double), ptr(ref, C.c_double)))
    with np.errstate(all="ignore"):
        want = a / b
    assert np.array_equal(ref.view(np.uint64), want.view(np.uint64))
    assert np.array_equal(fast.view(np.uint64), want.view(np.uint64))


def _oracle_first_conv(x, wpm, k, o, s, pd):
    n, h, w, c = x.shape
    P, Q = (h + 2 * pd - k) // s + 1, (w + 2 * pd - k) // s + 1
    want = np.zeros(P * Q * n * o)
    geo = capi.ConvGeom(k, k, s, pd)
    st = oracle().bo_first_conv_bwn(ptr(np.ascontiguousarray(x), C.c_float), n, h, w, c,
                                    ptr(np.ascontiguousarray(wpm), C.c_float), k, k, o, C.byref(geo),
                                    ptr(want, C.c_double))
    assert st == 0
    return want


@pytest.mark.parametrize("n,hw,k,o,pd,st", [(3, 224, 7, 64, 3, 4), (2, 61, 11, 48, 5, 4), (4, 36, 5, 16, 2, 4),
                                             (2, 224, 11, 128, 5, 4), (3, 40, 7, 100, 3, 4), (4, 32, 3, 128, 1, 1),
                                             (3, 30, 3, 72, 1, 1), (5, 17, 3, 20, 1, 1), (2, 33, 4, 40, 1, 1),
                                             (3, 28, 3, 128, 0, 1)])
def test_first_conv_exact_digits_adversarial(n, hw, k, o, pd, st, engine):
    """The tensor-core first layer (integer digit MMAs, kernels_first_tc.cu) is exact only
    on a per-tile grid; inputs here put values off that grid (tiny and subnormal values
    next to large ones, signed zeros, powers of two, an all-zero image, a huge outlier) so
    the sequential-f64 fix-up pass runs, and every output must still equal the
    reference's sequential sum bit for bit."""
    rng = np.random.default_rng(77 + hw)
    x = rng.standard_normal((n, hw, hw, 3)).astype(np.float32)
    flat = x.reshape(n, -1)
    m = flat.shape[1]
    idx = rng.integers(0, m, 40)
    flat[0, idx[:10]] = np.float32(1e-12)
    flat[0, idx[10:14]] = np.float32(-3e-39)  # subnormal
    flat[0, idx[14:18]] = -0.0
    flat[0, idx[18:22]] = np.exp2(rng.integers(-30, 10, 4)).astype(np.float32)
    flat[1, :] = 0.0
    flat[1, idx[22:26]] = np.float32(7.5e-8)
    if n > 2:
        flat[2, idx[26]] = np.float32(3e20)
        flat[2, idx[27:40]] = rng.standard_normal(13).astype(np.float32) * np.float32(1e-6)
    wpm = np.where(rng.standard_normal(o * k * k * 3) >= 0, 1.0, -1.0).astype(np.float32)
    got = B.first_conv_bwn(x, wpm, k, k, o, capi.ConvGeom(k, k, st, pd))
    if engine == "tc":  # the exact tensor-core kernel covers these shapes
        assert capi.last_tc_launch()[0] == f"first_conv/stride{st}", capi.last_tc_launch()
    want = _oracle_first_conv(x, wpm, k, o, st, pd)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
