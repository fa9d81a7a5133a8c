"""GPU parity at scale: every tensor-core kernel variant with at least three work units per
persistent CTA (so the mbarrier phase-1 waits of the tile pipeline and the TMEM
double-buffer parity run), checked against the reference compiled from its own headers
(oracle/_ref: bconv.hpp:160-194, bmm.hpp:219-274, inference.hpp:67-186) — plus the
benchmarked model configurations (BASELINE configs 2-5) at their full batch sizes.

btnn_cuda_last_tc_launch reports which kernel variant a call launched and how many
(tile, K-split) units it spread over how many CTAs, so each case proves the path it claims.
"""
import ctypes as C
import zlib

import numpy as np
import pytest

from oracle_lib import oracle, ptr, ref
from paper_2006_16578_b200 import btnn as B
from paper_2006_16578_b200 import capi
from paper_2006_16578_b200 import model as M
from paper_2006_16578_b200 import weights as Wt

pytestmark = pytest.mark.gpu


def _ref():
    r = ref()
    if r is None:
        pytest.skip("oracle/_ref (the compiled reference) is not built")
    return r


def _bn(rng, o, scale):
    return (rng.standard_normal(o), rng.standard_normal(o), rng.standard_normal(o) * scale, rng.uniform(0.25, 2.0, o))


def _ref_bconv_fused(ad, aw, fd, fw, g, P, Q, tau=None, kind=None, bn=None, rin=None, want_rout=False):
    """The reference's bconv_fused on the same operands (threaded)."""
    r = _ref()
    f = capi.ConvFused()
    keep = []
    if tau is not None:
        t, k = np.ascontiguousarray(tau, np.float64), np.ascontiguousarray(kind, np.uint8)
        keep += [t, k]
        f.tau, f.kind, f.n_thresholds = ptr(t, C.c_double), ptr(k, C.c_uint8), len(t)
    if bn is not None:
        arrs = [np.ascontiguousarray(x, np.float64) for x in bn]
        keep += arrs
        bnc = capi.Bn(*(ptr(a, C.c_double) for a in arrs), len(arrs[0]), 1e-5)
        keep.append(bnc)
        f.bn = C.pointer(bnc)
    if rin is not None:
        rr = np.ascontiguousarray(rin, np.float64)
        keep.append(rr)
        f.residual_in = ptr(rr, C.c_double)
    rout = np.zeros(P * Q * ad.batch * fd.out_channels) if want_rout else None
    if want_rout:
        f.residual_out = ptr(rout, C.c_double)
    od = capi.ActDesc(P, Q, ad.batch, fd.out_channels, 0, 8, 128)
    out = np.zeros(capi.lib().btnn_cuda_act_words(C.byref(od)), np.uint64)
    assert r.ref_bconv_fused(C.byref(ad), ptr(aw, C.c_uint64), C.byref(fd), ptr(fw, C.c_uint64), C.byref(g), C.byref(f),
                             ptr(out, C.c_uint64)) == 0, r.ref_last_error()
    return out, rout


def _assert_launch(expect, exclude=()):
    variant, units, grid = capi.last_tc_launch()
    for part in expect:
        assert part in variant.split("/"), (variant, expect)
    for part in exclude:
        assert part not in variant.split("/"), (variant, exclude)
    if not variant.startswith(("bmm_packed", "bmm_pipe")):  # (one tile per CTA by design: not persistent)
        assert units >= 3 * grid, f"{variant}: {units} units on {grid} CTAs — fewer than 3 per CTA"
    return variant


# (name, H=W, N, C, O, K, stride, route, expected variant parts, excluded parts)
VARIANT_CASES = [
    ("halo-thr-c64", 28, 128, 64, 64, 3, 1, "thr", ("halo", "thr"), ()),
    ("halo-thr-c128-s2", 28, 384, 128, 128, 3, 2, "thr", ("halo", "thr"), ()),
    ("halo-bn-c64", 28, 128, 64, 64, 3, 1, "bn", ("halo", "bn"), ()),
    ("halo-bn-c128-o256", 14, 256, 128, 256, 3, 1, "bn", ("halo", "bn"), ()),
    ("tmemA-thr-c256", 14, 320, 256, 128, 3, 1, "thr", ("tmemA", "thr"), ()),
    ("tmemA-thr-c96-k1", 16, 256, 96, 64, 1, 1, "thr", ("tmemA", "thr"), ()),
    ("tmemA-bn-c192", 14, 320, 192, 64, 3, 1, "bn", ("tmemA", "bn"), ("pg2",)),
    ("tmemA-bn-pg2-c256", 14, 320, 256, 128, 3, 1, "bn", ("tmemA", "bn", "pg2"), ()),
    ("tmemA-i32-c256", 14, 320, 256, 128, 3, 1, "i32", ("tmemA", "i32"), ()),
]


@pytest.mark.parametrize("case", VARIANT_CASES, ids=lambda c: c[0])
def test_tc_variant_many_tiles_per_cta(case):
    _, hw, n, c, o, k, s, route, expect, exclude = case
    capi.set_engine(capi.ENGINE_TC)
    try:
        rng = np.random.default_rng(zlib.crc32(case[0].encode()))
        pd = k // 2
        x = rng.standard_normal((n, hw, hw, c), dtype=np.float32)
        wt = rng.standard_normal(k * k * o * c, dtype=np.float32)
        aw, fw = Wt.pack_nhwc(x), Wt.pack_filter(wt, k, k, o, c)
        ad, fd, g = capi.ActDesc(hw, hw, n, c, 0, 8, 128), capi.FilterDesc(k, k, o, c, 0, 8, 128), capi.ConvGeom(k, k, s, pd)
        P = Q = (hw + 2 * pd - k) // s + 1
        if route == "i32":
            got = B.bconv_pm1(ad, aw, fd, fw, g)
            _assert_launch(expect, exclude)
            want = np.zeros(P * Q * n * o, np.int32)
            r = _ref()
            assert r.ref_bconv_pm1(C.byref(ad), ptr(aw, C.c_uint64), C.byref(fd), ptr(fw, C.c_uint64), C.byref(g), 0,
                                   ptr(want, C.c_int32)) == 0
            assert np.array_equal(got.reshape(-1), want)
            return
        if route == "thr":
            gamma, beta, mean, var = _bn(rng, o, np.sqrt(c * k * k) / 2)
            tau, kind = Wt.fold_bn_sign(gamma, beta, mean, var, 1e-5)
            got, _ = B.bconv_fused(ad, aw, fd, fw, g, tau=tau, kind=kind)
            _assert_launch(expect, exclude)
            want, _ = _ref_bconv_fused(ad, aw, fd, fw, g, P, Q, tau=tau, kind=kind)
            assert np.array_equal(got, want)
            return
        bn = _bn(rng, o, np.sqrt(c * k * k) / 2)
        rin = rng.standard_normal(P * Q * n * o) * 3.0
        got, rout = B.bconv_fused(ad, aw, fd, fw, g, bn=bn, residual_in=rin, want_residual_out=True)
        _assert_launch(expect, exclude)
        want, wrout = _ref_bconv_fused(ad, aw, fd, fw, g, P, Q, bn=bn, rin=rin, want_rout=True)
        assert np.array_equal(rout.view(np.uint64), wrout.view(np.uint64))
        assert np.array_equal(got, want)
    finally:
        capi.set_engine(capi.ENGINE_AUTO)


@pytest.mark.parametrize("kk,kind_,force", [(1024, "bmm_packed", 0), (2048, "bmm_pipe", 0), (1024, "bmm_pipe", 2)])
def test_bmm_many_tiles_per_cta(kk, kind_, force):
    """BMM 8192 x K x 1024 packed -> int32 and -> thresholded bits: K = 1024 runs the whole-K
    packed BMM (1024 CTAs), K = 2048 the K-pipelined one (512 128 x 128 tiles, two CTAs per SM),
    and K = 1024 forced onto the pipelined kernel."""
    capi.set_engine(capi.ENGINE_TC)
    capi.set_bmm_kernel(force)
    try:
        rng = np.random.default_rng(9)
        m, nn = 8192, 1024
        A = rng.integers(0, 2**64, m * kk // 64, dtype=np.uint64)
        Bw = rng.integers(0, 2**64, nn * kk // 64, dtype=np.uint64)
        da, db = capi.MatrixDesc(m, kk, capi.ROW_PACKED, 8, 128), capi.MatrixDesc(kk, nn, capi.COL_PACKED, 8, 128)
        got = B.bmm_pm1(da, A, db, Bw).reshape(-1)
        _assert_launch((kind_, "i32"))
        want = np.zeros(m * nn, np.int32)
        assert oracle().bo_bmm_pm1(C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(Bw, C.c_uint64), capi.BMM_BLOCKED,
                                   ptr(want, C.c_int32)) == 0
        assert np.array_equal(got, want)
        tau = rng.standard_normal(nn) * 20
        kind = rng.integers(0, 4, nn).astype(np.uint8)
        bits = B.bmm_pm1_bin(da, A, db, Bw, tau=tau, kind=kind)
        _assert_launch((kind_, "bin"))
        wbits = np.zeros_like(bits)
        assert oracle().bo_bmm_pm1_bin(C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(Bw, C.c_uint64),
                                       capi.BMM_BLOCKED, ptr(np.ascontiguousarray(tau), C.c_double),
                                       ptr(kind, C.c_uint8), nn, ptr(wbits, C.c_uint64)) == 0
        assert np.array_equal(bits, wbits)
    finally:
        capi.set_engine(capi.ENGINE_AUTO)
        capi.set_bmm_kernel(capi.BMM_AUTO)


def _ref_run(m, ws, x):
    r = _ref()
    spec, store = m.c_spec(), ws.c_store()
    lg = np.zeros(x.shape[0] * m.classes)
    lb = np.zeros(x.shape[0], np.int32)
    st = r.ref_run_store(C.byref(spec), C.byref(store), ptr(np.ascontiguousarray(x), C.c_float), x.shape[0],
                         ptr(lg, C.c_double), ptr(lb, C.c_int32))
    assert st == 0, r.ref_last_error()
    return lg.reshape(x.shape[0], m.classes), lb



def test_blocked_producer_and_split_k_many_tiles():
    """A 2x2-blocked tap producer (halved shortcut) with >= 3 tiles per CTA and a split-K
    FC layer, end to end against the reference's run_inference."""
    m = M.make_model("blk", "32C3-64C3-64C3-128C3/2-128C3-512FC-10FC", 32, 32, 3, 10, [(1, 4)])
    ws = Wt.build_weights(m, Wt.random_weights(m, 91))
    x = np.random.default_rng(92).standard_normal((256, 32, 32, 3), dtype=np.float32)
    plan = B.Plan(m, ws, 256)
    capi.set_engine(capi.ENGINE_AUTO)
    lg, lb = plan.run(x)
    assert plan.tap_dims(1)[2] == 1, "layer 1 should store its tap pre-averaged (blocked producer)"
    want, wl = _ref_run(m, ws, x)
    assert np.array_equal(lg.view(np.uint64), want.view(np.uint64)), plan.engines()
    assert np.array_equal(lb, wl)
    assert "tc_i8_splitk" in plan.engines(), plan.engines()


@pytest.mark.parametrize("name,batch,first", [
    ("resnet18", 512, 512), ("resnet18", 1024, 64), ("alexnet", 256, 256), ("cifar-vgg", 1024, 1024),
    ("cifar-vgg", 256, 256), ("mnist-mlp", 1024, 1024)])
def test_benchmarked_configs_vs_reference(name, batch, first):
    """The bench's own configurations at full batch: the whole batch runs on the GPU (every
    kernel at its steady-state tile count) and the first `first` images are compared with
    the reference's run_inference bit for bit (logits as f64 bit patterns, labels)."""
    m = M.stock_model(name)
    ws = Wt.build_weights(m, Wt.random_weights(m, 1))
    rng = np.random.default_rng(3)
    x = rng.standard_normal((batch, m.in_h, m.in_w, m.in_c), dtype=np.float32)
    plan = B.Plan(m, ws, batch)
    lg, lb = plan.run(x)
    want, wl = _ref_run(m, ws, x[:first])
    assert np.array_equal(lg[:first].view(np.uint64), want.view(np.uint64)), plan.engines()
    assert np.array_equal(lb[:first], wl)
    if first < batch:  # the tail of the batch: the same images in another batch position agree
        lg2, lb2 = plan.run(x[batch - first:])
        assert np.array_equal(lg2.view(np.uint64), lg[batch - first:].view(np.uint64))
        want2, wl2 = _ref_run(m, ws, x[batch - 8:])
        assert np.array_equal(lg[batch - 8:].view(np.uint64), want2.view(np.uint64))
