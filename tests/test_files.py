"""File ingestion on the GPU path: BTNN bit-weight files
(save_weights / load_weights, weights.hpp:298-445) and BTIN batches (write_batch /
read_batch, io.hpp:68-101) written by the reference itself (oracle/_ref) and read by
libbtnn_cuda's btnn_cuda_load_weights / btnn_cuda_read_batch.

CPU tests: the parsed store equals the reference's own store array for array (plain and tiled
files), and malformed files raise the reference's error classes. GPU test: load weights ->
read batch -> plan run (the `btnn infer` flow, btnn_cli.cpp:69-110) gives logits bit-identical
to the reference's load_weights + read_batch + run_inference on the same files."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle_lib import RefModel, RefWeights, ptr, ref
from paper_2006_16578_b200 import btnn as B
from paper_2006_16578_b200 import capi

MODELS = [
    # (name, tokens, hw, classes, shortcuts)
    ("res", "16C7/4-16C3-16C3-32C3/2-32C3-(2x64FC)", 32, 10, [(0, 2), (2, 4)]),
    ("vggish", "(2x32C3)-MP2-(2x64C3)-MP2-(64FC)", 16, 7, []),
    ("mlp", "256FC-128FC", 12, 5, []),
]


def _need_ref():
    if ref() is None:
        pytest.skip("compiled reference (oracle/_ref) not available")


def _arr(p, n, t):
    if not n:
        return np.zeros(0, dtype=t)
    return np.ctypeslib.as_array(p, shape=(n,)).astype(t, copy=True)


def _save(tmp_path, mdl, seed, tiled):
    model = RefModel.make(mdl[0], mdl[1], mdl[2], mdl[2], 3 if mdl[0] != "mlp" else 1, mdl[3], mdl[4])
    w = RefWeights(model, seed, tiled=tiled)
    path = str(tmp_path / f"{mdl[0]}_{int(tiled)}.btnn")
    assert ref().ref_save_weights(model.h, w.ws, path.encode()) == 0, ref().ref_last_error()
    return model, w, path


@pytest.mark.parametrize("tiled", [False, True])
@pytest.mark.parametrize("mdl", MODELS, ids=[m[0] for m in MODELS])
def test_weight_file_parse_equals_reference_store(tmp_path, mdl, tiled):
    _need_ref()
    model, w, path = _save(tmp_path, mdl, 5, tiled)
    lw = B.LoadedWeights(path, model.view)
    got = lw.c_store()
    want = w.store
    assert got.n_layers == want.n_layers and got.tiled == int(tiled) and (got.bh, got.bw) == (8, 128)
    for i in range(want.n_layers):
        g, r = got.layers[i], want.layers[i]
        assert g.kind == r.kind
        for f, nf, t in (("filter_words", "filter_n_words", np.uint64), ("fc_words", "fc_n_words", np.uint64),
                         ("conv_pm1", "conv_pm1_n", np.float32)):
            assert getattr(g, nf) == getattr(r, nf), (i, f)
            assert np.array_equal(_arr(getattr(g, f), getattr(g, nf), t), _arr(getattr(r, f), getattr(r, nf), t)), (i, f)
        assert g.n_thresholds == r.n_thresholds
        assert np.array_equal(_arr(g.tau, g.n_thresholds, np.float64).view(np.uint64),
                              _arr(r.tau, r.n_thresholds, np.float64).view(np.uint64))
        assert np.array_equal(_arr(g.tkind, g.n_thresholds, np.uint8), _arr(r.tkind, r.n_thresholds, np.uint8))
        assert g.has_bn == r.has_bn
        if r.has_bn:
            assert g.bn.channels == r.bn.channels and g.bn.eps == r.bn.eps
            for f in ("gamma", "beta", "mean", "var"):
                assert np.array_equal(_arr(getattr(g.bn, f), g.bn.channels, np.float64).view(np.uint64),
                                      _arr(getattr(r.bn, f), r.bn.channels, np.float64).view(np.uint64)), (i, f)


def _corrupt(src, dst, fn):
    b = bytearray(open(src, "rb").read())
    b = fn(b)
    open(dst, "wb").write(bytes(b))
    return dst


def test_weight_file_errors_match_reference_classes(tmp_path):
    """Malformed files raise the reference's classes (weights.hpp:354-445): io_error for
    magic/version/layout tag/truncation, validation_error for layer count/kind/dims."""
    _need_ref()
    model, w, path = _save(tmp_path, MODELS[0], 6, False)
    other = RefModel.make("other", "16C7/4-16C3-(2x64FC)", 32, 32, 3, 10)

    def code(p, m=model.view):
        with pytest.raises(capi.BtnnError) as e:
            B.LoadedWeights(p, m)
        return e.value.code

    t = tmp_path
    assert code(str(t / "missing.btnn")) == capi.BTNN_IO_ERROR
    assert code(_corrupt(path, str(t / "m.btnn"), lambda b: b"XTNN" + b[4:])) == capi.BTNN_IO_ERROR
    assert code(_corrupt(path, str(t / "v.btnn"), lambda b: b[:4] + (2).to_bytes(4, "little") + b[8:])) == \
        capi.BTNN_IO_ERROR
    assert code(_corrupt(path, str(t / "t.btnn"), lambda b: b[:len(b) // 2])) == capi.BTNN_IO_ERROR
    assert code(path, other.view) == capi.BTNN_VALIDATION_ERROR  # layer count
    # first record: kind byte at offset 12, dims at 13..28, layout tag at 29
    assert code(_corrupt(path, str(t / "k.btnn"), lambda b: b[:12] + bytes([1]) + b[13:])) == \
        capi.BTNN_VALIDATION_ERROR
    assert code(_corrupt(path, str(t / "d.btnn"), lambda b: b[:13] + (5).to_bytes(4, "little") + b[17:])) == \
        capi.BTNN_VALIDATION_ERROR
    assert code(_corrupt(path, str(t / "g.btnn"), lambda b: b[:29] + bytes([7]) + b[30:])) == capi.BTNN_IO_ERROR


def test_batch_file_roundtrip_and_errors(tmp_path):
    _need_ref()
    x = np.random.default_rng(3).standard_normal((5, 7, 6, 3), dtype=np.float32)
    x[0, 0, 0, 0] = -0.0
    p = str(tmp_path / "x.btin")
    assert ref().ref_write_batch(ptr(x, C.c_float), 5, 7, 6, 3, p.encode()) == 0
    got = B.read_batch(p)
    assert got.shape == x.shape and np.array_equal(got.view(np.uint32), x.view(np.uint32))
    bad = _corrupt(p, str(tmp_path / "b.btin"), lambda b: b[:-4])  # not a whole number of samples
    with pytest.raises(capi.BtnnError) as e:
        B.read_batch(bad)
    assert e.value.code == capi.BTNN_IO_ERROR
    zero = _corrupt(p, str(tmp_path / "z.btin"), lambda b: b[:4] + (0).to_bytes(4, "little") + b[8:])
    with pytest.raises(capi.BtnnError) as e:
        B.read_batch(zero)
    assert e.value.code == capi.BTNN_IO_ERROR
    mg = _corrupt(p, str(tmp_path / "g.btin"), lambda b: b"BTNN" + b[4:])
    with pytest.raises(capi.BtnnError) as e:
        B.read_batch(mg)
    assert e.value.code == capi.BTNN_IO_ERROR


@pytest.mark.gpu
@pytest.mark.parametrize("tiled", [False, True])
@pytest.mark.parametrize("mdl", MODELS, ids=[m[0] for m in MODELS])
def test_infer_from_files_matches_reference(tmp_path, mdl, tiled):
    """`btnn infer` on the GPU path: weights and batch from reference-written files."""
    _need_ref()
    model, w, path = _save(tmp_path, mdl, 9, tiled)
    v = model.view
    n = 6
    x = np.random.default_rng(10).standard_normal((n, v.in_h, v.in_w, v.in_c), dtype=np.float32)
    bpath = str(tmp_path / "in.btin")
    assert ref().ref_write_batch(ptr(x, C.c_float), n, v.in_h, v.in_w, v.in_c, bpath.encode()) == 0
    want = np.zeros(n * v.classes)
    wl = np.zeros(n, dtype=np.int32)
    got_n = C.c_size_t()
    assert ref().ref_infer_files(model.h, path.encode(), int(tiled), bpath.encode(), n, ptr(want, C.c_double),
                                 ptr(wl, C.c_int32), C.byref(got_n)) == 0, ref().ref_last_error()
    assert got_n.value == n
    lw = B.LoadedWeights(path, v)
    xb = B.read_batch(bpath)
    lg, lb = B.Plan(v, lw, n).run(xb)
    assert np.array_equal(lg.reshape(-1).view(np.uint64), want.view(np.uint64))
    assert np.array_equal(lb, wl)
