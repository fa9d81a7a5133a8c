"""Host-side logic (no GPU): the harness' model grammar and weight packing agree with the
reference; libbtnn_cuda.so loads and exports every symbol include/btnn_cuda.h declares;
C-ABI calls that fail validation return the reference's error class before touching a
device."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle_lib import RefModel, RefWeights, normal_floats, ptr, ref
from paper_2006_16578_b200 import capi
from paper_2006_16578_b200 import model as M
from paper_2006_16578_b200 import weights as Wt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(ref() is None, reason="oracle/_ref not built")


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "btnn_cuda.h")).read()
    declared = set(re.findall(r"\b(btnn_cuda_\w+)\s*\(", hdr))
    assert declared, "no symbols parsed"
    lib = capi.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(capi.EXPORTS)
    assert lib.btnn_cuda_abi_version() == 1


def test_grammar_known_answer():  # test_nn.cpp:92-102: 16C11/4 at 224 -> 56
    m = M.make_model("g", "16C11/4-8FC", 224, 224, 3, 10)
    assert m.layers[0].kind == capi.FIRST_CONV_BWN
    assert (m.layers[0].out_h, m.layers[0].out_w, m.layers[0].pad) == (56, 56, 5)
    assert m.layers[-1].kind == capi.LAST_FC and m.layers[-1].units == 10


def test_grammar_errors():  # test_nn.cpp:81-150
    with pytest.raises(M.ModelError) as e:
        M.make_model("bad", "8FC-4C3", 8, 8, 1, 3)
    assert e.value.code == capi.BTNN_VALIDATION_ERROR
    with pytest.raises(M.ModelError) as e:
        M.make_model("bad", "(4C3", 8, 8, 1, 3)
    assert e.value.code == capi.BTNN_INVALID_INPUT
    with pytest.raises(M.ModelError) as e:
        M.make_model("bad", "4C3-P2", 7, 7, 1, 3)
    assert e.value.code == capi.BTNN_VALIDATION_ERROR
    with pytest.raises(M.ModelError):
        M.make_model("bad", "4C3-4C3", 8, 8, 1, 3, [(1, 0)])


@needs_ref
@pytest.mark.parametrize("name", sorted(M.STOCK))
def test_stock_models_resolve_like_reference(name):
    import json
    ours = M.stock_model(name)
    theirs = RefModel.parse(json.dumps(M.STOCK[name]))
    assert len(ours.layers) == theirs.view.n_layers
    for a, b in zip(ours.layers, theirs.layers()):
        for f, _ in capi.LayerSpec._fields_:
            assert int(getattr(a, f)) == int(getattr(b, f)), (name, f)


@needs_ref
@pytest.mark.parametrize("tiled", [False, True])
def test_weight_packing_matches_reference(tiled):
    """pack_filter / pack_fc / unpack_first_conv / fold of the numpy harness vs build_weights."""
    rm = RefModel.make("w", "6C3-P2-8C3/2-12FC", 12, 12, 3, 5, [])
    rw = RefWeights(rm, 21, tiled=tiled)
    ours_m = M.make_model("w", "6C3-P2-8C3/2-12FC", 12, 12, 3, 5)
    # rebuild the float weights from the reference's own draw
    fw = []
    for i in range(rm.view.n_layers):
        w, n, g, b, mu, v, ch = (C.POINTER(C.c_float)(), C.c_size_t(), C.POINTER(C.c_double)(), C.POINTER(C.c_double)(),
                                 C.POINTER(C.c_double)(), C.POINTER(C.c_double)(), C.c_size_t())
        ref().ref_float_weights_get(rw.fw, i, C.byref(w), C.byref(n), C.byref(g), C.byref(b), C.byref(mu), C.byref(v),
                                    C.byref(ch))
        if n.value == 0:
            fw.append(None)
            continue
        arr = lambda p, k: np.ctypeslib.as_array(p, (k,)).copy()  # noqa: E731
        fw.append(dict(weights=arr(w, n.value), gamma=arr(g, ch.value), beta=arr(b, ch.value), mean=arr(mu, ch.value),
                       var=arr(v, ch.value)))
    ws = Wt.build_weights(ours_m, Wt.FloatWeights(fw), tiled=tiled)
    st = rw.store
    for i, rec in enumerate(ws.layers):
        L = st.layers[i]
        if "filter" in rec:
            assert np.array_equal(rec["filter"], np.ctypeslib.as_array(L.filter_words, (L.filter_n_words,)))
        if "conv_pm1" in rec:
            assert np.array_equal(rec["conv_pm1"], np.ctypeslib.as_array(L.conv_pm1, (L.conv_pm1_n,)))
        if "fc" in rec:
            assert np.array_equal(rec["fc"], np.ctypeslib.as_array(L.fc_words, (L.fc_n_words,)))
        if "tau" in rec:
            assert np.array_equal(rec["tau"].view(np.uint64),
                                  np.ctypeslib.as_array(L.tau, (L.n_thresholds,)).view(np.uint64))
            assert np.array_equal(rec["kind"], np.ctypeslib.as_array(L.tkind, (L.n_thresholds,)))


@needs_ref
def test_pack_matrix_nhwc_match_reference():
    x = normal_floats(3, 3 * 5 * 7 * 130).reshape(3, 5, 7, 130)
    for tiled in (False, True):
        want = np.zeros(Wt.act_words(5, 7, 3, 130, tiled), dtype=np.uint64)
        ref().ref_pack_nhwc(ptr(x, C.c_float), 3, 5, 7, 130, int(tiled), 8, 128, ptr(want, C.c_uint64))
        assert np.array_equal(Wt.pack_nhwc(x, tiled), want)
    v = normal_floats(4, 17 * 300)
    for lay in range(4):
        d = capi.MatrixDesc(17, 300, lay, 8, 128)
        want = np.zeros(ref().ref_matrix_words(C.byref(d)), dtype=np.uint64)
        ref().ref_pack_matrix(ptr(v, C.c_float), v.size, C.byref(d), ptr(want, C.c_uint64))
        assert np.array_equal(Wt.pack_matrix(v, 17, 300, lay), want), lay


def test_validation_errors_without_device():
    """Operand checks run host-side before any device work (bmm.hpp:57-76, bconv.hpp:163-171)."""
    from paper_2006_16578_b200 import btnn as B
    a = capi.MatrixDesc(4, 128, capi.ROW_PACKED, 8, 128)
    bshort = capi.MatrixDesc(64, 4, capi.COL_PACKED, 8, 128)
    with pytest.raises(capi.BtnnError) as e:
        B.bmm_pm1(a, np.zeros(8, np.uint64), bshort, np.zeros(8, np.uint64))
    assert e.value.code == capi.BTNN_INVALID_INPUT
    with pytest.raises(capi.BtnnError) as e:
        B.bmm_raw(capi.MatrixDesc(4, 200, capi.ROW_PACKED, 8, 128), np.zeros(16, np.uint64),
                  capi.MatrixDesc(200, 4, capi.COL_PACKED, 8, 128), np.zeros(16, np.uint64))
    assert e.value.code == capi.BTNN_UNSUPPORTED_SHAPE
    fsb_b = capi.MatrixDesc(128, 4, capi.FSB_COL, 4, 64)
    fsb_a = capi.MatrixDesc(4, 128, capi.FSB_ROW, 8, 128)
    with pytest.raises(capi.BtnnError) as e:
        B.bmm_pm1(fsb_a, np.zeros(16, np.uint64), fsb_b, np.zeros(16, np.uint64), variant=capi.BMM_FSB)
    assert e.value.code == capi.BTNN_UNSUPPORTED_SHAPE
    with pytest.raises(capi.BtnnError) as e:
        B.bmm_pm1(a, np.zeros(8, np.uint64), capi.MatrixDesc(128, 4, capi.COL_PACKED, 8, 128), np.zeros(8, np.uint64),
                  blocking=(8, 8, 100))
    assert e.value.code == capi.BTNN_INVALID_INPUT
    ad, fd, g = capi.ActDesc(4, 4, 1, 16, 0, 8, 128), capi.FilterDesc(3, 3, 8, 16, 0, 8, 128), capi.ConvGeom(3, 3, 1, 1)
    with pytest.raises(capi.BtnnError) as e:  # neither thresholds nor bn (test_bconv.cpp:343)
        B.bconv_fused(ad, np.zeros(64, np.uint64), fd, np.zeros(144, np.uint64), g)
    assert e.value.code == capi.BTNN_INVALID_INPUT
    with pytest.raises(capi.BtnnError) as e:  # mixed layouts
        B.bconv_pm1(ad, np.zeros(64, np.uint64), capi.FilterDesc(3, 3, 8, 16, 1, 8, 128), np.zeros(144, np.uint64), g)
    assert e.value.code == capi.BTNN_INVALID_INPUT
    with pytest.raises(capi.BtnnError) as e:  # or_pool partial coverage
        B.or_pool(capi.ActDesc(7, 7, 1, 8, 0, 8, 128), np.zeros(7 * 7 * 16, np.uint64), 2, 2)
    assert e.value.code == capi.BTNN_UNSUPPORTED_SHAPE
