"""GPU parity of the model driver (run_inference, inference.hpp:67-186): logits bit-exact
(f64) and labels equal to the reference on the reference's own models and weights, in
both weight layouts, and invariant to batch sharding across devices."""
import numpy as np
import pytest

from fixtures import fixture_models
from oracle_lib import oracle_run_inference
from paper_2006_16578_b200 import btnn as B
from paper_2006_16578_b200 import capi
from paper_2006_16578_b200 import model as M
from paper_2006_16578_b200 import weights as Wt

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("engine")]


@pytest.mark.parametrize("prefix,fm", fixture_models(), ids=lambda v: v if isinstance(v, str) else "")
def test_run_inference_golden(prefix, fm):
    plan = B.Plan(fm.spec, fm.store, fm.x.shape[0])
    lg, lb = plan.run(fm.x)
    assert np.array_equal(lg.view(np.uint64), fm.logits.view(np.uint64)), plan.engines()
    assert np.array_equal(lb, fm.labels)
    # the same plan again (graph replay) and a smaller batch reuse
    lg2, _ = plan.run(fm.x)
    assert np.array_equal(lg2.view(np.uint64), fm.logits.view(np.uint64))
    if fm.x.shape[0] > 1:
        lg3, lb3 = plan.run(fm.x[:1])
        assert np.array_equal(lg3[0].view(np.uint64), fm.logits[0].view(np.uint64))


@pytest.mark.parametrize("prefix,fm", fixture_models()[:6], ids=lambda v: v if isinstance(v, str) else "")
def test_sharded_plan_matches(prefix, fm):
    """Two shards on device 0 exercise the batch split; results equal the single run."""
    plan = B.Plan(fm.spec, fm.store, fm.x.shape[0], devices=(0, 0))
    lg, lb = plan.run(fm.x)
    assert np.array_equal(lg.view(np.uint64), fm.logits.view(np.uint64))
    assert np.array_equal(lb, fm.labels)


def test_nonfinite_input_rejected():  # test_nn.cpp:355-364
    m = M.make_model("bad", "4C3-8FC", 8, 8, 2, 3)
    ws = Wt.build_weights(m, Wt.random_weights(m, 67))
    plan = B.Plan(m, ws, 2)
    x = np.zeros((1, 8, 8, 2), np.float32)
    x.reshape(-1)[7] = np.nan
    with pytest.raises(capi.BtnnError) as e:
        plan.run(x)
    assert e.value.code == capi.BTNN_INVALID_INPUT
    mm = M.make_model("mlp", "8FC", 4, 4, 1, 3)
    p2 = B.Plan(mm, Wt.build_weights(mm, Wt.random_weights(mm, 3)), 2)
    xb = np.ones((1, 4, 4, 1), np.float32)
    xb[0, 1, 1, 0] = np.inf
    with pytest.raises(capi.BtnnError):
        p2.run(xb)


@pytest.mark.parametrize("tokens,hw,shortcuts", [
    # type-A shortcuts whose zero-filled channels end inside an output tile
    ("8C3-24C3-40C3/2-40C3-72C3/2-72C3-8FC", 16, [(1, 3), (3, 5)]),
    ("16C3-200C3-200C3/2-300C3-300C3", 12, [(1, 3), (3, 4)]),
    ("32C3-64C3-128C3/2-256C3-256C3/2-256C3", 16, [(1, 3), (3, 5)]),
])
def test_residual_variants_vs_oracle(tokens, hw, shortcuts):
    m = M.make_model("resvar", tokens, hw, hw, 3, 7, shortcuts)
    ws = Wt.build_weights(m, Wt.random_weights(m, 17))
    x = np.random.default_rng(18).standard_normal((5, hw, hw, 3), dtype=np.float32)
    lg, lb = B.Plan(m, ws, 5).run(x)
    want, wl = oracle_run_inference(m.c_spec(), ws.c_store(), x)
    assert np.array_equal(lg.view(np.uint64), want.view(np.uint64))
    assert np.array_equal(lb, wl)


@pytest.mark.parametrize("name,hw,batch", [("resnet18", 224, 2), ("resnet18", 224, 8), ("alexnet", 224, 2), ("cifar-vgg", 32, 8),
                                            ("mnist-mlp", 28, 64), ("cifar-resnet14", 32, 8), ("vgg16", 64, 2)])
def test_stock_models_vs_oracle(name, hw, batch):
    """The stock models (numpy-drawn weights) vs the C oracle; ResNet-18/AlexNet at full
    ImageNet shape are checked on the small batch the bit-serial oracle affords."""
    m = M.stock_model(name, hw, hw)
    ws = Wt.build_weights(m, Wt.random_weights(m, 1))
    rng = np.random.default_rng(2)
    x = rng.standard_normal((batch, m.in_h, m.in_w, m.in_c), dtype=np.float32)
    plan = B.Plan(m, ws, batch)
    lg, lb = plan.run(x)
    if name in ("resnet18", "alexnet", "vgg16"):
        ref = pytest.importorskip("oracle_lib").ref()
        if ref is None:
            pytest.skip("compiled reference not available")
    want, wl = oracle_run_inference(m.c_spec(), ws.c_store(), x) if name not in ("resnet18", "alexnet", "vgg16") else \
        _ref_run(m, ws, x)
    assert np.array_equal(lg.view(np.uint64), want.view(np.uint64)), plan.engines()
    assert np.array_equal(lb, wl)


def _ref_run(m, ws, x):
    """Large models: the reference's own run_inference (word-parallel, threaded) on the
    same store, via oracle/_ref."""
    import ctypes as C
    from oracle_lib import ptr, ref
    spec, store = m.c_spec(), ws.c_store()
    lg = np.zeros(x.shape[0] * m.classes)
    lb = np.zeros(x.shape[0], np.int32)
    st = ref().ref_run_store(C.byref(spec), C.byref(store), ptr(np.ascontiguousarray(x), C.c_float), x.shape[0],
                             ptr(lg, C.c_double), ptr(lb, C.c_int32))
    assert st == 0, ref().ref_last_error()
    return lg.reshape(x.shape[0], m.classes), lb


def test_halved_tap_equals_adapt_shortcut():
    """A layer whose tap only feeds a halving shortcut stores the 2x2 average directly
    (tensor-core engine, blocked row order). It must equal adapt_shortcut's
    ((a+b)+c)+d)*0.25 (inference.hpp:43-63) of the full tap the CUDA-core engine stores,
    including a batch that is not a multiple of the 32-image row group."""
    m = M.make_model("halve", "16C3-32C3-32C3-64C3/2-64C3", 12, 12, 3, 5, [(0, 2), (2, 4)])
    ws = Wt.build_weights(m, Wt.random_weights(m, 31))
    x = np.random.default_rng(32).standard_normal((37, 12, 12, 3), dtype=np.float32)
    capi.set_engine(capi.ENGINE_POPC)
    p_full = B.Plan(m, ws, 37)
    lg_full, _ = p_full.run(x)
    full = p_full.read_tap(2, 37).reshape(12, 12, 37, 32)
    capi.set_engine(capi.ENGINE_TC)
    p_half = B.Plan(m, ws, 37)
    lg_half, _ = p_half.run(x)
    assert p_half.tap_dims(2) == (6, 6, 1, 32)
    half = p_half.read_tap(2, 37).reshape(6, 6, 37, 32)
    a, b, c, d = full[0::2, 0::2], full[0::2, 1::2], full[1::2, 0::2], full[1::2, 1::2]
    want = (((a + b) + c) + d) * 0.25
    assert np.array_equal(half.view(np.uint64), want.view(np.uint64))
    assert np.array_equal(lg_half.view(np.uint64), lg_full.view(np.uint64))


def test_signed_zero_taps_fire():
    """bn-route outputs equal to -0.0 must fire (y >= 0.0 holds for -0.0, bconv.hpp:191):
    gamma < 0 and beta = -0.0 turn every v == mean into y = -0.0 (x = +0, q = +0, q*gamma = -0,
    -0 + -0 = -0), and a zero image makes that happen across whole first-layer tiles; the
    residual add then sees -0.0 + -0.0. The epilogues read the sign off the f64 bit pattern on
    channels with finite parameters (bnmath.cuh nonneg_bit), so this pins the -0.0 case."""
    m = M.make_model("negzero", "16C7/4-16C3-16C3-16C3-8FC", 32, 32, 3, 8, [(0, 2), (2, 3)])
    fw = Wt.random_weights(m, 41)
    for li in (0, 2, 3):
        lw = fw.layers[li]
        ch = lw["gamma"].shape[0]
        lw["gamma"] = -np.abs(lw["gamma"]) - 0.1
        lw["gamma"][::4] *= -1.0  # some channels keep gamma > 0: +0 + -0 = +0
        lw["beta"] = np.full(ch, -0.0)
        lw["mean"] = np.zeros(ch)
    ws = Wt.build_weights(m, fw)
    x = np.random.default_rng(42).standard_normal((6, 32, 32, 3), dtype=np.float32)
    x[0] = 0.0
    x[3, :16] = 0.0
    lg, lb = B.Plan(m, ws, 6).run(x)
    want, wl = oracle_run_inference(m.c_spec(), ws.c_store(), x)
    assert np.array_equal(lg.view(np.uint64), want.view(np.uint64))
    assert np.array_equal(lb, wl)


@pytest.mark.parametrize("batch", [8, 16, 13])
def test_uncleared_outputs_pad_words(batch):
    """With N % 8 == 0 the plan does not clear packed outputs before tensor-core layers; the
    epilogues write the channel-pad words themselves (O = 48 / 40 / 72 leave pad words in the
    128-bit rows, including the tensor-core first conv). Stale bits from the previous use of
    the ping-pong buffers must not leak: a second run on different inputs must match too."""
    m = M.make_model("padw", "48C7/4-40C3-72C3-40C3-24FC", 64, 64, 3, 9, [(1, 3)])
    ws = Wt.build_weights(m, Wt.random_weights(m, 51))
    plan = B.Plan(m, ws, batch)
    for seed in (52, 53):
        x = np.random.default_rng(seed).standard_normal((batch, 64, 64, 3), dtype=np.float32)
        lg, lb = plan.run(x)
        want, wl = oracle_run_inference(m.c_spec(), ws.c_store(), x)
        assert np.array_equal(lg.view(np.uint64), want.view(np.uint64)), plan.engines()
        assert np.array_equal(lb, wl)


def test_plan_tuner_measured_choices(engine):
    """The plan tuner (north star (2)): every tensor-core conv layer of a residual model lists
    its feasible geometries with measured times and runs the fastest; tuned and untuned plans
    both equal the oracle bit for bit."""
    m = M.make_model("tune", "64C3-64C3-64C3-128C3/2-128C3-128C3-10FC", 28, 28, 3, 10, [(0, 2), (2, 5)])
    ws = Wt.build_weights(m, Wt.random_weights(m, 77))
    x = np.random.default_rng(78).standard_normal((40, 28, 28, 3), dtype=np.float32)
    want, wl = oracle_run_inference(m.c_spec(), ws.c_store(), x)
    try:
        capi.lib().btnn_cuda_set_autotune(0)
        plain = B.Plan(m, ws, 40)
    finally:
        capi.lib().btnn_cuda_set_autotune(1)
    tuned = B.Plan(m, ws, 40)
    for plan in (plain, tuned):
        lg, lb = plan.run(x)
        assert np.array_equal(lg.view(np.uint64), want.view(np.uint64)) and np.array_equal(lb, wl)
    tc_layers = [i for i, e in enumerate(tuned.engines()) if e.startswith("tc_i8") and i > 0]
    if engine == "popc":
        assert not tc_layers
        return
    assert tc_layers
    multi = 0
    for i in tc_layers:
        names, pick, ms = tuned.layer_choice(i)
        if m.layers[i].kind == capi.BIT_CONV:
            assert names and 0 <= pick < len(names) and all(t > 0 for t in ms), (i, names, ms)
            assert ms[pick] == min(ms)
            multi += len(names) > 1
        assert plain.layer_choice(i)[0] == []  # untuned: the cost model, no candidates measured
    assert multi >= 1


@pytest.mark.parametrize("prefix,fm", fixture_models(), ids=lambda v: v if isinstance(v, str) else "")
def test_every_tuner_candidate_bit_exact(prefix, fm, engine):
    """Each geometry the tuner may pick, forced layer by layer, equals the reference."""
    if engine == "popc":
        return
    plan = B.Plan(fm.spec, fm.store, fm.x.shape[0])
    for i in range(fm.spec.n_layers):
        names, pick, _ = plan.layer_choice(i)
        for k in range(len(names)):
            plan.set_layer_choice(i, k)
            lg, lb = plan.run(fm.x)
            assert np.array_equal(lg.view(np.uint64), fm.logits.view(np.uint64)), (i, names[k], plan.engines())
        if names:
            plan.set_layer_choice(i, pick)


def test_device_run_reports_nonfinite_input(engine):
    """plan_run_device cannot throw mid-stream; input_status reports run_inference's
    invalid_input condition for the last device run (and clears for a finite input)."""
    import torch
    m = M.make_model("bad", "8C3-8FC", 8, 8, 3, 3)
    ws = Wt.build_weights(m, Wt.random_weights(m, 5))
    plan = B.Plan(m, ws, 4)
    x = torch.randn((4, 8, 8, 3), dtype=torch.float32, device="cuda")
    plan.run_device(x.data_ptr(), 4)
    torch.cuda.synchronize()
    assert not plan.input_status()
    x[2, 3, 4, 1] = float("inf")
    plan.run_device(x.data_ptr(), 4)
    torch.cuda.synchronize()
    assert plan.input_status()
    x[2, 3, 4, 1] = 0.5
    plan.run_device(x.data_ptr(), 4)
    torch.cuda.synchronize()
    assert not plan.input_status()


def test_fused_input_check_of_stride4_first_conv(engine):
    """The 7x7/4 first conv checks the input itself (no separate input pass): a non-finite
    value anywhere is still run_inference's invalid_input, through plan_run and through
    plan_run_device's status, and finite inputs stay bit-exact."""
    import torch
    m = M.make_model("s4", "32C7/4-32C3-10FC", 32, 32, 3, 10)
    ws = Wt.build_weights(m, Wt.random_weights(m, 91))
    x = np.random.default_rng(92).standard_normal((5, 32, 32, 3), dtype=np.float32)
    plan = B.Plan(m, ws, 5)
    lg, lb = plan.run(x)
    want, wl = oracle_run_inference(m.c_spec(), ws.c_store(), x)
    assert np.array_equal(lg.view(np.uint64), want.view(np.uint64)) and np.array_equal(lb, wl)
    for pos, val in (((4, 31, 31, 2), np.inf), ((0, 0, 0, 0), np.nan), ((2, 17, 5, 1), -np.inf)):
        bad = x.copy()
        bad[pos] = val
        with pytest.raises(capi.BtnnError) as e:
            plan.run(bad)
        assert e.value.code == capi.BTNN_INVALID_INPUT
        xd = torch.from_numpy(bad).cuda()
        plan.run_device(xd.data_ptr(), 5)
        torch.cuda.synchronize()
        assert plan.input_status()
    lg2, _ = plan.run(x)
    assert np.array_equal(lg2.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("name,hw,batch", [("mnist-mlp", 128, 200), ("mnist-mlp", 128, 37), ("mnist-mlp", 28, 333)])
def test_e2e_chunked_pipeline_pinned_and_pageable(name, hw, batch):
    """plan_run's measured input pipelining (chunk schedule from the calibrated copy / graph
    model; per-chunk result copies on their own stream when the host buffers are pinned):
    pinned and pageable host buffers both give the oracle's logits, whatever the schedule."""
    import ctypes as C

    import torch

    m = M.stock_model(name, hw, hw)
    ws = Wt.build_weights(m, Wt.random_weights(m, 3))
    x = np.random.default_rng(4).standard_normal((batch, m.in_h, m.in_w, m.in_c), dtype=np.float32)
    plan = B.Plan(m, ws, batch)
    lg, lb = plan.run(x)  # pageable (numpy) buffers; the first host run calibrates the model
    sched = plan.e2e_schedule(batch)
    if m.in_h * m.in_w * m.in_c * 4 >= 64 * 1024:  # pipelined: a measured multi-chunk schedule
        assert sched is not None and sum(sched["chunks"]) == batch and all(c > 0 for c in sched["chunks"])
    else:  # small inputs: one graph, no calibration
        assert sched is None
    xh = torch.from_numpy(x).pin_memory()
    lh = torch.zeros((batch, m.classes), dtype=torch.float64).pin_memory()
    bh = torch.zeros((batch,), dtype=torch.int32).pin_memory()
    for k in range(2):
        capi.check(capi.lib().btnn_cuda_plan_run(plan.h, C.cast(xh.data_ptr(), C.POINTER(C.c_float)), batch,
                                                 C.cast(lh.data_ptr(), C.POINTER(C.c_double)),
                                                 C.cast(bh.data_ptr(), C.POINTER(C.c_int32))))
        assert np.array_equal(lh.numpy().view(np.uint64), lg.view(np.uint64)), (k, sched)
        assert np.array_equal(bh.numpy(), lb)
        lh.zero_()
        bh.zero_()
    want, wl = oracle_run_inference(m.c_spec(), ws.c_store(), x)
    assert np.array_equal(lg.view(np.uint64), want.view(np.uint64))
    assert np.array_equal(lb, wl)


def test_e2e_pipeline_two_shards():
    """Two shards on device 0 (two host threads), each calibrating and pipelining its half of a
    large-input batch: the oracle's logits."""
    m = M.stock_model("mnist-mlp", 128, 128)
    ws = Wt.build_weights(m, Wt.random_weights(m, 5))
    x = np.random.default_rng(6).standard_normal((150, m.in_h, m.in_w, m.in_c), dtype=np.float32)
    plan = B.Plan(m, ws, 150, devices=(0, 0))
    for _ in range(2):
        lg, lb = plan.run(x)
        want, wl = oracle_run_inference(m.c_spec(), ws.c_store(), x)
        assert np.array_equal(lg.view(np.uint64), want.view(np.uint64))
        assert np.array_equal(lb, wl)
    for shard in (0, 1):
        sched = plan.e2e_schedule(75, shard)
        assert sched is not None and sum(sched["chunks"]) == 75


@pytest.mark.parametrize("hot", [(), (200, 260), (70, 63)])
def test_fused_cross_tile_argmax_ties(hot):
    """First-index argmax over many column tiles of the last FC (300 classes = 5 tiles of the
    packed BMM): identical logits everywhere -> 0; a tie between two tiles -> the earlier
    index; a tie across a tile boundary -> the earlier one (inference.hpp:177-184)."""
    m = M.make_model("tie", "128FC", 16, 16, 1, 300, [])
    fw = Wt.random_weights(m, 9)
    last = fw.layers[-1]
    U, K = m.layers[-1].units, m.layers[-1].in_channels
    w = last["weights"].reshape(U, K)
    w[:] = w[0]
    for k in ("gamma", "mean", "var"):
        last[k][:] = last[k][0]
    last["gamma"][:] = abs(last["gamma"][0]) + 0.5
    last["beta"][:] = 0.0
    for h in hot:
        last["beta"][h] = 100.0
    ws = Wt.build_weights(m, fw)
    x = np.random.default_rng(3).standard_normal((200, 16, 16, 1), dtype=np.float32)
    plan = B.Plan(m, ws, 200)
    for _ in range(2):  # (first run captures the graph, second replays it)
        lg, lb = plan.run(x)
        want, wl = oracle_run_inference(m.c_spec(), ws.c_store(), x)
        assert np.array_equal(lg.view(np.uint64), want.view(np.uint64))
        assert np.array_equal(lb, wl)
        assert (lb == (min(hot) if hot else 0)).all()
