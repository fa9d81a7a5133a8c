"""BENN ensembles: hard / soft bagging and boosting
(weighted votes / weighted logits) of K member BNNs, combined on the device
(btnn_cuda_benn_combine). The combine rules are restated here in plain numpy loops (member-order f64 sum,
first-max argmax, lowest-index vote ties) and checked against the package; the N>1 combine
runs on a world-size-2 gloo group with the C oracle standing in for each rank's device; the
GPU test runs three member plans and compares with the oracle members combined the same way."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle_lib import oracle_run_inference
from paper_2006_16578_b200 import ensemble as E
from paper_2006_16578_b200 import model as M
from paper_2006_16578_b200 import weights as W


def _members(k=3):
    m = M.make_model("benn", "8C3-P2-8C3-16FC", 8, 8, 3, 5, [(0, 2)])
    return m, [W.build_weights(m, W.random_weights(m, 100 + i)) for i in range(k)]


def _loop_soft(logits):
    k, b, c = len(logits), logits[0].shape[0], logits[0].shape[1]
    mean = np.zeros((b, c))
    lab = np.zeros(b, dtype=np.int32)
    for i in range(b):
        for j in range(c):
            s = logits[0][i, j]
            for m in range(1, k):
                s = s + logits[m][i, j]
            mean[i, j] = s / k
        best = 0
        for j in range(1, c):
            if mean[i, j] > mean[i, best]:
                best = j
        lab[i] = best
    return mean, lab


def test_combine_rules_vs_loop_restatement():
    rng = np.random.default_rng(7)
    logits = [rng.standard_normal((9, 6)) * 10 for _ in range(4)]
    logits[1][0] = logits[0][0]  # ties in the mean
    mean, lab = E.combine_soft(logits)
    wm, wl = _loop_soft(logits)
    assert np.array_equal(mean.view(np.uint64), wm.view(np.uint64)) and np.array_equal(lab, wl)
    labels = [rng.integers(0, 6, 9) for _ in range(4)]
    labels[0][0], labels[1][0], labels[2][0], labels[3][0] = 4, 2, 4, 2  # a 2-2 tie -> class 2
    votes, hl = E.combine_hard(labels, 6)
    assert hl[0] == 2
    for i in range(9):
        cnt = [sum(int(labels[m][i] == j) for m in range(4)) for j in range(6)]
        assert list(votes[i]) == cnt and hl[i] == int(np.argmax(cnt))


def _loop_boost(labels, alpha, classes):
    k, b = len(labels), len(labels[0])
    score = np.zeros((b, classes))
    for i in range(b):
        for j in range(classes):
            acc = 0.0
            for m in range(k):
                if labels[m][i] == j:
                    acc = acc + alpha[m]
            score[i, j] = acc
    return score, np.array([_first_max(r) for r in score], dtype=np.int32)


def _loop_boost_soft(logits, alpha):
    k, b, c = len(logits), logits[0].shape[0], logits[0].shape[1]
    score = np.zeros((b, c))
    for i in range(b):
        for j in range(c):
            acc = alpha[0] * logits[0][i, j]
            for m in range(1, k):
                acc = acc + alpha[m] * logits[m][i, j]
            score[i, j] = acc
    return score, np.array([_first_max(r) for r in score], dtype=np.int32)


def _first_max(row):
    best = 0
    for j in range(1, len(row)):
        if row[j] > row[best]:
            best = j
    return best


def _same(a, b):
    return np.array_equal(np.asarray(a, np.float64).view(np.uint64), np.asarray(b, np.float64).view(np.uint64))


def test_boosting_rules_vs_loop_restatement():
    rng = np.random.default_rng(17)
    logits = [rng.standard_normal((13, 7)) * 10 for _ in range(5)]
    labels = [rng.integers(0, 7, 13) for _ in range(5)]
    alpha = [0.7, 0.1, 0.2, 0.30000000000000004, 1e-3]
    labels[0][0], labels[1][0], labels[2][0] = 3, 1, 1  # 0.7 vs 0.1 + 0.2 (+...): rounding-sensitive
    sc, lb = E.combine_boost(labels, alpha, 7)
    wsc, wlb = _loop_boost(labels, alpha, 7)
    assert _same(sc, wsc) and np.array_equal(lb, wlb)
    sc, lb = E.combine_boost_soft(logits, alpha)
    wsc, wlb = _loop_boost_soft(logits, alpha)
    assert _same(sc, wsc) and np.array_equal(lb, wlb)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    from oracle_lib import oracle_run_inference as run
    from paper_2006_16578_b200 import ensemble as EE
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, ws = _members(world)
    x = np.random.default_rng(8).standard_normal((6, 8, 8, 3), dtype=np.float32)
    lg, lb = run(m.c_spec(), ws[rank].c_store(), x)  # this rank's member
    alpha = [0.6, 0.4]
    got = {mode: EE.combine_across_ranks(lg, lb, mode, alpha=alpha) for mode in EE.MODES}
    if rank == 0:
        outs = [run(m.c_spec(), w.c_store(), x) for w in ws]
        ok = []
        for mode, (sc, lab) in got.items():
            want, wl = EE.combine_host(mode, [o[0] for o in outs], [o[1] for o in outs], m.classes, alpha)
            ok.append(np.array_equal(np.asarray(sc, np.float64).view(np.uint64), want.view(np.uint64))
                      and np.array_equal(lab, wl))
        q.put((all(ok[:2]), all(ok)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_ensemble_combine():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    soft_ok, hard_ok = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
    assert soft_ok and hard_ok


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["soft", "hard", "boost", "boost_soft"])
def test_gpu_ensemble_matches_oracle_members(mode):
    """Three member plans on cuda:0, combined on the device, vs the oracle's members combined
    by the loop restatements."""
    m, ws = _members(3)
    x = np.random.default_rng(9).standard_normal((11, 8, 8, 3), dtype=np.float32)
    alpha = [0.5, 0.25, 0.30000000000000004]
    ens = E.Ensemble([(m, w) for w in ws], 11)
    got, gl = ens.run(x, mode, alpha if mode.startswith("boost") else None)
    outs = [oracle_run_inference(m.c_spec(), w.c_store(), x) for w in ws]
    lg, lb = [o[0] for o in outs], [o[1] for o in outs]
    if mode == "soft":
        want, wl = _loop_soft(lg)
    elif mode == "hard":
        v, wl = E.combine_hard(lb, m.classes)
        want = v.astype(np.float64)
    elif mode == "boost":
        want, wl = _loop_boost(lb, alpha, m.classes)
    else:
        want, wl = _loop_boost_soft(lg, alpha)
    assert _same(got, want)
    assert np.array_equal(gl, wl)


@pytest.mark.gpu
def test_gpu_benn_combine_kernel_adversarial():
    """The device combine alone on many members with ties, negative weights and rounding-
    sensitive sums, every mode vs the loop restatements."""
    import ctypes as C

    import torch

    from paper_2006_16578_b200 import capi
    rng = np.random.default_rng(23)
    k, b, c = 37, 129, 10
    lg = rng.standard_normal((k, b, c)) * np.exp(rng.uniform(-30, 30, (k, b, 1)))
    lg[:, 0, :] = 1.0  # all-equal row: first max is class 0
    lb = rng.integers(0, c, (k, b)).astype(np.int32)
    alpha = list(rng.uniform(-1, 2, k))
    dev = torch.device("cuda", 0)
    dlg, dlb = torch.from_numpy(lg).to(dev), torch.from_numpy(lb).to(dev)
    for mode, code in E.MODES.items():
        sc = torch.empty((b, c), dtype=torch.float64, device=dev)
        out = torch.empty((b,), dtype=torch.int32, device=dev)
        capi.check(capi.lib().btnn_cuda_benn_combine(dlg.data_ptr(), dlb.data_ptr(), k, b, c, (C.c_double * k)(*alpha),
                                                      code, sc.data_ptr(), out.data_ptr(), None))
        torch.cuda.synchronize()
        want, wl = {"soft": lambda: _loop_soft(list(lg)), "hard": lambda: E.combine_host("hard", None, list(lb), c),
                    "boost": lambda: _loop_boost(list(lb), alpha, c),
                    "boost_soft": lambda: _loop_boost_soft(list(lg), alpha)}[mode]()
        assert _same(sc.cpu().numpy(), want), mode
        assert np.array_equal(out.cpu().numpy(), wl), mode
