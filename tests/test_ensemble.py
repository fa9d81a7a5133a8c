"""BENN ensembles: hard / soft bagging of K member
BNNs. The combine rules are restated here in plain numpy loops (member-order f64 sum,
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
    soft = EE.combine_across_ranks(lg, lb, "soft")
    hard = EE.combine_across_ranks(lg, lb, "hard")
    if rank == 0:
        outs = [run(m.c_spec(), w.c_store(), x) for w in ws]
        ws_, wl_ = EE.combine_soft([o[0] for o in outs])
        hv, hl = EE.combine_hard([o[1] for o in outs], m.classes)
        q.put((np.array_equal(soft[0].view(np.uint64), ws_.view(np.uint64)) and np.array_equal(soft[1], wl_),
               np.array_equal(hard[0], hv) and np.array_equal(hard[1], hl)))
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
@pytest.mark.parametrize("mode", ["soft", "hard"])
def test_gpu_ensemble_matches_oracle_members(mode):
    m, ws = _members(3)
    x = np.random.default_rng(9).standard_normal((11, 8, 8, 3), dtype=np.float32)
    ens = E.Ensemble([(m, w) for w in ws], 11)
    got, gl = ens.run(x, mode)
    outs = [oracle_run_inference(m.c_spec(), w.c_store(), x) for w in ws]
    if mode == "soft":
        want, wl = E.combine_soft([o[0] for o in outs])
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    else:
        want, wl = E.combine_hard([o[1] for o in outs], m.classes)
        assert np.array_equal(got, want)
    assert np.array_equal(gl, wl)
