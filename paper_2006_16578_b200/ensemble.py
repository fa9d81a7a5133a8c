"""BENN ensembles over device plans (the paper's §8):
K independently trained BNNs ("members") classify the same batch and their outputs are
combined — hard bagging (majority vote of the members' labels), soft bagging (the mean of
the members' f64 logits) or boosting (Zhu et al.'s BENN: member weights alpha_k, a weighted
vote of the labels or a weighted sum of the logits), then the first-max argmax of
run_inference (inference.hpp:177-184).

Ensemble.run combines on the device (btnn_cuda_benn_combine, csrc/ensemble.cu) when every
member runs on one device: the members write their logits into one K x B x classes device
buffer and only the combined scores come back. The numpy combine_* functions below are the
same member-order folds on the host (the checker in tests/, and the cross-rank combine).

One member per device (or several per device); across processes each rank runs its member(s)
and the combine needs the other members' outputs. The combine is defined in member order so
that every rank — and the CPU check in tests/ — gets bit-identical results: the logits are
all-gathered (not all-reduced: a reduction tree would make the f64 sum order depend on the
collective's algorithm) and summed in member order on every rank.
"""
from __future__ import annotations

import numpy as np


def combine_soft(member_logits):
    """Mean of the members' logits, summed in member order (K x B x classes -> B x classes),
    and the first-max labels (inference.hpp:177-184)."""
    it = iter(member_logits)
    acc = np.array(next(it), dtype=np.float64, copy=True)
    k = 1
    for lg in it:
        acc = acc + np.asarray(lg, dtype=np.float64)
        k += 1
    mean = acc / float(k)
    return mean, np.argmax(mean, axis=1).astype(np.int32)


def combine_hard(member_labels, classes: int):
    """Majority vote of the members' labels; ties go to the lowest class index (the
    first-max rule). Returns (votes B x classes int32, labels)."""
    lab = np.asarray(member_labels, dtype=np.int64)
    votes = np.zeros((lab.shape[1], classes), dtype=np.int32)
    for k in range(lab.shape[0]):
        np.add.at(votes, (np.arange(lab.shape[1]), lab[k]), 1)
    return votes, np.argmax(votes, axis=1).astype(np.int32)


def combine_boost(member_labels, alpha, classes: int):
    """Boosting, weighted vote: score[c] = sum_k (label_k == c ? alpha_k : 0), summed in member
    order from 0.0; first-max labels."""
    lab = np.asarray(member_labels, dtype=np.int64)
    score = np.zeros((lab.shape[1], classes), dtype=np.float64)
    rows = np.arange(lab.shape[1])
    for k in range(lab.shape[0]):
        score[rows, lab[k]] = score[rows, lab[k]] + float(alpha[k])
    return score, np.argmax(score, axis=1).astype(np.int32)


def combine_boost_soft(member_logits, alpha):
    """Boosting, weighted logits: score = fl(alpha_0 l_0) + fl(alpha_1 l_1) + ... in member
    order; first-max labels."""
    it = iter(member_logits)
    acc = float(alpha[0]) * np.asarray(next(it), dtype=np.float64)
    for k, lg in enumerate(it, start=1):
        acc = acc + float(alpha[k]) * np.asarray(lg, dtype=np.float64)
    return acc, np.argmax(acc, axis=1).astype(np.int32)


MODES = {"hard": 0, "soft": 1, "boost": 2, "boost_soft": 3}


def combine_host(mode: str, logits, labels, classes: int, alpha=None):
    if mode == "soft":
        return combine_soft(logits)
    if mode == "hard":
        v, lb = combine_hard(labels, classes)
        return v.astype(np.float64), lb
    if mode == "boost":
        return combine_boost(labels, alpha, classes)
    if mode == "boost_soft":
        return combine_boost_soft(logits, alpha)
    raise ValueError(f"unknown ensemble mode {mode!r}")


class Ensemble:
    """Members = [(model, weight store), ...] on `devices` (member i on devices[i % n]).
    run(x, mode) returns (combined scores, labels): mode "soft" -> mean logits, "hard" ->
    vote counts."""

    def __init__(self, members, max_batch: int, devices=(0,)):
        from .btnn import Plan

        self.plans = [Plan(m, ws, max_batch, devices=(devices[i % len(devices)],)) for i, (m, ws) in
                      enumerate(members)]
        self.classes = self.plans[0].classes
        if any(p.classes != self.classes for p in self.plans):
            raise ValueError("ensemble members must share the class count")

    def member_outputs(self, x):
        outs = [p.run(x) for p in self.plans]
        return [o[0] for o in outs], [o[1] for o in outs]

    def run(self, x, mode: str = "soft", alpha=None):
        """(scores, labels): mode "soft" -> mean logits, "hard" -> vote counts (f64),
        "boost" -> weighted votes, "boost_soft" -> weighted logit sums (alpha: K weights).
        On one device the members' outputs stay on the GPU and btnn_cuda_benn_combine folds
        them there; members spread over devices are combined on the host."""
        if mode not in MODES:
            raise ValueError(f"unknown ensemble mode {mode!r}")
        if mode.startswith("boost") and (alpha is None or len(alpha) != len(self.plans)):
            raise ValueError("boosting needs one weight per member")
        devs = {p.device for p in self.plans}
        if len(devs) == 1 and -1 not in devs:
            return self._run_device(x, mode, alpha)
        logits, labels = self.member_outputs(x)
        return combine_host(mode, logits, labels, self.classes, alpha)

    def _run_device(self, x, mode, alpha):
        import ctypes as C

        import torch

        from . import capi

        x = np.ascontiguousarray(x, dtype=np.float32)
        dev = torch.device("cuda", self.plans[0].device)
        k, b = len(self.plans), x.shape[0]
        with torch.cuda.device(dev):
            st = torch.cuda.current_stream(dev)
            dx = torch.from_numpy(x).to(dev, non_blocking=False)
            lg = torch.empty((k, b, self.classes), dtype=torch.float64, device=dev)
            lb = torch.empty((k, b), dtype=torch.int32, device=dev)
            for i, p in enumerate(self.plans):
                p.run_device(dx.data_ptr(), b, lg[i].data_ptr(), lb[i].data_ptr(), st.cuda_stream)
            sc = torch.empty((b, self.classes), dtype=torch.float64, device=dev)
            out = torch.empty((b,), dtype=torch.int32, device=dev)
            al = (C.c_double * k)(*(alpha if alpha is not None else [1.0] * k))
            capi.check(capi.lib().btnn_cuda_benn_combine(lg.data_ptr(), lb.data_ptr(), k, b, self.classes, al,
                                                          MODES[mode], sc.data_ptr(), out.data_ptr(), st.cuda_stream))
            st.synchronize()
            return sc.cpu().numpy(), out.cpu().numpy()


def combine_across_ranks(local_logits, local_labels, mode: str = "soft", device=None, alpha=None):
    """Distributed combine: each rank holds its member's (B x classes) logits and labels for
    the same batch; all-gather them in rank (= member) order and combine identically on
    every rank (torch.distributed; NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        lg, lb = [np.asarray(local_logits)], [np.asarray(local_labels)]
    else:
        world = dist.get_world_size()
        t = torch.as_tensor(np.ascontiguousarray(local_logits), dtype=torch.float64, device=device)
        bufs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(bufs, t)
        lt = torch.as_tensor(np.ascontiguousarray(local_labels).astype(np.int64), device=device)
        lbufs = [torch.empty_like(lt) for _ in range(world)]
        dist.all_gather(lbufs, lt)
        lg = [b.cpu().numpy() for b in bufs]
        lb = [b.cpu().numpy() for b in lbufs]
    return combine_host(mode, lg, lb, np.asarray(local_logits).shape[1], alpha)
