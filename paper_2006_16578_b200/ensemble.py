"""BENN ensembles over device plans (the paper's §8):
K independently trained BNNs ("members") classify the same batch and their outputs are
combined — hard bagging (majority vote of the members' labels) or soft bagging (the mean of
the members' f64 logits, then the first-max argmax of run_inference, inference.hpp:177-184).

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

    def run(self, x, mode: str = "soft"):
        logits, labels = self.member_outputs(x)
        if mode == "soft":
            return combine_soft(logits)
        if mode == "hard":
            return combine_hard(labels, self.classes)
        raise ValueError(f"unknown ensemble mode {mode!r}")


def combine_across_ranks(local_logits, local_labels, mode: str = "soft", device=None):
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
    if mode == "soft":
        return combine_soft(lg)
    return combine_hard(lb, np.asarray(local_logits).shape[1])
