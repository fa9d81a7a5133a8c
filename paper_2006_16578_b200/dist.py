"""Multi-GPU plumbing for batch-sharded inference (one process per GPU).

BNN inference couples no samples (bn uses frozen statistics, layer_math.hpp:32-34), so
the data path has no collective: each rank runs its contiguous shard of the batch on its
own device. The only cross-rank traffic is bookkeeping — a barrier and a
max-reduce of the timed region, and optionally one gather of the logits/labels at the
end (the paper's ensemble-free analogue of its NCCL reduce).
"""
from __future__ import annotations

import os


def env():
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [start, start+count) of `total` samples for `rank`: ceil split,
    the same rule btnn_cuda_plan_run uses across the devices of one plan."""
    per = -(-total // world)
    start = min(rank * per, total)
    return start, max(0, min(per, total - start))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the timed region is reported as the slowest rank)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local, device=None):
    """All-gather of per-rank row blocks (e.g. logits) into the global batch order.
    Shards may differ in length by the ceil split; rows are padded to the max and cut."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world = dist.get_world_size()
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    mx = int(max(int(s.item()) for s in sizes))
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([b[: int(s.item())] for b, s in zip(bufs, sizes)], dim=0)
