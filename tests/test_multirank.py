"""World-size-2 gloo coverage of the N>1 path (CPU): each rank runs its contiguous shard
of the batch (through the C oracle standing in for its device), the timed region is
max-reduced, and the gathered logits equal the single-process run bit for bit."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2006_16578_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_covers_batch():
    for total in (1, 7, 8, 511, 512, 4096):
        for world in (1, 2, 3, 4, 8):
            spans = [D.shard_range(total, r, world) for r in range(world)]
            got = []
            for st, n in spans:
                got += list(range(st, st + n))
            assert got == list(range(total)), (total, world)


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist

    from oracle_lib import oracle_run_inference
    from paper_2006_16578_b200 import model as M
    from paper_2006_16578_b200 import weights as W
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = M.make_model("mr", "8C3-P2-8C3-16FC", 8, 8, 3, 5, [(0, 2)])
    ws = W.build_weights(m, W.random_weights(m, 3))
    x = np.random.default_rng(4).standard_normal((7, 8, 8, 3), dtype=np.float32)
    st, n = D.shard_range(7, rank, world)
    lg, lb = oracle_run_inference(m.c_spec(), ws.c_store(), x[st:st + n])
    t = D.max_over_ranks(float(rank + 1))
    full = D.gather_rows(torch.from_numpy(lg))
    labels = D.gather_rows(torch.from_numpy(lb.astype(np.int64)))
    if rank == 0:
        want, wl = oracle_run_inference(m.c_spec(), ws.c_store(), x)
        q.put((t, np.array_equal(full.numpy().view(np.uint64), want.view(np.uint64)),
               np.array_equal(labels.numpy(), wl)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_inference():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    t, logits_ok, labels_ok = q.get(timeout=10)
    assert t == 2.0
    assert logits_ok and labels_ok
