"""Multi-process sharding of molecule queues (world_size 2, gloo on CPU): the sharded run
with a host-side per-molecule function merges back to the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_01135_b200 import nuclear_repulsion, synth
from paper_2311_01135_b200.queue import merge, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mols = synth.batch(n, 3, seed=3)
    mine, idx = shard(mols, rank, world)
    res = [nuclear_repulsion(m) for m in mine]
    parts = [None] * world
    dist.all_gather_object(parts, (idx, res))
    merged = merge(parts)
    # max-over-ranks timing reduction used by bench.py
    t = torch_tensor(float(rank + 1))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        out_q.put((merged, float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def torch_tensor(x):
    import torch

    return torch.tensor([x], dtype=torch.float64)


def test_shard_merge_roundtrip():
    items = list(range(11))
    parts = []
    for r in range(3):
        mine, idx = shard(items, r, 3)
        assert all(k % 3 == r for k in idx)
        parts.append((idx, [x * 10 for x in mine]))
    assert merge(parts) == [x * 10 for x in items]
    with pytest.raises(ValueError):
        shard(items, 3, 3)


def test_gloo_world2_sharded_queue():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n = 7
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = [nuclear_repulsion(m) for m in synth.batch(n, 3, seed=3)]
    np.testing.assert_array_equal(np.array(merged), np.array(ref))
    assert tmax == 2.0
