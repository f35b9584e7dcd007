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


def test_relaunch_torchrun_gloo():
    """The launch path of `bench.py --gpus N` (relaunch under torch.distributed.run, one
    process per rank, 127.0.0.1 rendezvous) with world size 2 on gloo: every rank labels
    its shard, the max-over-ranks time and the molecule sum come back to rank 0."""
    import json
    import subprocess
    import sys

    from paper_2311_01135_b200.launch import torchrun_argv

    here = os.path.dirname(os.path.abspath(__file__))
    cmd = torchrun_argv(2, os.path.join(here, "dist_probe.py"), [])
    env = dict(os.environ, OMP_NUM_THREADS="1")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["world"] == 2 and d["max"] == 2.0 and d["n"] == 5
    ref = sum(nuclear_repulsion(m) for m in synth.batch(5, 3, seed=3))
    assert abs(d["enn"] - ref) < 1e-9 * abs(ref)
    del sys


def test_bench_gpus_flag_relaunches(monkeypatch):
    """`bench.py --gpus 2` started as a plain process re-executes itself under torchrun with
    two ranks instead of running one (the round-1 bug: --gpus was parsed and ignored)."""
    import importlib.util
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    seen = {}

    def fake_relaunch(n, script, argv, env=None):
        seen["n"], seen["script"], seen["argv"] = n, script, argv
        return 0

    import paper_2311_01135_b200.launch as launch

    monkeypatch.setattr(launch, "relaunch_torchrun", fake_relaunch)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2", "--steps", "3"])
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert ex.value.code == 0
    assert seen["n"] == 2 and seen["script"].endswith("bench.py") and seen["argv"] == ["--gpus", "2", "--steps", "3"]
    # under a launcher whose world size disagrees with --gpus the bench refuses to run
    monkeypatch.setenv("WORLD_SIZE", "1")
    monkeypatch.setenv("RANK", "0")
    with pytest.raises(SystemExit) as ex2:
        bench.main()
    assert "launcher started 1" in str(ex2.value.code)
