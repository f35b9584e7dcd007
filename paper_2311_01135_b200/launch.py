"""One process per GPU on one node: launch helpers shared by bench.py and the
labeling pipeline.

The data path has no collective (molecules are independent).  `torch.distributed` is used
only for the plumbing the measurement needs - a barrier around the timed region and the
max-over-ranks reduction of the device time - so NCCL on a GPU box, gloo for the CPU tests.

* `relaunch_torchrun(n, script, argv)` re-executes `script` under
  `python -m torch.distributed.run --nnodes=1 --nproc-per-node n --master-addr 127.0.0.1`
  (the command form the benchmark driver uses), so `bench.py --gpus N` started as a plain
  process runs N ranks instead of silently running one;
* `Ranks` wraps the process group: barrier, max over ranks, teardown.
"""

from __future__ import annotations

import os
import socket
import subprocess
import sys


def dist_env() -> tuple[int, int, int]:
    """(world size, rank, local rank) from the torchrun environment (1, 0, 0 when absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def under_launcher() -> bool:
    return "WORLD_SIZE" in os.environ and "RANK" in os.environ


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def torchrun_argv(nproc: int, script: str, argv: list[str], port: int | None = None) -> list[str]:
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr=127.0.0.1", f"--master-port={port or free_port()}", script, *argv]


def relaunch_torchrun(nproc: int, script: str, argv: list[str], env: dict | None = None) -> int:
    """Run `script argv` as `nproc` ranks on this node; returns the launcher's exit code."""
    e = dict(os.environ if env is None else env)
    e.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(torchrun_argv(nproc, script, argv), env=e)


class Ranks:
    """The process group of a launched job (or a no-op world of one)."""

    def __init__(self, backend: str | None = None, device=None):
        self.world, self.rank, self.local = dist_env()
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist

            kw = {}
            if backend == "nccl" and device is not None:
                kw["device_id"] = device
            dist.init_process_group(backend, **kw)
            self.dist = dist
            self.backend = backend

    def barrier(self) -> None:
        if self.dist is not None:
            self.dist.barrier()

    def max(self, x: float) -> float:
        """max over ranks of a scalar (the slowest rank's time)."""
        if self.dist is None:
            return float(x)
        import torch

        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.dist is None:
            return float(x)
        import torch

        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self) -> None:
        if self.dist is not None:
            self.dist.destroy_process_group()
            self.dist = None
