"""Rank body for tests/test_multiproc.py::test_relaunch_torchrun_gloo: started by
paper_2311_01135_b200.launch.relaunch_torchrun (the path `bench.py --gpus N` takes), it
labels its shard of a molecule list with a host function, then does what bench.py does
with the process group - barrier, max over ranks of a time, sum over ranks of a count - on
gloo, and rank 0 prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2311_01135_b200 import nuclear_repulsion, synth  # noqa: E402
from paper_2311_01135_b200.launch import Ranks  # noqa: E402
from paper_2311_01135_b200.queue import shard  # noqa: E402


def main():
    ranks = Ranks("gloo")
    mols = synth.batch(5, 3, seed=3)
    mine, idx = shard(mols, ranks.rank, ranks.world)
    enn = sum(nuclear_repulsion(m) for m in mine)
    ranks.barrier()
    t = ranks.max(float(ranks.rank + 1))
    n = ranks.sum(len(mine))
    e = ranks.sum(enn)
    if ranks.rank == 0:
        print(json.dumps({"world": ranks.world, "max": t, "n": n, "enn": e}), flush=True)
    ranks.close()


if __name__ == "__main__":
    main()
