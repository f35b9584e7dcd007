"""Per-GPU molecule queues: molecules are independent, so a job is
sharded round-robin over ranks (molecule k -> rank k mod world) with no data-path
collective; results are merged back into input order on the host."""

from __future__ import annotations


def shard(items: list, rank: int, world: int) -> tuple[list, list[int]]:
    """(items of this rank, their global indices)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world size {world}")
    idx = list(range(rank, len(items), world))
    return [items[k] for k in idx], idx


def merge(parts: list[tuple[list[int], list]]) -> list:
    """Inverse of shard: [(indices, results) per rank] -> results in global order."""
    n = sum(len(ix) for ix, _ in parts)
    out = [None] * n
    for ix, res in parts:
        if len(ix) != len(res):
            raise ValueError("indices/results length mismatch")
        for k, r in zip(ix, res):
            out[k] = r
    if any(o is None for o in out):
        raise ValueError("merge: missing results")
    return out


def run_sharded(mols: list, basis, opts, rank: int, world: int, gather=None) -> list:
    """Label this rank's shard on its GPU; with `gather` (e.g. an all_gather_object wrapper)
    return the merged global list, else this rank's (indices, results)."""
    from .scf import scf_batch

    mine, idx = shard(mols, rank, world)
    res = scf_batch(mine, basis, opts, errors="return") if mine else []
    if gather is None:
        return [(idx, res)]
    return merge(gather((idx, res)))
