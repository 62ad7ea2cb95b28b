"""Multi-GPU scenario sharding (BASELINE config 4: independent scenarios over N GPUs).

One process per GPU (torchrun).  Scenarios are split contiguously and evenly over
the ranks; each rank solves its shard in one device launch; there is no data-path
collective.  ``gather_reports`` (tests, tooling) collects the per-rank results on
every rank in scenario order; the benchmark only reduces its timing (max).
"""

from __future__ import annotations


def shard_bounds(total: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the scenarios owned by ``rank`` (contiguous, sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    return rank * total // world, (rank + 1) * total // world


def solve_shard(specs, rank: int, world: int, solve_batch):
    """Solve this rank's contiguous shard with ``solve_batch(list_of_specs) -> list``."""
    lo, hi = shard_bounds(len(specs), rank, world)
    return lo, list(solve_batch(specs[lo:hi])) if hi > lo else []


def gather_reports(local, world: int):
    """All-gather per-rank result lists (any picklable items) -> one list in rank order."""
    if world == 1:
        return list(local)
    import torch.distributed as dist
    parts = [None] * world
    dist.all_gather_object(parts, list(local))
    return [x for part in parts for x in part]
