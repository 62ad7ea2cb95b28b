"""Multi-GPU paths.

1. Scenario sharding (BASELINE config 4: independent scenarios over N GPUs).
   One process per GPU (torchrun).  Scenarios are split contiguously and evenly over
   the ranks; each rank solves its shard in one device launch; there is no data-path
   collective.  ``gather_reports`` (tests, tooling) collects the per-rank results on
   every rank in scenario order; the benchmark only reduces its timing (max).

2. Pair sharding of ONE very large scenario (BASELINE config 5, n = 256).
   ``am_solve_pair_sharded`` — every rank calls it with the same spec.  For n > 64 (the
   large-fleet kernel) each GPU owns a contiguous, cost-balanced range of the
   (agent-block pair x sample) units -- a range of agent pairs at all samples -- run by
   one CTA per SM; the one per-iteration exchange (its 3 x n x n_v partial right-hand
   sides plus two residual scalars) happens INSIDE the persistent kernel through
   peer-mapped buffers (CUDA IPC over NVLink) and a system-scope barrier, summed in rank
   order so every GPU computes identical iterates.  (n <= 64: the multi-cluster kernel,
   each GPU a slice of the time samples, bitwise the single-GPU result.)
   torch.distributed only moves the 64-byte IPC handles and provides the host barrier;
   there is no NCCL call on the data path (the exchange is fused into the solve).
"""

from __future__ import annotations

import os
import time

import numpy as np


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


MAX_PAIR_SHARDS = 8  # st_solve_sharded: G <= 8


class ShardGroup:
    """The peer-mapped exchange buffers of one plan over the ranks of a process group.

    Collective (every rank constructs it, same plan fingerprint): allocates this GPU's
    buffer, all-gathers the IPC handles, maps the peers' buffers, and has rank 0 zero
    the barrier word before a host barrier.  ``bufs[g]`` is group g's buffer as seen
    from this process.  Reusable across solves of the same plan (the in-kernel
    barrier resets itself); ``close()`` is collective too.
    """

    def __init__(self, plan, rank: int, world: int, group=None):
        import torch.distributed as dist
        if not 1 <= world <= MAX_PAIR_SHARDS:
            raise ValueError(f"pair sharding supports 1..{MAX_PAIR_SHARDS} GPUs, got {world}")
        self.plan, self.rank, self.world, self.group = plan, rank, world, group
        self.layout = plan.shard_layout(world)
        ptr, handle = plan.shard_buffer(self.layout["buffer_bytes"])
        handles = [None] * world
        dist.all_gather_object(handles, handle, group=group)
        if handles[rank] != handle:
            raise RuntimeError("IPC handle exchange returned handles out of rank order")
        self.bufs = [ptr if g == rank else plan.shard_open(h) for g, h in enumerate(handles)]
        if rank == 0:
            plan.shard_reset(self.bufs[0])
        dist.barrier(group=group)
        self._open = True

    def close(self) -> None:
        import torch.distributed as dist
        if not self._open:
            return
        dist.barrier(group=self.group)  # no peer may still be inside a kernel using our buffer
        for g, b in enumerate(self.bufs):
            if g != self.rank:
                self.plan.shard_close(b, True)
        self.plan.shard_close(self.bufs[self.rank], False)
        self._open = False


def am_solve_pair_sharded(spec, config=None, cache=None, group=None, shard_group: ShardGroup | None = None):
    """Solve ONE scenario with its agent pairs sharded over the GPUs of ``group``.

    Every rank calls this with the same ``spec``/``config`` (torchrun, one process per
    GPU, ``config.device`` = this rank's GPU; default LOCAL_RANK).  Returns the
    ``SolveReport`` on rank 0 and ``None`` elsewhere.  Same validation and errors as
    ``am_solve`` (reference solver.py:363-367); every GPU holds identical iterates (the
    single-GPU solve's within the parity bar; bitwise for one rank).
    """
    import torch.distributed as dist
    from . import engine, kkt, poly
    from .spec import validate

    config = config or engine.SolverConfig()
    if config.track_descent or config.keep_state:
        raise NotImplementedError("pair-sharded solves support neither track_descent nor keep_state")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = engine._opt(config, "device", None)
    if dev is None or (dev == 0 and "LOCAL_RANK" in os.environ):
        config = _with_device(config, int(os.environ.get("LOCAL_RANK", 0)))
    v = validate(spec)
    if v:
        raise engine._infeasible(v)
    t0 = time.perf_counter()
    n, n_obs = len(spec.start), len(spec.obstacles)
    basis = poly.for_spec(spec)
    fp = kkt.fingerprint(basis, n, n_obs)
    c0, beq, geom = engine.pack([spec], basis)
    t1 = time.perf_counter()
    cache, foreign = engine._resolve_cache(cache)
    schedule = config.schedule()
    before = cache.stats()
    plan = engine._plan_for(cache, fp, basis, schedule, n, n_obs, config.device)
    engine._sync_foreign(cache, foreign, before)
    own = shard_group is None
    sg = ShardGroup(plan, rank, world, group) if own else shard_group
    try:
        t2 = time.perf_counter()
        out = plan.solve_sharded(world, rank, sg.bufs, c0, beq, geom, schedule.switch_every, config.max_iters,
                                 config.tolerance)
        t3 = time.perf_counter()
    finally:
        if own:
            sg.close()
    if rank != 0:
        return None
    out = dict(out, lam=None, d=None)
    rep = engine._make_reports([spec], out, basis, plan, cache, schedule, config, (t0, t1, t2, t3),
                               foreign=foreign)[0]
    rep.timings["pair_shards"] = world
    return rep


class _DeviceConfig:
    """A solver config (ours or the reference's) seen with a different device ordinal."""

    def __init__(self, config, device: int):
        self._config, self.device = config, device

    def __getattr__(self, name):
        return getattr(self._config, name)


def _with_device(config, device: int):
    return _DeviceConfig(config, device)


def pair_shard_samples(m: int, world: int, cluster: int, clusters_per_gpu: int) -> list[tuple[int, int]]:
    """Time samples [lo, hi) each GPU owns (mirror of the kernel's split over the
    ``world * clusters_per_gpu * cluster`` CTAs: CTA q of P*C takes [q*m/(P*C), (q+1)*m/(P*C)))."""
    parts = world * clusters_per_gpu * cluster
    per_gpu = clusters_per_gpu * cluster
    return [(g * per_gpu * m // parts, (g + 1) * per_gpu * m // parts) for g in range(world)]
