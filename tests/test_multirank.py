"""N>1 path on CPU: world_size-2 gloo processes shard a scenario batch exactly as the
multi-GPU benchmark does (contiguous shards, no data-path collective), solve their
shard (the CPU oracle stands in for the device solver here) and all-gather the
reports; the result must equal the single-rank solve, scenario by scenario.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2011_04240_b200.dist import gather_reports, shard_bounds, solve_shard


def test_shard_bounds_partition():
    for total in (1, 7, 1024):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, seeds, out_q):
    import torch.distributed as dist

    from oracle import am_oracle
    from paper_2011_04240_b200 import generate_random
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    specs = [generate_random(5, (8, 8, 3), 0.4, s) for s in seeds]

    def solve_batch(batch):
        return [(am_oracle.solve(sp, max_iters=40)["coefficients"], am_oracle.solve(sp, max_iters=40)["iterations"])
                for sp in batch]

    lo, local = solve_shard(specs, rank, world, solve_batch)
    allr = gather_reports(local, world)
    if rank == 0:
        out_q.put([(c.tolist(), it) for c, it in allr])
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_matches_single_rank():
    from oracle import am_oracle
    from paper_2011_04240_b200 import generate_random
    seeds = list(range(5))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seeds, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert len(got) == len(seeds)
    for s, (c, it) in zip(seeds, got):
        ref = am_oracle.solve(generate_random(5, (8, 8, 3), 0.4, s), max_iters=40)
        assert it == ref["iterations"]
        np.testing.assert_array_equal(np.array(c), ref["coefficients"])


# ---- pair sharding plumbing (the device exchange itself is covered by the GPU tests) ------


class _FakePlan:
    """Stands in for native.Plan: records the shard calls a rank makes."""

    def __init__(self, rank, n, nv):
        self.rank, self.n, self.nv = rank, n, nv
        self.calls = []

    def shard_layout(self, groups):
        return {"cluster": 4, "clusters_per_gpu": 2, "buffer_bytes": 4096, "participants": 2 * groups}

    def shard_buffer(self, nbytes):
        self.calls.append(("buffer", nbytes))
        return 1000 + self.rank, b"h%d" % self.rank + bytes(62)

    def shard_open(self, handle):
        self.calls.append(("open", handle[:2]))
        return 2000 + int(handle[1:2])

    def shard_close(self, ptr, opened):
        self.calls.append(("close", ptr, opened))

    def shard_reset(self, buf0):
        self.calls.append(("reset", buf0))

    def solve_sharded(self, groups, rank, bufs, c0, beq, geom, switch_every, max_iters, tol):
        self.calls.append(("solve", groups, rank, list(bufs), float(np.abs(c0).sum()), float(np.abs(beq).sum())))
        hist = np.zeros((1, 3, max_iters))
        hist[0, :, :3] = 0.5
        return {"c": c0.copy(), "hist": hist, "iters": np.array([3], np.int32), "converged": np.array([True]),
                "timings_ms": (0.0, 1.0, 0.0)}


def _pair_worker(rank, world, port, out_q):
    import torch.distributed as dist

    from paper_2011_04240_b200 import SolverConfig, engine, generate_random
    from paper_2011_04240_b200.dist import am_solve_pair_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = generate_random(6, (8, 8, 3), 0.4, 3)
    fake = {}

    def plan_for(cache, fp, basis, schedule, n, n_obs, device):
        fake.setdefault("p", _FakePlan(rank, n, basis.num_coeffs))
        fake["device"] = device
        return fake["p"]

    engine._plan_for = plan_for
    # no GPU here: the post-solve collision check runs through the host restatement
    from paper_2011_04240_b200 import metrics
    def host_summary(trajs, specs, device=0):
        cols = [metrics.check_collisions(t, sp.geometry, sp.obstacles) for t, sp in zip(trajs, specs)]
        return [(c.min_normalized_distance, len(c.violations)) for c in cols]

    metrics.collision_summary_device_batch = host_summary
    rep = am_solve_pair_sharded(spec, SolverConfig(max_iters=20, device=rank))
    out_q.put((rank, fake["p"].calls, None if rep is None else (rep.iterations, rep.converged,
                                                                 np.asarray(rep.coefficients).shape)))
    dist.barrier()
    dist.destroy_process_group()


def test_pair_sharded_orchestration_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pair_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, (calls, rep)) for r, calls, rep in (q.get(timeout=300), q.get(timeout=300)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    solves = {}
    for r in (0, 1):
        calls, rep = got[r]
        kinds = [c[0] for c in calls]
        assert kinds[0] == "buffer" and calls[0][1] == 4096
        assert kinds.count("open") == 1 and calls[kinds.index("open")][1] == b"h%d" % (1 - r)
        assert kinds.count("reset") == (1 if r == 0 else 0)
        solve = calls[kinds.index("solve")]
        assert solve[1:3] == (2, r)
        # group g's buffer: own allocation locally, the mapped peer allocation otherwise
        assert solve[3] == [1000 + g if g == r else 2000 + g for g in range(2)]
        solves[r] = solve[4:]
        # peer mapping closed, then own buffer freed, after the solve
        assert kinds[-2:] == ["close", "close"] and calls[-1][2] is False
        if r == 0:
            assert rep == (3, True, (3, 6, rep[2][2]))
        else:
            assert rep is None
    assert solves[0] == solves[1]  # every rank solves the same scenario


def test_pair_shard_samples_partition():
    from paper_2011_04240_b200.dist import pair_shard_samples
    for m, world, C, K in ((100, 2, 16, 3), (100, 8, 4, 3), (17, 3, 1, 5)):
        spans = pair_shard_samples(m, world, C, K)
        assert spans[0][0] == 0 and spans[-1][1] == m
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        # matches the kernel's per-CTA split, CTA q = (g*K + k)*C + rank
        ctas = [(q * m // (world * K * C), (q + 1) * m // (world * K * C)) for q in range(world * K * C)]
        for g, (lo, hi) in enumerate(spans):
            mine = ctas[g * K * C:(g + 1) * K * C]
            assert mine[0][0] == lo and mine[-1][1] == hi
