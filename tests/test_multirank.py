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
