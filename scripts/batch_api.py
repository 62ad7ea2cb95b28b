"""Whole-call throughput of am_solve_batch (validation, packing, device loop, reports with the
batched device collision verdict) for 1024 rand32 scenarios."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_04240_b200 import FactorCache, am_solve_batch, generate_random  # noqa: E402

specs = [generate_random(32, (8, 8, 3), 0.4, s) for s in range(1024)]
cache = FactorCache()
am_solve_batch(specs, cache=cache)
for with_metrics in (False, True):
    t = time.perf_counter()
    reps = am_solve_batch(specs, cache=cache, with_metrics=with_metrics)
    wall = time.perf_counter() - t
    print(f"am_solve_batch(1024 rand32, with_metrics={with_metrics}): {wall * 1e3:.1f} ms -> "
          f"{1024 / wall:.0f} solves/s (device loop {reps[0].timings['loop_s'] * 1e3:.1f} ms)", flush=True)

if len(sys.argv) > 1:
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    am_solve_batch(specs, cache=cache, with_metrics=True)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
