"""Whole-call throughput of am_solve_batch (validation, packing, device loop + device report
pass, reports) for 1024 rand32 scenarios, by pipeline chunk count; optional cProfile."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_04240_b200 import FactorCache, am_solve_batch, generate_random  # noqa: E402

specs = [generate_random(32, (8, 8, 3), 0.4, s) for s in range(1024)]
cache = FactorCache()
am_solve_batch(specs, cache=cache)
for chunks in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "3", "4"]):
    os.environ["SWARM_PIPE_CHUNKS"] = chunks
    for with_metrics in (False, True):
        best = 1e9
        reps = None
        for _ in range(3):
            reps = None  # free the previous reports outside the timed region
            t = time.perf_counter()
            reps = am_solve_batch(specs, cache=cache, with_metrics=with_metrics)
            best = min(best, time.perf_counter() - t)
        print(f"am_solve_batch(1024 rand32, with_metrics={with_metrics}, chunks={chunks}): {best * 1e3:.1f} ms -> "
              f"{1024 / best:.0f} solves/s (device loop of one launch {reps[0].timings['loop_s'] * 1e3:.1f} ms)",
              flush=True)

if len(sys.argv) > 2:
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    am_solve_batch(specs, cache=cache, with_metrics=True)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
