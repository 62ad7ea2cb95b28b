"""Per-iteration device time of small fleets (n <= 16, with and without obstacles) by cluster size:
the latency cluster-size rule for small scenarios."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve, generate_random, generate_random_with_obstacles  # noqa

cache = FactorCache()
cases = [("rand3", generate_random(3, (8.0, 8.0, 3.0), 0.4, 0)), ("rand5", generate_random(5, (8.0, 8.0, 3.0), 0.4, 1)),
         ("rand8", generate_random(8, (8.0, 8.0, 3.0), 0.4, 0)), ("rand12", generate_random(12, (8.0, 8.0, 3.0), 0.4, 0)),
         ("rand16", generate_random(16, (8.0, 8.0, 3.0), 0.4, 0))]
cases += [(f"obs8x{k}", generate_random_with_obstacles(8, (8.0, 8.0, 3.0), 0.4, k, 0.5, seed=1)) for k in (4, 8, 16, 32)]
for name, spec in cases:
    row = []
    for C in (4, 8, 16):
        best = None
        for _ in range(3):
            r = am_solve(spec, SolverConfig(max_iters=60, tolerance=1e-12, cluster_size=C), cache=cache)
            v = r.timings["loop_s"] / r.iterations * 1e6
            best = v if best is None else min(best, v)
        row.append(f"C={C}: {best:7.3f}")
    print(f"{name:10s} us/iter  " + "  ".join(row), flush=True)
