"""Run a named scenario twice (warm-up + measured) -- the target for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_04240_b200 import SolverConfig, am_solve, am_solve_batch, named, generate_random
name = sys.argv[1] if len(sys.argv) > 1 else "rand32_s0"
C = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if name.startswith("batch"):
    B = int(name[5:])
    specs = [generate_random(32, (8, 8, 3), 0.4, s) for s in range(B)]
    for _ in range(2):
        r = am_solve_batch(specs, SolverConfig(cluster_size=C), with_metrics=False)
    print(name, r[0].timings["loop_s"] * 1e3, "ms")
else:
    for _ in range(2):
        r = am_solve(named(name), SolverConfig(cluster_size=C))
    print(name, r.iterations, r.timings["loop_s"] * 1e3, "ms")
