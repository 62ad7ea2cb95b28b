"""Where the whole am_solve call goes for a small scenario (circ16j): wall time vs device loop,
and a cProfile of repeated calls."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve, named  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "circ16j"
spec = named(name)
cache = FactorCache()
cfg = SolverConfig()
for _ in range(5):
    am_solve(spec, cfg, cache=cache)
walls, loops = [], []
for _ in range(20):
    t = time.perf_counter()
    r = am_solve(spec, cfg, cache=cache)
    walls.append(time.perf_counter() - t)
    loops.append(r.timings["loop_s"])
print(f"{name}: whole call {min(walls) * 1e3:.3f} ms (median {sorted(walls)[10] * 1e3:.3f}), "
      f"device loop {min(loops) * 1e3:.3f} ms", flush=True)
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    am_solve(spec, cfg, cache=cache)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
