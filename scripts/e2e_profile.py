"""cProfile of warm single am_solve calls (host overhead around the device loop)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve, scenarios  # noqa: E402

for name in sys.argv[1:] or ["rand32_s0", "sph64j"]:
    spec = scenarios.named(name)
    cache = FactorCache()
    cfg = SolverConfig()
    for _ in range(3):
        rep = am_solve(spec, cfg, cache=cache)
    t = time.perf_counter()
    for _ in range(10):
        rep = am_solve(spec, cfg, cache=cache)
    wall = (time.perf_counter() - t) / 10
    print(f"== {name}: wall {wall * 1e3:.3f} ms/solve, loop {rep.timings['loop_s'] * 1e3:.3f} ms, "
          f"timings { {k: round(v * 1e3, 3) for k, v in rep.timings.items() if k.endswith('_s')} }")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(10):
        am_solve(spec, cfg, cache=cache)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)
