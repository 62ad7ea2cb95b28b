"""A/B timing of the device loop (SWARM_LIB selects the library build): named single solves
(best of 3 loop_s) and the 1024-scenario rand32 batch, FP64 (and FP32 with --fp32)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_04240_b200 import (FactorCache, SolverConfig, am_solve, am_solve_batch, generate_random,  # noqa
                                   named)

fp32 = "--fp32" in sys.argv
names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["circ16j", "rand32_s0", "sph64j", "rand256_s0",
                                                                 "batch1024"]
cache = FactorCache()
tag = os.path.basename(os.environ.get("SWARM_LIB", "current")) + (" fp32" if fp32 else "")
for nm in names:
    if nm.startswith("batch"):
        B = int(nm[5:])
        specs = [generate_random(32, (8.0, 8.0, 3.0), 0.4, s) for s in range(B)]
        best = None
        for _ in range(3):
            r = am_solve_batch(specs, SolverConfig(fp32=fp32), cache=cache, with_metrics=False)
            t = r[0].timings["loop_s"]
            best = t if best is None else min(best, t)
        print(f"[{tag}] {nm}: {best * 1e3:.3f} ms -> {B / best:.0f} solves/s", flush=True)
    else:
        spec = named(nm)
        best = None
        for _ in range(3):
            r = am_solve(spec, SolverConfig(fp32=fp32), cache=cache)
            t = r.timings["loop_s"]
            best = t if best is None else min(best, t)
        print(f"[{tag}] {nm}: {best * 1e3:.3f} ms ({r.iterations} it)", flush=True)
