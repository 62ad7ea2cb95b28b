"""rand256_s0 FP64 loop time alone, after an FP32 large solve, and after the batch kernel (L2 state
left behind by earlier launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve, am_solve_batch, generate_random, named  # noqa

cache = FactorCache()
big = named("rand256_s0")


def t(spec, fp32=False, reps=2):
    best = None
    for _ in range(reps):
        r = am_solve(spec, SolverConfig(fp32=fp32), cache=cache)
        best = r.timings["loop_s"] if best is None else min(best, r.timings["loop_s"])
    return best * 1e3


print("rand256 fp64 alone", round(t(big), 3), flush=True)
print("rand128 fp32", round(t(named("rand128_s0"), True), 3), flush=True)
print("rand256 fp64 after fp32", round(t(big), 3), flush=True)
specs = [generate_random(32, (8.0, 8.0, 3.0), 0.4, s) for s in range(1024)]
am_solve_batch(specs, SolverConfig(), cache=cache, with_metrics=False)
print("rand256 fp64 after batch", round(t(big), 3), flush=True)
print("rand256 fp32", round(t(big, True), 3), flush=True)
print("rand256 fp64 after rand256 fp32", round(t(big), 3), flush=True)
