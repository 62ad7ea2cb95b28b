"""Determinism stress: the same solve must give identical bits regardless of what ran before."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import load_golden, golden_names
from paper_2011_04240_b200 import SolverConfig, FactorCache, am_solve, am_solve_batch, generate_random
target = sys.argv[1] if len(sys.argv) > 1 else "rand48_s0"
spec, cfg, ref = load_golden(target)
base = am_solve(spec, SolverConfig(**cfg), cache=FactorCache())
print("first", base.iterations, base.converged, "ref", int(ref["iterations"]))
bad = 0
for rnd in range(3):
    for nm in golden_names():
        if nm in ("rand256_s0",):
            continue
        s2, c2, _ = load_golden(nm)
        am_solve(s2, SolverConfig(**c2), cache=FactorCache())
        r = am_solve(spec, SolverConfig(**cfg), cache=FactorCache())
        same = r.iterations == base.iterations and np.array_equal(r.coefficients, base.coefficients)
        if not same:
            bad += 1
            print(f"round {rnd} after {nm}: iters {r.iterations} (base {base.iterations}) "
                  f"maxdiff {np.abs(r.coefficients - base.coefficients).max():.3e}", flush=True)
    am_solve_batch([generate_random(32, (8, 8, 3), 0.4, s) for s in range(64)], with_metrics=False)
print("mismatches", bad)
