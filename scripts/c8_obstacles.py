"""Acceptance C8 on the GPU (reference tests/test_acceptance.py:210-233): per-iteration loop
time vs obstacle count for 8 agents, max_iters 60, tol 1e-12, min over 5 reps; R^2 of a line fit."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve, engine, generate_random_with_obstacles, kkt, poly

counts = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "4,8,16,32".split(","))]
hints = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "0".split(","))]
for hint in hints:
    cache = FactorCache()
    per = []
    for n_obs in counts:
        spec = generate_random_with_obstacles(8, (8.0, 8.0, 3.0), 0.4, n_obs, 0.5, seed=1)
        cfg = SolverConfig(max_iters=60, tolerance=1e-12, cluster_size=hint)
        ts = []
        for _ in range(5):
            r = am_solve(spec, cfg, cache=cache)
            ts.append(r.timings["loop_s"] / r.iterations)
        basis = poly.for_spec(spec)
        plan = engine._plan_for(cache, kkt.fingerprint(basis, 8, n_obs), basis, cfg.schedule(), 8, n_obs, 0)
        lc = plan.query_launch(1, hint)
        per.append(min(ts))
        print(f"hint={hint} n_obs={n_obs:3d} per-iter {min(ts) * 1e6:8.3f} us  (max {max(ts) * 1e6:8.3f})  "
              f"C={lc['cluster']} W={lc['lane_width']} steps={lc['steps_per_task']} smem={lc['lambda_in_smem']}")
    x, y = np.array(counts, float), np.array(per)
    print(f"hint={hint} R^2 = {np.corrcoef(x, y)[0, 1] ** 2:.4f}")
