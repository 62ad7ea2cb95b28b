import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_04240_b200 import SolverConfig, am_solve, named, generate_random, FactorCache
name = sys.argv[1] if len(sys.argv) > 1 else "rand256_s0"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 150
C = int(sys.argv[3]) if len(sys.argv) > 3 else 0
spec = named(name)
cache = FactorCache()
t0 = time.time()
r = am_solve(spec, SolverConfig(max_iters=its, cluster_size=C), cache=cache)
t1 = time.time()
r = am_solve(spec, SolverConfig(max_iters=its, cluster_size=C), cache=cache)
print(name, "iters", r.iterations, "conv", r.converged, "loop_ms", round(r.timings["loop_s"] * 1e3, 3),
      "per_iter_ms", round(r.timings["per_iteration_s"] * 1e3, 4), "res", r.residual_max_abs,
      "first_call_s", round(t1 - t0, 2), "metrics_s", round(r.timings["metrics_s"], 3), flush=True)
