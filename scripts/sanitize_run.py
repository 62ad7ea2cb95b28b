"""Small solves for compute-sanitizer: circ16j (16-CTA cluster, DSMEM exchanges), a rand32 batch
(2-CTA clusters, L2 slabs, cluster reuse), sph64j (multi-cluster grid barrier) and rand128_s0
(large-fleet kernel: TMA row streams, block publish/acquire).  Few iterations each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve, am_solve_batch, generate_random, named  # noqa

cache = FactorCache()
which = sys.argv[1:] or ["circ16j", "batch", "sph64j", "rand128_s0"]
for w in which:
    if w == "batch":
        specs = [generate_random(32, (8.0, 8.0, 3.0), 0.4, s) for s in range(160)]
        r = am_solve_batch(specs, SolverConfig(max_iters=8), cache=cache, with_metrics=False)[0]
    else:
        r = am_solve(named(w), SolverConfig(max_iters=8), cache=cache)
    print(w, r.iterations, r.residual_max_abs, flush=True)
