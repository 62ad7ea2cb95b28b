"""Quick device timing probe (not the bench): single solves and a batch."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2011_04240_b200 import SolverConfig, am_solve, am_solve_batch, named, generate_random, FactorCache, kkt, poly, pack
from paper_2011_04240_b200 import engine

cache = FactorCache()
for name in ["circ16j", "rand32_s0", "sph64j"]:
    spec = named(name)
    for hint in (0, 8, 4):
        rep = am_solve(spec, SolverConfig(cluster_size=hint), cache=cache)
        rep = am_solve(spec, SolverConfig(cluster_size=hint), cache=cache)
        print(f"{name} C={hint}: it={rep.iterations} conv={rep.converged} loop={rep.timings['loop_s']*1e3:.3f} ms "
              f"per_it={rep.timings['per_iteration_s']*1e6:.1f} us total={rep.timings['total_s']*1e3:.1f} ms", flush=True)
for B in (148, 1024):
    specs = [generate_random(32, (8, 8, 3), 0.4, s) for s in range(B)]
    reps = am_solve_batch(specs, cache=cache, with_metrics=False)
    reps = am_solve_batch(specs, cache=cache, with_metrics=False)
    its = np.array([r.iterations for r in reps])
    loop = reps[0].timings["loop_s"]
    print(f"batch {B} rand32: loop {loop*1e3:.2f} ms -> {B/loop:.0f} solves/s; iters mean {its.mean():.1f} "
          f"conv {np.mean([r.converged for r in reps]):.3f}", flush=True)
basis = poly.for_spec(named("rand32_s0"))
fp = kkt.fingerprint(basis, 32, 0)
plan = engine._plan_for(cache, fp, basis, SolverConfig().schedule(), 32, 0, 0)
print("launch B=1024:", plan.query_launch(1024), "B=1:", plan.query_launch(1))
