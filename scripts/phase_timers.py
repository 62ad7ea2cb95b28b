"""Per-phase cycles per AM iteration (SWARM_PHASE_TIMERS=1, CTA 0 of scenario 0) for named scenarios
and the C8 obstacle family; the latency breakdown of small single solves."""
import os
import sys

os.environ.setdefault("SWARM_PHASE_TIMERS", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_04240_b200 import SolverConfig, am_solve, generate_random_with_obstacles, named  # noqa: E402

for arg in sys.argv[1:]:
    name, _, C = arg.partition(":")
    if name.startswith("obs"):
        spec = generate_random_with_obstacles(8, (8.0, 8.0, 3.0), 0.4, int(name[3:]), 0.5, seed=1)
        cfg = SolverConfig(max_iters=60, tolerance=1e-12, cluster_size=int(C or 0))
    else:
        spec, cfg = named(name), SolverConfig(cluster_size=int(C or 0))
    r = am_solve(spec, cfg)
    sys.stderr.flush()
    print(f"{arg}: {r.iterations} it, loop {r.timings['loop_s'] * 1e3:.3f} ms, "
          f"{r.timings['loop_s'] / r.iterations * 1e6:.2f} us/iter", flush=True)
