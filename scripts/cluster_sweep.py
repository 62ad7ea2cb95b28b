"""Single-solve device loop (best of 3) by cluster size, for named scenarios and the tiny random
family: the data behind choose_launch's latency rule (profiles/cluster_sweep_r2.txt)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve, generate_random, named  # noqa: E402

cache = FactorCache()
sizes = (1, 2, 4, 8, 16)
for nm in sys.argv[1:]:
    if nm.startswith("tiny"):  # tiny<n>_s<seed>: generate_random(n, (8,8,3), 0.4, seed)
        n_s, s_s = nm[4:].split("_s")
        spec = generate_random(int(n_s), (8, 8, 3), 0.4, int(s_s))
    else:
        spec = named(nm)
    row = []
    for C in sizes:
        best = None
        try:
            for _ in range(3):
                r = am_solve(spec, SolverConfig(cluster_size=C), cache=cache)
                t = r.timings["loop_s"] * 1e3
                best = t if best is None else min(best, t)
            row.append(f"C={C}: {best:.3f}")
        except Exception as exc:  # a cluster shape the scenario cannot use
            row.append(f"C={C}: n/a")
    print(f"{nm:10s} it={r.iterations:3d}  " + " | ".join(row), flush=True)
