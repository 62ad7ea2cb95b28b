"""Batch throughput vs cluster size (device loop only)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2011_04240_b200 import SolverConfig, am_solve_batch, generate_random, FactorCache
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
os.environ.setdefault("SWARM_PIPE_CHUNKS", "1")  # one launch: loop_s is the whole batch
specs = [generate_random(32, (8, 8, 3), 0.4, s) for s in range(B)]
cache = FactorCache()
for C in [int(c) for c in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "2", "4", "8"])]:
    try:
        reps = am_solve_batch(specs, SolverConfig(cluster_size=C), cache=cache, with_metrics=False)
        reps = am_solve_batch(specs, SolverConfig(cluster_size=C), cache=cache, with_metrics=False)
    except Exception as e:
        print("C", C, "failed:", e); continue
    loop = reps[0].timings["loop_s"]
    print(f"C={C}: batch {B} loop {loop*1e3:.2f} ms -> {B/loop:.0f} solves/s; iters mean "
          f"{np.mean([r.iterations for r in reps]):.1f}", flush=True)
