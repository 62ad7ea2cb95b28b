"""Solve a fixed set of instances and save every output array (A/B bitwise checks of kernel changes).

usage: [SWARM_LIB=...] python scripts/dump_coeffs.py out.npz
       python scripts/dump_coeffs.py --compare a.npz b.npz
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if k not in b.files or a[k].shape != b[k].shape or not np.array_equal(a[k], b[k])]
    for k in bad:
        if k in b.files and a[k].shape == b[k].shape:
            d = np.max(np.abs(a[k] - b[k])) / max(1e-300, np.max(np.abs(a[k])))
            print(f"DIFF {k}: max rel {d:.3e}")
        else:
            print(f"DIFF {k}: missing/shape")
    print(f"{len(a.files) - len(bad)}/{len(a.files)} arrays bitwise equal")
    sys.exit(1 if bad else 0)

from conftest import load_golden
from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve, am_solve_batch, generate_random

out = {}
cache = FactorCache()
for name in ["circ16j", "rand32_s0", "sph64j", "rand48_s0", "obs8", "hallway4j", "rand8_s1", "single_agent",
             "sph16j", "rand128_s0", "rand256_s0"]:
    spec, cfg, ref = load_golden(name)
    mi = 60 if name in ("rand128_s0", "rand256_s0") else cfg.get("max_iters", 150)
    r = am_solve(spec, SolverConfig(max_iters=mi), cache=cache)
    out[name + "/c"] = np.asarray(r.coefficients)
    out[name + "/it"] = np.array([r.iterations])
    out[name + "/h"] = np.array([r.residual_norm_history, r.residual_max_history, r.boundary_max_history])
specs = [generate_random(32, (8, 8, 3), 0.4, s) for s in range(300)]
reps = am_solve_batch(specs, SolverConfig(), cache=cache, with_metrics=False)
out["batch32/c"] = np.stack([r.coefficients for r in reps])
out["batch32/it"] = np.array([r.iterations for r in reps])
specs = [generate_random(12, (6, 6, 3), 0.4, s) for s in range(100)]
reps = am_solve_batch(specs, SolverConfig(), cache=cache, with_metrics=False)
out["batch12/c"] = np.stack([r.coefficients for r in reps])
np.savez(sys.argv[1], **out)
print("saved", len(out), "arrays")
