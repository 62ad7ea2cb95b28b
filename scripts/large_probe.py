"""Large-fleet kernel vs the reference fixtures (and vs the multi-cluster path): errors and times.
Env: SWARM_LARGE=2 forces the large kernel for any n; SWARM_VIRTUAL_GROUPS=g emulates g GPUs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import coeff_tol, load_golden, rel_err  # noqa: E402
from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve  # noqa: E402

fp32 = "--fp32" in sys.argv
names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["rand128_s0", "rand256_s0"]
for name in names:
    spec, cfg, ref = load_golden(name)
    cache = FactorCache()
    best = None
    for _ in range(3):
        r = am_solve(spec, SolverConfig(**cfg, fp32=fp32), cache=cache)
        best = r.timings["loop_s"] if best is None else min(best, r.timings["loop_s"])
    err = rel_err(r.coefficients, ref["coefficients"])
    print(f"{name:12s} fp32={fp32} it {r.iterations}/{int(ref['iterations'])} conv {r.converged} err {err:.2e} "
          f"(tol {coeff_tol(ref):.1e}) loop {best * 1e3:.3f} ms  hist0 {r.residual_max_history[:2]} "
          f"ref {list(ref['residual_max_history'][:2])}", flush=True)
