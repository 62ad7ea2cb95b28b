"""FP32 mode vs the reference fixtures: coefficient error, iterations, residual, clearance."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

from conftest import load_golden, rel_err  # noqa: E402
from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve  # noqa: E402

names = sys.argv[1:] or ["rand8_s0", "rand20_s0", "circ16j", "rand32_s0", "rand32_s1", "sph64j", "obs8", "rand256_s0"]
for name in names:
    spec, cfg, ref = load_golden(name)
    r64 = am_solve(spec, SolverConfig(**cfg), cache=FactorCache())
    r32 = am_solve(spec, SolverConfig(**cfg, fp32=True), cache=FactorCache())
    k = min(len(r32.residual_max_history), len(ref["residual_max_history"]))
    hist = np.max(np.abs(np.array(r32.residual_max_history[:k]) / ref["residual_max_history"][:k] - 1))
    md = r32.metrics["min_normalized_distance"]
    print(f"{name:12s} it {r32.iterations:3d}/{int(ref['iterations']):3d} conv {r32.converged} "
          f"c_err {rel_err(r32.coefficients, ref['coefficients']):.2e} (fp64 {rel_err(r64.coefficients, ref['coefficients']):.1e}) "
          f"res {r32.residual_norm / float(ref['residual_norm_history'][-1]) - 1:+.1e} "
          f"maxhist {hist:.1e} clr {md - float(ref['min_normalized_distance']) if md is not None else 0:+.1e} "
          f"loop {r32.timings['loop_s'] * 1e3:.3f} ms vs {r64.timings['loop_s'] * 1e3:.3f} ms", flush=True)
