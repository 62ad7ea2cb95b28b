"""Golden vectors for the batched config-4 path (BASELINE configs[3]), from the REAL reference.

Run in the build container, where ``/root/reference`` exists:

    python tests/golden/make_batch_golden.py

Writes ``batch_rand32.npz``: for SEEDS (spread over 0..1023), the scenario
``generate_random(32, (8,8,3), 0.4, seed)`` (problem.py:282-315) solved by
``swarmtraj.am_solve`` with the default SolverConfig and a fresh FactorCache,
one process, OPENBLAS_NUM_THREADS=1 -- exactly the per-scenario call the
reference bench makes (bench.py:101).  Stored per seed: coefficients
(3,n,nv), iterations, converged, the three histories (padded to 150 with NaN),
the collision verdict, and the self-noise envelope (final normwise change
under a 1e-15 relative perturbation of every KKT solve).
"""

from __future__ import annotations

import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference, run  # noqa: E402

SEEDS = [2, 3, 7, 64, 127, 200, 255, 333, 400, 511, 600, 700, 800, 900, 1000, 1023]
MAX_IT = 150


def main():
    st = import_reference()
    P = st.problem
    out = {k: [] for k in ("seeds", "coefficients", "iterations", "converged", "residual_norm_history",
                           "residual_max_history", "boundary_max_history", "min_normalized_distance",
                           "num_collision_violations", "envelope")}
    for seed in SEEDS:
        t0 = time.time()
        spec = P.generate_random(32, (8, 8, 3), 0.4, seed)
        rep = run(st, spec, {}, False)
        noisy = run(st, spec, {}, False, perturb=True)
        c = rep.coefficients
        env = float(np.linalg.norm(noisy.coefficients - c) / np.linalg.norm(c))

        def pad(h):
            a = np.full(MAX_IT, np.nan)
            a[: len(h)] = h
            return a

        out["seeds"].append(seed)
        out["coefficients"].append(c)
        out["iterations"].append(rep.iterations)
        out["converged"].append(rep.converged)
        out["residual_norm_history"].append(pad(rep.residual_norm_history))
        out["residual_max_history"].append(pad(rep.residual_max_history))
        out["boundary_max_history"].append(pad(rep.boundary_max_history))
        md = rep.metrics["min_normalized_distance"]
        out["min_normalized_distance"].append(np.nan if md is None else md)
        out["num_collision_violations"].append(rep.metrics["num_collision_violations"])
        out["envelope"].append(env)
        print(f"seed {seed:5d} it={rep.iterations:3d} conv={rep.converged} env={env:.1e} "
              f"({time.time() - t0:.1f}s)", flush=True)
    np.savez_compressed(os.path.join(HERE, "batch_rand32.npz"), **{k: np.asarray(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
