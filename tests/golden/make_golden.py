"""Generate golden fixtures by running the REAL reference (``swarmtraj``).

Run in the build container, where ``/root/reference`` exists:

    python tests/golden/make_golden.py [--only NAME ...]

Each fixture ``<name>.npz`` holds the scenario (reference JSON schema), the
solver config, and the reference's outputs: coefficients (3,n,nv), the three
histories, iterations, converged, collision verdict, and -- so tests can
scale their tolerance -- the reference's own self-noise envelope: the final
normwise coefficient change when every KKT solve result is multiplied by
(1 + 1e-15).  Small keep_state fixtures also store
the final alpha/beta/d/lambda.  The reference is imported from a writable
copy of its sources; it is run with OPENBLAS_NUM_THREADS=1.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import shutil
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "8" if "--big" in sys.argv else "1")
import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
COPY = "/tmp/graft_ref_src"


def import_reference():
    if not os.path.exists(os.path.join(COPY, "swarmtraj")):
        shutil.copytree(REF_SRC, COPY, dirs_exist_ok=True)
    sys.path.insert(0, COPY)
    import swarmtraj
    return swarmtraj


def scenarios(st):
    P = st.problem
    AG, BS, OB, PS = st.AgentGeometry, st.BoundaryState, st.Obstacle, st.ProblemSpec

    def lines(pairs, radius=0.4, num_samples=20, degree=6, duration=2.0, obstacles=()):
        return PS(start=tuple(BS.at_rest(a) for a, _ in pairs), goal=tuple(BS.at_rest(b) for _, b in pairs),
                  geometry=AG.sphere_from_radius(radius), obstacles=tuple(obstacles),
                  num_samples=num_samples, degree=degree, duration=duration)

    def head_on(**kw):
        return lines([((-4.0, 0.0, 1.0), (4.0, 0.0, 1.0)), ((4.0, 0.0, 1.0), (-4.0, 0.0, 1.0))], **kw)

    def jit(spec, amp=0.05, seed=0):
        rng = np.random.default_rng(seed)
        s = [tuple(np.asarray(x.position) + rng.uniform(-amp, amp, 3)) for x in spec.start]
        g = [tuple(np.asarray(x.position) + rng.uniform(-amp, amp, 3)) for x in spec.goal]
        return dataclasses.replace(spec, start=tuple(BS.at_rest(p) for p in s), goal=tuple(BS.at_rest(p) for p in g))

    def circle(n, amp):
        import math
        st_, gl = [], []
        for i in range(n):
            th = 2 * math.pi * i / n
            s = (4 * math.cos(th), 4 * math.sin(th), 1.5 + 0.5 * (1 if i % 2 == 0 else -1))
            st_.append(BS.at_rest(s))
            gl.append(BS.at_rest((-s[0], -s[1], 3.0 - s[2])))
        spec = PS(start=tuple(st_), goal=tuple(gl), geometry=AG.sphere_from_radius(0.4))
        return jit(spec, amp) if amp else spec

    def sphere(n, amp):
        import math
        ga = math.pi * (3 - math.sqrt(5))
        st_, gl = [], []
        for i in range(n):
            z = 1 - 2 * (i + 0.5) / n
            r = math.sqrt(1 - z * z)
            s = (4 * r * math.cos(ga * i), 4 * r * math.sin(ga * i), 4 + 4 * z)
            st_.append(BS.at_rest(s))
            gl.append(BS.at_rest((-s[0], -s[1], 8 - s[2])))
        spec = PS(start=tuple(st_), goal=tuple(gl), geometry=AG.sphere_from_radius(0.4))
        return jit(spec, amp) if amp else spec

    cfg = st.SolverConfig
    derivs = PS(
        start=(BS(position=(-4, 0, 1), velocity=(1.0, 0, 0), acceleration=(0, 0, 0)),
               BS(position=(4, 0.6, 1), velocity=(-1.0, 0, 0), acceleration=(0, 0, 0))),
        goal=(BS(position=(4, 0, 1), velocity=(1.0, 0, 0), acceleration=(0, 0, 0)),
              BS(position=(-4, 0.6, 1), velocity=(-1.0, 0, 0), acceleration=(0, 0, 0))),
        geometry=AG.sphere_from_radius(0.4), num_samples=60, degree=10, duration=8.0)
    hall = P.generate_hallway(4, 10.0, 3.0, 0.3)
    out = {
        # name: (spec, config kwargs, keep_state)
        "head_on_m40": (head_on(num_samples=40), {}, False),
        "head_on_m60_state": (head_on(num_samples=60, degree=10, duration=10.0), {}, True),
        "head_on_m40_2iters": (head_on(num_samples=40), {"max_iters": 2}, False),
        "single_agent": (lines([((0, 0, 0), (1, 0, 0))], num_samples=30, degree=10), {}, False),
        "single_agent_obstacle": (lines([((-4, 0, 1), (4, 0, 1))], radius=0.4,
                                        obstacles=[OB(center=(0.0, 0.0, 1.0), radius=0.6)],
                                        num_samples=60, degree=10, duration=6.0), {}, False),
        "boundary_derivatives": (derivs, {}, False),
        "rand3_s0": (P.generate_random(3, (8, 8, 3), 0.4, 0), {}, False),
        "rand5_s1": (P.generate_random(5, (8, 8, 3), 0.4, 1), {}, False),
        "rand8_s0": (P.generate_random(8, (8, 8, 3), 0.4, 0), {}, False),
        "rand8_s1": (P.generate_random(8, (8, 8, 3), 0.4, 1), {}, False),
        "rand8_s2_sched": (P.generate_random(8, (8, 8, 3), 0.4, 2),
                           {"rho_initial": 2.0, "rho_growth": 3.0, "rho_stages": 4, "max_iters": 40,
                            "tolerance": 5e-3}, False),
        "rand20_s0": (P.generate_random(20, (8, 8, 3), 0.4, 0), {}, False),
        "circ16j": (circle(16, 0.05), {}, False),
        "circ16_prefix": (circle(16, 0.0), {"max_iters": 5}, False),
        "sph16j": (sphere(16, 0.05), {}, False),
        "rand32_s0": (P.generate_random(32, (8, 8, 3), 0.4, 0), {}, False),
        "rand32_s1": (P.generate_random(32, (8, 8, 3), 0.4, 1), {}, False),
        "obs8": (P.generate_random_with_obstacles(8, (8, 8, 3), 0.4, 4, 0.5, 1), {}, False),
        "hallway4j": (jit(hall), {}, False),
        # the reference CLI/service default corridor (cli.py:80-83): 16 agents, 22 wall obstacles,
        # symmetry broken like the swaps (the exact corridor is chaotic: envelope 0.6)
        "hall16j": (jit(P.generate_hallway(16, 20.0, 4.0, 0.4)), {}, False),
        "square4_monomial": (dataclasses.replace(P.generate_square(4, 8.0, 0.4, num_samples=50),
                                                 basis_kind=st.BasisKind.MONOMIAL, degree=6), {}, False),
        "rand48_s0": (P.generate_random(48, (10, 10, 4), 0.4, 0), {}, False),
        "sph64j": (sphere(64, 0.05), {}, False),
        # chaotic (symmetric) instances: short prefixes pin the arithmetic, full runs pin verdicts only
        "head_on_m60_state_prefix": (head_on(num_samples=60, degree=10, duration=10.0), {"max_iters": 6}, True),
        "single_agent_obstacle_prefix": (lines([((-4, 0, 1), (4, 0, 1))], radius=0.4,
                                               obstacles=[OB(center=(0.0, 0.0, 1.0), radius=0.6)],
                                               num_samples=60, degree=10, duration=6.0), {"max_iters": 6}, False),
        "square4_monomial_prefix": (dataclasses.replace(P.generate_square(4, 8.0, 0.4, num_samples=50),
                                                        basis_kind=st.BasisKind.MONOMIAL, degree=6),
                                    {"max_iters": 6}, False),
        "obs8_state": (P.generate_random_with_obstacles(8, (8, 8, 3), 0.4, 4, 0.5, 1), {}, True),
        # large fleets (slow on the reference: minutes); BASELINE config 5 and an NB=4 case
        "rand128_s0": (P.generate_random(128, (20, 20, 6), 0.4, 0), {}, False),
        "rand256_s0": (P.generate_random(256, (20, 20, 6), 0.4, 0), {}, False),
    }
    return out


def run(st, spec, kwargs, keep, perturb=False):
    from swarmtraj import kkt_cache
    orig = kkt_cache.KktFactor.solve_with_multipliers
    if perturb:
        def noisy(self, b, e):
            c, nu = orig(self, b, e)
            return c * (1.0 + 1e-15), nu
        kkt_cache.KktFactor.solve_with_multipliers = noisy
    try:
        return st.am_solve(spec, st.SolverConfig(keep_state=keep, **kwargs), cache=st.FactorCache())
    finally:
        kkt_cache.KktFactor.solve_with_multipliers = orig


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--big", action="store_true", help="large fleets with 8 BLAS threads")
    args = ap.parse_args()
    st = import_reference()
    for name, (spec, kwargs, keep) in scenarios(st).items():
        if args.only and name not in args.only:
            continue
        if not args.only and not args.big and len(spec.start) > 64:
            continue  # large fleets take minutes on the reference: regenerate with --big
        t0 = time.time()
        rep = run(st, spec, kwargs, keep)
        noisy = run(st, spec, kwargs, False, perturb=True)
        c = rep.coefficients
        env = float(np.linalg.norm(noisy.coefficients - c) / max(np.linalg.norm(c), 1e-300))
        data = {
            "spec_json": json.dumps(st.spec_to_dict(spec)),
            "config_json": json.dumps(kwargs),
            "coefficients": c,
            "trajectories_first_last": rep.trajectories[:, [0, -1], :],
            "iterations": rep.iterations,
            "converged": rep.converged,
            "residual_norm_history": np.array(rep.residual_norm_history),
            "residual_max_history": np.array(rep.residual_max_history),
            "boundary_max_history": np.array(rep.boundary_max_history),
            "min_normalized_distance": np.nan if rep.metrics["min_normalized_distance"] is None
            else rep.metrics["min_normalized_distance"],
            "num_collision_violations": rep.metrics["num_collision_violations"],
            "mean_arc_length": rep.metrics["mean_arc_length"],
            "mean_smoothness": rep.metrics["mean_smoothness"],
            "envelope": env,
            "noisy_iterations": noisy.iterations,
        }
        if keep:
            s = rep.diagnostics["final_state"]
            data.update(alpha=s.pair_vars.alpha, beta=s.pair_vars.beta, d=s.pair_vars.d,
                        lam=np.stack([s.multipliers.lambda_x, s.multipliers.lambda_y, s.multipliers.lambda_z]))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **data)
        print(f"{name:24s} n={len(spec.start):3d} it={rep.iterations:3d} conv={rep.converged} env={env:.1e} "
              f"noisy_it={noisy.iterations} ({time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
