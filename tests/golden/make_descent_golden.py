"""Golden ``descent_slack`` vectors from the real reference (run in the build container).

    python tests/golden/make_descent_golden.py

Writes ``descent_head_on.npz`` (test_solver.py:474-478's instance: head-on swap,
m = 30, max_iters = 40) and ``descent_rand4.npz`` (acceptance C10's first seed,
test_acceptance.py:254-275: generate_random(4, (8,8,3), 0.4, 1000, m = 50),
max_iters = 15, one rho stage, tol 1e-6).
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference  # noqa: E402


def main():
    st = import_reference()
    from swarmtraj.problem import AgentGeometry, BoundaryState, ProblemSpec, generate_random

    def spec_from_lines(lines, radius=0.4, num_samples=20, degree=6, duration=2.0):
        # the reference test helper (test_solver.py:36-47)
        return ProblemSpec(start=tuple(BoundaryState.at_rest(a) for a, _ in lines),
                           goal=tuple(BoundaryState.at_rest(b) for _, b in lines),
                           geometry=AgentGeometry.sphere_from_radius(radius), obstacles=(),
                           num_samples=num_samples, degree=degree, duration=duration)
    from swarmtraj.solver import SolverConfig, am_solve
    cases = {
        "descent_head_on": (spec_from_lines([((-4.0, 0.0, 1.0), (4.0, 0.0, 1.0)),
                                             ((4.0, 0.0, 1.0), (-4.0, 0.0, 1.0))], num_samples=30),
                            dict(max_iters=40)),
        "descent_rand4": (generate_random(4, (8.0, 8.0, 3.0), 0.4, seed=1000, num_samples=50),
                          dict(max_iters=15, rho_stages=1, rho_initial=1.0, tolerance=1e-6)),
    }
    for name, (spec, kw) in cases.items():
        rep = am_solve(spec, SolverConfig(track_descent=True, **kw))
        np.savez_compressed(os.path.join(HERE, name + ".npz"),
                            spec_json=json.dumps(st.spec_to_dict(spec)), config_json=json.dumps(kw),
                            descent_slack=np.array(rep.diagnostics["descent_slack"]),
                            iterations=rep.iterations, coefficients=rep.coefficients)
        print(name, rep.iterations, len(rep.diagnostics["descent_slack"]),
              max(rep.diagnostics["descent_slack"]), min(rep.diagnostics["descent_slack"]))


if __name__ == "__main__":
    main()
