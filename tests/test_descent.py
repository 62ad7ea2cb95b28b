"""``track_descent`` diagnostic (reference solver.py:413-421, augmented_cost 285-303).

Mirrors test_solver.py:474-478 (axis steps never raise the augmented cost,
slack <= 1e-9) and acceptance C10 (test_acceptance.py:254-275, 20 random
4-agent seeds), and compares the slack vectors with the reference's own
(tests/golden/descent_*.npz, made by make_descent_golden.py).
"""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden(name):
    from paper_2011_04240_b200 import spec_from_dict
    z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    return spec_from_dict(json.loads(str(z["spec_json"]))), json.loads(str(z["config_json"])), z


@pytest.mark.parametrize("name", ["descent_head_on", "descent_rand4"])
def test_descent_slack_matches_reference(cuda_ok, name):
    from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve
    spec, cfg, z = _golden(name)
    rep = am_solve(spec, SolverConfig(track_descent=True, **cfg), cache=FactorCache())
    slack = np.array(rep.diagnostics["descent_slack"])
    assert rep.iterations == int(z["iterations"])
    assert slack.shape == z["descent_slack"].shape
    # cost differences: rounding of the two costs (~1e-12 of their size) bounds the agreement
    np.testing.assert_allclose(slack, z["descent_slack"], rtol=1e-6, atol=1e-9)
    assert slack.max() <= 1e-9


def test_criterion_10_descent_property(cuda_ok):
    from paper_2011_04240_b200 import SolverConfig, am_solve, generate_random
    config = SolverConfig(max_iters=15, rho_stages=1, rho_initial=1.0, tolerance=1e-6, track_descent=True)
    worst, steps = -np.inf, 0
    for seed in range(20):
        spec = generate_random(4, (8.0, 8.0, 3.0), 0.4, 1000 + seed, num_samples=50)
        rep = am_solve(spec, config)
        slack = rep.diagnostics["descent_slack"]
        steps += len(slack)
        if slack:
            worst = max(worst, max(slack))
    assert steps > 0 and worst <= 1e-9


def test_descent_tracking_does_not_change_the_solve(cuda_ok):
    from paper_2011_04240_b200 import SolverConfig, am_solve, generate_random
    spec = generate_random(6, (8.0, 8.0, 3.0), 0.4, 3)
    a = am_solve(spec, SolverConfig(max_iters=30))
    b = am_solve(spec, SolverConfig(max_iters=30, track_descent=True))
    assert a.iterations == b.iterations
    np.testing.assert_array_equal(a.coefficients, b.coefficients)
    assert len(b.diagnostics["descent_slack"]) == 3 * (b.iterations - 1)
