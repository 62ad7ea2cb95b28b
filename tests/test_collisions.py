"""Post-solve collision verdict (reference validation.py:39-93, check_collisions).

CPU: the scalar oracle restatement pins the host (numpy) version exactly.
GPU (``-m gpu``): ``st_check_collisions`` equals the scalar oracle bit for bit --
minimum, violation count, and every ((kind, i, j), sample, value) entry in the
reference's order -- plus empty, obstacle-only and overflowing-capacity cases.
"""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import am_oracle


def _case(n, m, n_obs, seed, spread=2.0):
    from paper_2011_04240_b200.spec import AgentGeometry, Obstacle
    rng = np.random.default_rng(seed)
    traj = rng.uniform(-spread, spread, (n, m, 3))
    geom = AgentGeometry(0.8, 0.8 if seed % 2 else 1.1)
    obstacles = tuple(Obstacle(tuple(rng.uniform(-spread, spread, 3).tolist()), float(rng.uniform(0.1, 0.6)))
                      for _ in range(n_obs))
    return traj, geom, obstacles


def _oracle(traj, geom, obstacles):
    return am_oracle.check_collisions_scalar(traj, geom.l_xy, geom.l_z,
                                             [(tuple(o.center), o.radius) for o in obstacles])


@pytest.mark.parametrize("n,m,n_obs,seed", [(5, 17, 0, 0), (7, 40, 3, 1), (1, 10, 2, 2), (12, 33, 1, 3)])
def test_host_check_collisions_matches_scalar_oracle(n, m, n_obs, seed):
    from paper_2011_04240_b200 import metrics
    traj, geom, obstacles = _case(n, m, n_obs, seed)
    mn, viol = _oracle(traj, geom, obstacles)
    col = metrics.check_collisions(traj, geom, obstacles)
    assert col.min_normalized_distance == mn
    assert col.violations == viol


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,n_obs,seed", [(5, 17, 0, 0), (7, 40, 3, 1), (1, 10, 2, 2), (12, 33, 1, 3),
                                            (40, 100, 4, 4), (3, 1, 0, 5), (33, 65, 2, 6)])
def test_device_check_collisions_bitwise_vs_scalar_oracle(cuda_ok, n, m, n_obs, seed):
    from paper_2011_04240_b200 import metrics
    traj, geom, obstacles = _case(n, m, n_obs, seed)
    mn, viol = _oracle(traj, geom, obstacles)
    col = metrics.check_collisions_device(traj, geom, obstacles)
    assert col.min_normalized_distance == mn
    assert len(col.violations) == len(viol)
    assert viol or n * m < 50  # the larger cases exercise the entry writer
    assert col.violations == viol  # same order, same bits


@pytest.mark.gpu
def test_device_check_collisions_empty_and_capacity(cuda_ok):
    from paper_2011_04240_b200 import metrics, native
    from paper_2011_04240_b200.spec import AgentGeometry
    g = AgentGeometry(0.8, 0.8)
    single = np.zeros((1, 20, 3))
    col = metrics.check_collisions_device(single, g, ())
    assert math.isinf(col.min_normalized_distance) and col.violations == []
    # every pair collides at every sample: the list outgrows the first capacity and is re-fetched
    traj = np.zeros((30, 100, 3))
    mn, viol = native.check_collisions(traj, 0.8, 0.8, np.zeros((0, 5)), cap=7)
    assert mn == 0.0 and len(viol) == 435 * 100
    assert viol[0] == (("agent", 0, 1), 0, 0.0) and viol[-1] == (("agent", 28, 29), 99, 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["rand256_s0", "rand32_s0", "obs8"])
def test_device_check_collisions_equals_host_on_solutions(cuda_ok, name):
    from paper_2011_04240_b200 import metrics, poly
    spec, _, ref = load_golden(name)
    basis = poly.for_spec(spec)
    traj = np.ascontiguousarray(np.einsum("ank,tk->nta", ref["coefficients"], basis.P))
    host = metrics.check_collisions(traj, spec.geometry, spec.obstacles)
    dev = metrics.check_collisions_device(traj, spec.geometry, spec.obstacles)
    assert dev.min_normalized_distance == host.min_normalized_distance
    assert dev.violations == host.violations
    assert len(dev.violations) == int(ref["num_collision_violations"])


@pytest.mark.gpu
def test_device_batch_equals_per_scenario(cuda_ok):
    from paper_2011_04240_b200 import metrics
    from paper_2011_04240_b200.spec import AgentGeometry, Obstacle
    rng = np.random.default_rng(11)
    B, n, m, n_obs = 6, 9, 37, 2
    trajs = rng.uniform(-0.5, 0.5, (B, n, m, 3))
    specs = []
    for b in range(B):
        geom = AgentGeometry(0.8, 0.6 + 0.1 * b)
        obstacles = tuple(Obstacle(tuple(rng.uniform(-2, 2, 3).tolist()), float(rng.uniform(0.1, 0.5)))
                          for _ in range(n_obs))
        specs.append(type("S", (), {"geometry": geom, "obstacles": obstacles})())
    got = metrics.check_collisions_device_batch(trajs, specs)
    assert sum(len(g.violations) for g in got) > 4096  # the entry list outgrows the first capacity
    for b in range(B):
        mn, viol = _oracle(trajs[b], specs[b].geometry, specs[b].obstacles)
        assert got[b].min_normalized_distance == mn
        assert got[b].violations == viol


@pytest.mark.gpu
def test_batch_reports_carry_the_per_scenario_verdicts(cuda_ok):
    from paper_2011_04240_b200 import am_solve_batch, generate_random, metrics
    specs = [generate_random(8, (8, 8, 3), 0.4, s) for s in range(5)]
    reps = am_solve_batch(specs)
    for spec, rep in zip(specs, reps):
        # one batched device verdict per launch == the host restatement on the same trajectories;
        # arc length / smoothness come from the batched coefficient-difference products (the same
        # definitions, summed in another order)
        want = metrics.final_metrics(spec, rep.trajectories)
        got = rep.metrics
        assert got["min_normalized_distance"] == want["min_normalized_distance"]
        assert got["num_collision_violations"] == want["num_collision_violations"]
        for key in ("arc_length", "smoothness"):
            np.testing.assert_allclose(got[key], want[key], rtol=1e-12)
        for key in ("mean_arc_length", "mean_smoothness"):
            assert got[key] == pytest.approx(want[key], rel=1e-12)
