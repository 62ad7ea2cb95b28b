"""Parity of the batched config-4 path (BASELINE configs[3]) -- the path behind the bench headline.

The bench solves seeds 0..1023 of ``generate_random(32, (8,8,3), 0.4, seed)`` in one
launch: 2-CTA clusters, multipliers in L2 slabs with on-chip tails, the n = 32
full-block pair loop, and clusters pulling scenarios from the atomic dispenser (each
cluster solves ~14 scenarios in sequence).  These tests run exactly that launch and
compare scenarios at early and late batch positions (late ones land on reused
clusters) against golden vectors produced by the real reference
(``tests/golden/make_batch_golden.py``, reference bench.py:101 per-scenario call),
and against a batch-of-one solve with the same cluster shape bit for bit.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel_err

BATCH = 1024


def _batch_golden():
    z = np.load(os.path.join(GOLDEN, "batch_rand32.npz"))
    return {k: z[k] for k in z.files}


def test_batch_golden_covers_late_positions():
    g = _batch_golden()
    assert len(g["seeds"]) >= 16
    assert g["seeds"].max() >= 1000 and g["seeds"].min() < 10
    assert np.all(g["converged"])


def test_oracle_matches_batch_golden_subset():
    """The CPU oracle agrees with the reference on two of the batch seeds (oracle pinning)."""
    from oracle import am_oracle
    from paper_2011_04240_b200 import generate_random
    g = _batch_golden()
    for i in (0, len(g["seeds"]) - 1):
        spec = generate_random(32, (8.0, 8.0, 3.0), 0.4, int(g["seeds"][i]))
        ora = am_oracle.solve(spec)
        assert ora["iterations"] == int(g["iterations"][i])
        assert rel_err(ora["coefficients"], g["coefficients"][i]) <= max(1e-9, 10 * g["envelope"][i])


@pytest.fixture(scope="module")
def bench_batch(cuda_ok):
    from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve_batch, generate_random
    specs = [generate_random(32, (8.0, 8.0, 3.0), 0.4, s) for s in range(BATCH)]
    cache = FactorCache()
    reps = am_solve_batch(specs, SolverConfig(), cache=cache)
    return specs, reps, cache


@pytest.mark.gpu
def test_bench_launch_layout_is_the_measured_one(cuda_ok, bench_batch):
    from paper_2011_04240_b200 import FactorCache, SolverConfig, engine, kkt, poly
    specs, _, _ = bench_batch
    basis = poly.for_spec(specs[0])
    cfg = SolverConfig()
    plan = engine._plan_for(FactorCache(), kkt.fingerprint(basis, 32, 0), basis, cfg.schedule(), 32, 0, 0)
    lc = plan.query_launch(BATCH)
    assert lc["cluster"] == 2 and lc["lambda_in_smem"] == 0
    assert lc["clusters"] < BATCH // 4  # every cluster solves several scenarios in sequence


@pytest.mark.gpu
def test_batch_positions_match_reference_golden(cuda_ok, bench_batch):
    _, reps, _ = bench_batch
    g = _batch_golden()
    for i, seed in enumerate(g["seeds"]):
        rep = reps[int(seed)]
        it = int(g["iterations"][i])
        tol = max(1e-9, 10 * float(g["envelope"][i]))
        assert rep.iterations == it, f"seed {seed}: {rep.iterations} vs {it} iterations"
        assert rep.converged == bool(g["converged"][i])
        err = rel_err(rep.coefficients, g["coefficients"][i])
        assert err <= tol, f"seed {seed}: coefficients off by {err:.3e} (tol {tol:.1e})"
        np.testing.assert_allclose(rep.residual_norm_history, g["residual_norm_history"][i, :it], rtol=1e-8,
                                   atol=1e-13)
        np.testing.assert_allclose(rep.residual_max_history, g["residual_max_history"][i, :it], rtol=1e-8,
                                   atol=1e-13)
        np.testing.assert_allclose(rep.boundary_max_history, g["boundary_max_history"][i, :it], atol=1e-9)
        assert rep.metrics["num_collision_violations"] == int(g["num_collision_violations"][i])
        assert rep.metrics["min_normalized_distance"] == pytest.approx(float(g["min_normalized_distance"][i]),
                                                                       rel=1e-7)


@pytest.mark.gpu
@pytest.mark.parametrize("name,pos", [("rand32_s0", 0), ("rand32_s1", 1)])
def test_fixture_scenarios_at_reused_cluster_positions(cuda_ok, name, pos):
    """rand32_s0/s1 planted early and late in a 300-scenario batch: same answer at every position."""
    from conftest import coeff_tol
    from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve_batch, generate_random
    spec, _, ref = load_golden(name)
    specs = [generate_random(32, (8.0, 8.0, 3.0), 0.4, 2000 + s) for s in range(300)]
    slots = (pos, 150, 299)
    for s in slots:
        specs[s] = spec
    reps = am_solve_batch(specs, SolverConfig(), cache=FactorCache(), with_metrics=False)
    for s in slots:
        assert reps[s].iterations == int(ref["iterations"])
        assert rel_err(reps[s].coefficients, ref["coefficients"]) <= coeff_tol(ref)
        np.testing.assert_array_equal(reps[s].coefficients, reps[slots[0]].coefficients)


@pytest.mark.gpu
def test_late_batch_entries_bitwise_equal_batch_of_one(cuda_ok, bench_batch):
    """Cluster reuse leaves no state behind: the last scenarios equal a batch-of-one C = 2 solve bit for bit."""
    from paper_2011_04240_b200 import SolverConfig, am_solve_batch
    specs, reps, cache = bench_batch
    for idx in (BATCH - 1, BATCH - 2, 777):
        one = am_solve_batch([specs[idx]], SolverConfig(cluster_size=2), cache=cache, with_metrics=False)[0]
        assert one.iterations == reps[idx].iterations
        np.testing.assert_array_equal(one.coefficients, reps[idx].coefficients)
        np.testing.assert_array_equal(one.residual_max_history, reps[idx].residual_max_history)
