"""The device report pass (``st_solve_report``) and the pipelined batch entry.

``am_solve_batch`` forms the reports' trajectories, arc length / smoothness and the
collision summary on the device in the solve call (replacing the host work after the
reference's loop: SolveReport.trajectories = c_axis @ P.T, solver.py:133-136, and
_final_metrics, solver.py:497-509 -> validation.py:39-132), and runs large batches as a
pipeline of chunks.  Checked here against the host formulas on the same coefficients, the
scalar collision loop, and the unchunked launch (bitwise).
"""

import numpy as np
import pytest


def _specs(B, n=32, seed0=0, obstacles=0):
    from paper_2011_04240_b200 import generate_random, generate_random_with_obstacles
    if obstacles:
        return [generate_random_with_obstacles(n, (8.0, 8.0, 3.0), 0.4, obstacles, 0.5, seed=seed0 + s)
                for s in range(B)]
    return [generate_random(n, (8, 8, 3), 0.4, seed0 + s) for s in range(B)]


@pytest.mark.gpu
@pytest.mark.parametrize("obstacles", [0, 4])
def test_report_pass_matches_host_formulas(cuda_ok, obstacles):
    from paper_2011_04240_b200 import am_solve_batch, metrics, poly
    specs = _specs(40, n=12 if obstacles else 32, obstacles=obstacles)
    reps = am_solve_batch(specs)
    basis = poly.for_spec(specs[0])
    for spec, r in zip(specs, reps):
        host_traj = np.stack([r.coefficients[a] @ basis.P.T for a in range(3)], axis=-1)
        np.testing.assert_allclose(r.trajectories, host_traj, rtol=1e-13, atol=1e-13)
        q = metrics.trajectory_metrics(host_traj)
        np.testing.assert_allclose(r.metrics["arc_length"], q.arc_length, rtol=1e-12)
        np.testing.assert_allclose(r.metrics["smoothness"], q.smoothness, rtol=1e-12)
        assert r.metrics["mean_arc_length"] == pytest.approx(np.mean(q.arc_length), rel=1e-12)
        # verdict on the report's own trajectories: identical to the scalar loop of the reference
        col = metrics.check_collisions(r.trajectories, spec.geometry, spec.obstacles)
        assert r.metrics["num_collision_violations"] == len(col.violations)
        md = r.metrics["min_normalized_distance"]
        assert (md is None) == np.isinf(col.min_normalized_distance)
        if md is not None:
            assert md == col.min_normalized_distance


@pytest.mark.gpu
def test_pipelined_batch_is_bitwise_the_single_launch(cuda_ok, monkeypatch):
    from paper_2011_04240_b200 import am_solve_batch, engine
    specs = _specs(300)
    monkeypatch.setenv("SWARM_PIPE_CHUNKS", "1")
    one = am_solve_batch(specs)
    monkeypatch.setenv("SWARM_PIPE_CHUNKS", "3")
    three = am_solve_batch(specs)
    monkeypatch.setenv("SWARM_PIPE_CHUNKS", "7")
    seven = am_solve_batch(specs, with_metrics=False)
    b3 = engine._chunk_bounds(300, 3)
    assert b3 == [0, 60, 180, 300]  # first chunk half the others
    assert [r.timings["batch"] for r in three] == [b - a for a, b in zip(b3, b3[1:]) for _ in range(b - a)]
    for a, b, c in zip(one, three, seven):
        assert a.iterations == b.iterations == c.iterations
        assert np.array_equal(a.coefficients, b.coefficients) and np.array_equal(a.coefficients, c.coefficients)
        assert np.array_equal(a.trajectories, b.trajectories) and np.array_equal(a.trajectories, c.trajectories)
        assert a.residual_norm_history == b.residual_norm_history
        assert a.metrics == b.metrics
        assert c.metrics == {}


@pytest.mark.gpu
def test_pipelined_batch_raises_on_a_late_invalid_scenario(cuda_ok, monkeypatch):
    from paper_2011_04240_b200 import InfeasibleProblemError, am_solve_batch
    specs = _specs(300)
    bad = specs[250]
    # two agents at the same start: infeasible (reference problem.py:162-194)
    start = (bad.start[1],) + tuple(bad.start[1:])
    specs[250] = type(bad)(start=start, goal=bad.goal, geometry=bad.geometry, obstacles=bad.obstacles,
                           num_samples=bad.num_samples, degree=bad.degree, duration=bad.duration,
                           basis_kind=bad.basis_kind, seed=bad.seed)
    monkeypatch.setenv("SWARM_PIPE_CHUNKS", "3")
    with pytest.raises(InfeasibleProblemError):
        am_solve_batch(specs)
    # the plan is left usable
    assert am_solve_batch(specs[:5])[0].converged


def test_pipeline_chunking_rule(monkeypatch):
    from paper_2011_04240_b200 import engine
    monkeypatch.delenv("SWARM_PIPE_CHUNKS", raising=False)
    assert engine._pipeline_chunks(1) == 1 and engine._pipeline_chunks(255) == 1
    assert engine._pipeline_chunks(1024) == 4
    monkeypatch.setenv("SWARM_PIPE_CHUNKS", "5")
    assert engine._pipeline_chunks(3) == 3 and engine._pipeline_chunks(100) == 5
    # chunk bounds: first chunk half the others, every chunk within one report launch
    for B, K in ((1024, 3), (7, 7), (300, 4), (200000, 3)):
        b = engine._chunk_bounds(B, K)
        sizes = [y - x for x, y in zip(b, b[1:])]
        assert b[0] == 0 and b[-1] == B and min(sizes) >= 1 and max(sizes) <= 65535 and len(b) - 1 >= K


@pytest.mark.gpu
def test_pooled_trajectory_buffers_are_never_shared_with_live_reports(cuda_ok):
    """Report trajectories live in pooled page-locked buffers: a buffer goes back to the pool only
    when every array over it is gone, so later calls never overwrite reports still held."""
    import gc

    from paper_2011_04240_b200 import am_solve_batch
    a = am_solve_batch(_specs(8))
    keep = [r.trajectories.copy() for r in a]
    for seed in (100, 200, 300):
        am_solve_batch(_specs(8, seed0=seed))  # dropped at once: their buffer returns to the pool
        gc.collect()
    b = am_solve_batch(_specs(8, seed0=400))
    for r, t in zip(a, keep):
        assert np.array_equal(r.trajectories, t)
    assert not any(np.shares_memory(x.trajectories, y.trajectories) for x in a for y in b)


@pytest.mark.gpu
def test_begin_end_equals_one_call_and_guards_the_plan(cuda_ok):
    """st_solve_report_begin / st_solve_end: the same outputs as st_solve_report, page-locked
    outputs, other host-pointer calls on the plan refused while a solve is pending, and a
    pending solve dropped without end() does not leave the plan refusing calls."""
    import gc

    from paper_2011_04240_b200 import SolverConfig, engine, kkt, poly
    specs = _specs(20, n=16, obstacles=2)
    basis = poly.for_spec(specs[0])
    cfg = SolverConfig()
    sch = cfg.schedule()
    cache = kkt.FactorCache()
    plan = engine._plan_for(cache, kkt.fingerprint(basis, 16, 2), basis, sch, 16, 2, 0)
    _, _, c0, beq, geom, cg, co = engine._prep_chunk(specs, basis, 2)
    args = (c0, beq, geom, sch.switch_every, cfg.max_iters, cfg.tolerance, cg, co)
    one = plan.solve_report(*args)
    pend = plan.solve_report_begin(*args)
    with pytest.raises(ValueError, match="not ended"):
        plan.solve_report(*args)
    two = pend.end()
    for k in ("c", "hist", "iters", "traj", "arc", "smooth", "min_dist", "n_viol"):
        assert np.array_equal(one[k], two[k]), k
    assert np.array_equal(one["converged"], two["converged"])
    with pytest.raises(RuntimeError):
        pend.end()
    pend = plan.solve_report_begin(*args)
    del pend
    gc.collect()
    three = plan.solve_report(*args)  # the finalizer ended the dropped solve
    assert np.array_equal(one["c"], three["c"])


@pytest.mark.gpu
def test_pipelined_obstacle_batch_is_bitwise_the_single_launch(cuda_ok, monkeypatch):
    """The begin/end pipeline with obstacle rows (collision inputs staged per chunk) and FP32."""
    from paper_2011_04240_b200 import SolverConfig, am_solve_batch
    specs = _specs(260, n=8, obstacles=3)
    for cfg in (SolverConfig(), SolverConfig(fp32=True)):
        monkeypatch.setenv("SWARM_PIPE_CHUNKS", "1")
        one = am_solve_batch(specs, cfg)
        monkeypatch.setenv("SWARM_PIPE_CHUNKS", "4")
        four = am_solve_batch(specs, cfg)
        for a, b in zip(one, four):
            assert a.iterations == b.iterations and a.converged == b.converged
            assert np.array_equal(a.coefficients, b.coefficients)
            assert np.array_equal(a.trajectories, b.trajectories)
            assert a.metrics == b.metrics
