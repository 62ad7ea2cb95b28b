"""Host-side logic on CPU: problem types, generators, basis, structured KKT algebra,
rho schedule, factor cache census, packing, validation errors, collision metrics and
the C-ABI library's exported symbols.  No GPU needed.
"""

import json
import os
import re
import threading

import numpy as np
import pytest

from conftest import ROOT, golden_names, load_golden
from oracle import am_oracle
from paper_2011_04240_b200 import (AgentGeometry, BoundaryState, FactorCache, InfeasibleProblemError, Obstacle,
                                   ProblemSpec, SolverConfig, build_basis, build_rho_schedule, check_collisions,
                                   circle_swap, generate_hallway, generate_random, generate_random_with_obstacles,
                                   generate_square, kkt, pack, poly, spec_from_dict, spec_to_dict, sphere_swap,
                                   validate)
from paper_2011_04240_b200 import engine


# --- generators reproduce the reference's instances ------------------------------------------

def _same_spec(a, b):
    return json.dumps(spec_to_dict(a), sort_keys=True) == json.dumps(spec_to_dict(b), sort_keys=True)


@pytest.mark.parametrize("name,build", [
    ("rand3_s0", lambda: generate_random(3, (8, 8, 3), 0.4, 0)),
    ("rand5_s1", lambda: generate_random(5, (8, 8, 3), 0.4, 1)),
    ("rand8_s0", lambda: generate_random(8, (8, 8, 3), 0.4, 0)),
    ("rand20_s0", lambda: generate_random(20, (8, 8, 3), 0.4, 0)),
    ("rand32_s0", lambda: generate_random(32, (8, 8, 3), 0.4, 0)),
    ("rand48_s0", lambda: generate_random(48, (10, 10, 4), 0.4, 0)),
    ("obs8", lambda: generate_random_with_obstacles(8, (8, 8, 3), 0.4, 4, 0.5, 1)),
    ("circ16j", lambda: circle_swap(16)),
    ("sph16j", lambda: sphere_swap(16)),
    ("sph64j", lambda: sphere_swap(64)),
])
def test_generators_match_reference_instances(name, build):
    spec, _, _ = load_golden(name)
    assert _same_spec(build(), spec)


def test_square_and_hallway_generators():
    sq = generate_square(8, 8.0, 0.4)
    assert len(sq.start) == 8 and not validate(sq)
    hw = generate_hallway(4, 10.0, 3.0, 0.3)
    assert hw.num_obstacles > 0 and not validate(hw)


def test_json_round_trip():
    for name in ("obs8", "boundary_derivatives", "square4_monomial"):
        spec, _, _ = load_golden(name)
        assert _same_spec(spec_from_dict(json.loads(json.dumps(spec_to_dict(spec)))), spec)


# --- basis -------------------------------------------------------------------------------------

@pytest.mark.parametrize("kind", ["bernstein", "monomial"])
def test_basis_matches_oracle_bitwise(kind):
    b = build_basis(37, 3.3, 7, kind)
    P, Pd, Pdd = am_oracle.basis(37, 3.3, 7, kind)
    for x, y in ((b.P, P), (b.Pdot, Pd), (b.Pddot, Pdd)):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))


def test_bernstein_partition_of_unity_and_derivatives():
    b = build_basis(4001, 2.0, 10)
    np.testing.assert_allclose(b.P.sum(axis=1), 1.0, atol=1e-14)
    c = np.random.default_rng(0).normal(size=11)
    x, v = b.P @ c, b.Pdot @ c
    h = b.samples[1] - b.samples[0]
    fd = (x[2:] - x[:-2]) / (2 * h)
    assert np.max(np.abs(fd - v[1:-1])) <= 1e-4 * np.max(np.abs(v))
    fd2 = (x[2:] - 2 * x[1:-1] + x[:-2]) / h ** 2
    assert np.max(np.abs(fd2 - (b.Pddot @ c)[1:-1])) <= 1e-3 * np.max(np.abs(b.Pddot @ c))


def test_basis_rejects_bad_arguments():
    with pytest.raises(ValueError):
        build_basis(1, 1.0, 6)
    with pytest.raises(ValueError):
        build_basis(10, 0.0, 6)
    with pytest.raises(ValueError):
        build_basis(10, 1.0, 4)


# --- structured KKT algebra (kkt.py) vs a dense KKT solve --------------------------------------

def _spec(n, n_obs, m=15, deg=6):
    rng = np.random.default_rng(n * 10 + n_obs)
    starts = tuple(BoundaryState(position=tuple(rng.uniform(-5, 5, 3)), velocity=tuple(rng.normal(size=3)))
                   for _ in range(n))
    goals = tuple(BoundaryState(position=tuple(rng.uniform(-5, 5, 3)), acceleration=tuple(rng.normal(size=3)))
                  for _ in range(n))
    obs = tuple(Obstacle(center=tuple(rng.uniform(-9, 9, 3)), radius=0.3 + 0.1 * k) for k in range(n_obs))
    return ProblemSpec(start=starts, goal=goals, geometry=AgentGeometry(0.8, 0.6), obstacles=obs, num_samples=m,
                       degree=deg, duration=2.0)


@pytest.mark.parametrize("n,n_obs", [(1, 0), (1, 2), (2, 0), (3, 0), (5, 2), (8, 0)])
@pytest.mark.parametrize("rho", [0.0, 1.0, 37.5, 512.0])
def test_structured_solve_equals_dense_kkt(n, n_obs, rho):
    spec = _spec(n, n_obs)
    basis = poly.for_spec(spec)
    op = kkt.stage_operator(basis, n, n_obs, rho)
    pr = am_oracle.Problem(spec)
    rng = np.random.default_rng(7)
    for _ in range(3):
        b = rng.normal(size=(pr.p, pr.m))
        R = (pr.S.T @ b) @ pr.P  # (n, nv), the S'b P of one axis
        beq = pr.b_eq[0].reshape(n, 6)
        dense = np.linalg.solve(pr.kkt(rho), np.concatenate([rho * R.ravel(), beq.ravel()]))[: n * pr.nv]
        bb = beq.mean(axis=0)
        c = (rho * R @ op.G.T + rho * R.mean(axis=0) @ op.Gm.T + (beq - bb) @ op.F.T + bb @ op.Fm.T)
        scale = max(1.0, np.linalg.norm(dense))
        assert np.linalg.norm(c.ravel() - dense) <= 1e-8 * scale


def test_stage_operator_rejects_negative_rho_and_singular_basis():
    basis = build_basis(20, 2.0, 6)
    with pytest.raises(ValueError):
        kkt.stage_operator(basis, 2, 0, -1.0)


# --- rho schedule (reference kkt_cache.py:356-382; test_kkt.py:322-345) -------------------------

def test_schedule_geometric_values():
    s = build_rho_schedule(1.0, 2.0, 10, 150)
    assert list(s.values) == [1, 2, 4, 8, 16, 32, 64, 128, 256, 512]
    assert s.switch_every == 15
    assert (s.stage_for(0), s.stage_for(14), s.stage_for(15), s.stage_for(149), s.stage_for(1000)) == (0, 0, 1, 9, 9)


@pytest.mark.parametrize("args", [(0.0, 2.0, 10, 150), (-1.0, 2.0, 10, 150), (1.0, 1.0, 10, 150), (1.0, 2.0, 0, 150),
                                  (1.0, 2.0, 10, 0)])
def test_schedule_rejects_bad_parameters(args):
    with pytest.raises(ValueError):
        build_rho_schedule(*args)


# --- factor cache census -------------------------------------------------------------------------

def test_factor_cache_counts_and_single_flight():
    spec = _spec(3, 0)
    basis = poly.for_spec(spec)
    fp = kkt.fingerprint(basis, 3, 0)
    cache = FactorCache()
    sched = build_rho_schedule(1.0, 2.0, 10, 150)
    threads = [threading.Thread(target=cache.prefactorize, args=(fp, basis, sched)) for _ in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    st = cache.stats()
    assert st["factorizations"] == 10 and st["entries"] == 10 and st["misses"] == 10
    assert st["hits"] == 70
    cache.prefactorize(fp, basis, sched)
    assert cache.stats()["factorizations"] == 10


def test_fingerprint_ignores_boundary_values():
    a, b = generate_random(8, (8, 8, 3), 0.4, 0), generate_random(8, (8, 8, 3), 0.4, 1)
    fa = kkt.fingerprint(poly.for_spec(a), 8, 0).key()
    fb = kkt.fingerprint(poly.for_spec(b), 8, 0).key()
    assert fa == fb
    assert kkt.fingerprint(poly.for_spec(a), 9, 0).key() != fa


# --- packing (boundary rows and straight lines) ----------------------------------------------------

def test_pack_layout_matches_reference_assembly():
    specs = [_spec(4, 2), _spec(4, 2)]
    basis = poly.for_spec(specs[0])
    c0, beq, geom = pack(specs, basis)
    pr = am_oracle.Problem(specs[0])
    for ax in range(3):
        np.testing.assert_array_equal(beq[0, ax].ravel(), pr.b_eq[ax])
    assert c0.shape == (2, 3, 4, basis.num_coeffs)
    s = specs[0]
    np.testing.assert_allclose(basis.P @ c0[0, 0, 1], np.linspace(s.start[1].position[0], s.goal[1].position[0],
                                                                   basis.num_samples), atol=1e-12)
    assert geom.shape == (2, 2 + 5 * 2)
    np.testing.assert_allclose(geom[0, 2:7], (*s.obstacles[0].center, 0.4 + 0.3, 0.3 + 0.3))


# --- validation and config errors are raised before any device work --------------------------------

def test_infeasible_spec_raises_before_device_work():
    spec = ProblemSpec(start=(BoundaryState.at_rest((0, 0, 0)), BoundaryState.at_rest((0.1, 0, 0))),
                       goal=(BoundaryState.at_rest((5, 0, 0)), BoundaryState.at_rest((5, 1, 0))),
                       geometry=AgentGeometry.sphere_from_radius(0.5))
    with pytest.raises(InfeasibleProblemError) as err:
        engine.am_solve(spec)
    assert err.value.violations


def test_solver_config_validation():
    for kw in ({"max_iters": 0}, {"tolerance": 0.0}, {"initialization": "random"}):
        with pytest.raises(ValueError):
            SolverConfig(**kw)


def test_batch_must_share_a_fingerprint():
    with pytest.raises(ValueError, match="fingerprint"):
        engine.am_solve_batch([generate_random(4, (8, 8, 3), 0.4, 0), generate_random(5, (8, 8, 3), 0.4, 0)])


def test_track_descent_needs_a_single_solve():
    specs = [generate_random(4, (8, 8, 3), 0.4, s) for s in (0, 1)]
    with pytest.raises(ValueError, match="single"):
        engine.am_solve_batch(specs, SolverConfig(track_descent=True))


# --- collision metrics (reference validation.py) ------------------------------------------------------

@pytest.mark.parametrize("name", ["obs8", "rand8_s0", "hallway4j"])
def test_collision_metrics_match_oracle(name):
    spec, cfg, _ = load_golden(name)
    out = am_oracle.solve(spec, max_iters=5)
    col = check_collisions(out["trajectories"], spec.geometry, spec.obstacles)
    md, nviol = am_oracle.min_normalized_distance(spec, out["trajectories"])
    assert col.min_normalized_distance == pytest.approx(md, rel=1e-12)
    assert len(col.violations) == nviol


# --- the C ABI library -----------------------------------------------------------------------------------

def test_native_library_exports_every_declared_symbol():
    import ctypes

    from paper_2011_04240_b200 import native
    header = open(os.path.join(ROOT, "include", "swarm_am.h")).read()
    declared = set(re.findall(r"\b(st_[a-z_]+)\s*\(", header))
    assert declared >= {"st_plan_create", "st_solve", "st_solve_device", "st_plan_destroy", "st_last_error"}
    lib = native.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.st_version() >= 1
    # argument errors are reported without touching a device
    h = ctypes.c_void_p()
    assert lib.st_plan_create(0, 0, 10, 11, 1, None, None, None, None, None, None, None, 0, ctypes.byref(h)) == 1
    assert b"dimensions" in lib.st_last_error()


def test_vectorized_validate_equals_scalar_loop():
    """validate's prefilter must not change the reference's violations, order or text (problem.py:162-194)."""
    import dataclasses

    from paper_2011_04240_b200.spec import Violation, _separation, obstacle_axes, validate

    def scalar(spec):
        out, g, n = [], spec.geometry, len(spec.start)
        for label, states in (("start", spec.start), ("goal", spec.goal)):
            pos = [s.position for s in states]
            for i in range(n):
                for j in range(i + 1, n):
                    sep = _separation(pos[i], pos[j], g.l_xy, g.l_z)
                    if sep < 1.0:
                        out.append(Violation(f"{label} pair ({i}, {j})", f"normalized separation {sep:.4f} < 1"))
            for i in range(n):
                for k, obs in enumerate(spec.obstacles):
                    lxy, lz = obstacle_axes(spec, obs)
                    sep = _separation(pos[i], obs.center, lxy, lz)
                    if sep < 1.0:
                        out.append(Violation(f"{label} agent {i} vs obstacle {k}",
                                             f"normalized separation {sep:.4f} < 1"))
        return out

    rng = np.random.default_rng(0)
    total = 0
    for trial in range(25):
        spec = generate_random(int(rng.integers(1, 25)), (8, 8, 3), 0.4, trial)
        starts = tuple(dataclasses.replace(s, position=tuple((np.array(s.position) * rng.uniform(0.05, 1)).tolist()))
                       for s in spec.start)
        spec = dataclasses.replace(spec, start=starts)
        got = validate(spec)
        assert got == scalar(spec)
        total += len(got)
    assert total > 0


def test_position_and_batch_validation_equal_validate():
    """The array-fed validators of the solve path (single: validate_positions, batch: validate_batch,
    both with the obstacle prefilter) report validate's violations, order and text, obstacles included."""
    import dataclasses

    from paper_2011_04240_b200 import metrics
    from paper_2011_04240_b200.spec import Obstacle as Ob, validate, validate_batch, validate_positions

    rng = np.random.default_rng(5)
    specs, total = [], 0
    for trial in range(30):
        n = int(rng.integers(1, 20))
        spec = generate_random(n, (8, 8, 3), 0.4, trial)
        scale = rng.uniform(0.05, 1)
        starts = tuple(dataclasses.replace(s, position=tuple((np.array(s.position) * scale).tolist()))
                       for s in spec.start)
        obs = tuple(Ob(center=tuple(rng.uniform(-4, 4, 3).tolist()), radius=float(rng.uniform(0.2, 1.5)))
                    for _ in range(3))
        specs.append(dataclasses.replace(spec, start=starts, obstacles=obs))
    for spec in specs:
        bnd = engine.boundary_arrays([spec])
        rows = metrics._obstacle_rows(spec.geometry, spec.obstacles)
        want = validate(spec)
        assert validate_positions(spec, bnd[0, 0, 0], bnd[0, 1, 0], rows) == want
        assert validate_positions(spec, bnd[0, 0, 0], bnd[0, 1, 0]) == want
        total += sum("obstacle" in v.subject for v in want)
    assert total > 0
    for n in (1, 3, 11):  # a batch shares one shape: rebuild the specs at n agents
        group = []
        for trial, base in enumerate(specs[:8]):
            spec = generate_random(n, (8, 8, 3), 0.4, 100 + trial)
            starts = tuple(dataclasses.replace(s, position=tuple((np.array(s.position) * 0.2).tolist()))
                           for s in spec.start)
            group.append(dataclasses.replace(spec, start=starts, obstacles=base.obstacles))
        bnd = engine.boundary_arrays(group)
        rows = np.stack([metrics._obstacle_rows(g.geometry, g.obstacles) for g in group])
        assert validate_batch(group, bnd[:, 0, 0], bnd[:, 1, 0], rows) == [validate(g) for g in group]
        assert validate_batch(group, bnd[:, 0, 0], bnd[:, 1, 0]) == [validate(g) for g in group]


def test_vectorized_trajectory_metrics_bitwise():
    from paper_2011_04240_b200 import metrics
    rng = np.random.default_rng(3)
    for n, m in ((1, 3), (7, 10), (40, 100)):
        traj = rng.normal(size=(n, m, 3)) * 3
        q = metrics.trajectory_metrics(traj)
        assert q.arc_length == tuple(metrics.arc_length(t) for t in traj)
        assert q.smoothness == tuple(metrics.smoothness(t) for t in traj)


def test_disk_cache_roundtrip(tmp_path):
    """Mirrors the reference's test_kkt.py:292-316 for the structured stage operators."""
    from paper_2011_04240_b200 import kkt, poly
    spec = generate_random(2, (8, 8, 3), 0.4, 0)
    basis = poly.for_spec(spec)
    fp = kkt.fingerprint(basis, 2, 0)
    schedule = kkt.build_rho_schedule(1.0, 2.0, 3, 30)
    writer = kkt.FactorCache(disk_dir=tmp_path)
    manifest = writer.persist(fp, basis, schedule)
    assert manifest["rho_values"] == [1.0, 2.0, 4.0]
    entry = tmp_path / manifest["fingerprint"]
    assert (entry / kkt.OPERATORS_FILE).exists()
    before = (entry / kkt.MANIFEST_FILE).read_bytes()
    kkt.FactorCache(disk_dir=tmp_path).persist(fp, basis, schedule)
    assert (entry / kkt.MANIFEST_FILE).read_bytes() == before  # idempotent rebuild
    reader = kkt.FactorCache(disk_dir=tmp_path)
    op = reader.get(fp, basis, 2.0)
    assert reader.stats()["factorizations"] == 0 and reader.stats()["hits"] == 1  # loaded, not rebuilt
    fresh = kkt.stage_operator(basis, 2, 0, 2.0)
    for name in ("G", "Gm", "F", "Fm"):
        np.testing.assert_array_equal(getattr(op, name), getattr(fresh, name))
    # a rho outside the manifest is built, and a corrupt entry is ignored with a rebuild
    reader.get(fp, basis, 8.0)
    assert reader.stats()["factorizations"] == 1
    (entry / kkt.OPERATORS_FILE).write_bytes(b"not an npz")
    broken = kkt.FactorCache(disk_dir=tmp_path)
    broken.get(fp, basis, 1.0)
    assert broken.stats()["factorizations"] == 1


def test_pinned_pool_release_is_reentrant():
    """The pool's release runs as a weakref finalizer, i.e. from the garbage collector, which can
    fire inside the pool's own critical section: releasing with the lock held must not deadlock."""
    import threading

    from paper_2011_04240_b200 import native
    pool = native._PinnedPool(keep=4)
    done = []

    def run():
        with pool._lock:
            pool._release(0x1000, 64)  # a finalizer firing while the lock is held
        done.append(True)

    t = threading.Thread(target=run, daemon=True)
    t.start()
    t.join(5.0)
    assert done == [True] and pool._free[64] == [0x1000]
