"""The drop-in under the reference's own objects and callers.

The reference package is the sanctioned offline install under ``baseline/_ref``
(pip --target; git-ignored, travels to the GPU box); tests skip without it.
* host-only: a reference ``SolverConfig`` / ``FactorCache`` / ``InfeasibleProblemError``
  are accepted and honoured by the drop-in's host logic;
* GPU: the reference's own test suite (pkg/tests, 198 tests) runs with
  ``swarmtraj.am_solve`` rebound to the drop-in (``compat.install()``,
  scripts/refsuite/), and a live reference spec/config/cache solve matches the
  golden fixture.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, coeff_tol, load_golden, rel_err

REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def swarmtraj():
    if not os.path.isdir(os.path.join(REF, "swarmtraj")):
        pytest.skip("reference not installed under baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import swarmtraj
    return swarmtraj


def test_reference_config_and_cache_are_accepted_on_the_host(swarmtraj):
    from paper_2011_04240_b200 import engine
    cfg = swarmtraj.SolverConfig(max_iters=40)
    assert engine._opt(cfg, "device", 0) == 0 and engine._opt(cfg, "fp32", False) is False
    ref_cache = swarmtraj.FactorCache()
    side, foreign = engine._resolve_cache(ref_cache)
    assert foreign is ref_cache and engine._resolve_cache(ref_cache)[0] is side
    before = side.stats()
    side.count_solve(6)
    engine._sync_foreign(side, foreign, before)
    assert ref_cache.solves == 6 and ref_cache.stats()["solves"] == 6


def test_validation_error_is_catchable_as_the_reference_class(swarmtraj):
    from paper_2011_04240_b200 import InfeasibleProblemError, am_solve
    P = swarmtraj.problem
    spec = P.ProblemSpec(start=(P.BoundaryState.at_rest((0, 0, 0)), P.BoundaryState.at_rest((0.1, 0, 0))),
                         goal=(P.BoundaryState.at_rest((5, 0, 0)), P.BoundaryState.at_rest((6, 0, 0))),
                         geometry=P.AgentGeometry.sphere_from_radius(0.4))
    with pytest.raises(swarmtraj.InfeasibleProblemError) as ei:
        am_solve(spec)  # validation runs before any device work: no GPU needed
    assert isinstance(ei.value, InfeasibleProblemError) and ei.value.violations


def test_keep_state_export_supports_reference_state_functions(swarmtraj):
    """reference update_multipliers / compute_residual run on our SystemView (host only)."""
    from paper_2011_04240_b200 import engine, poly
    spec = swarmtraj.problem.generate_random_with_obstacles(5, (8.0, 8.0, 3.0), 0.4, 2, 0.5, 1)
    from swarmtraj.basis import build_basis, build_time_grid
    from swarmtraj.kkt_cache import assemble
    ref_sys = assemble(spec, build_basis(build_time_grid(spec.num_samples, spec.duration), spec.degree))
    view = engine.SystemView(spec, poly.for_spec(spec))
    c = np.random.default_rng(3).standard_normal(5 * 11)
    np.testing.assert_allclose(view.pairs.apply(c), ref_sys.pairs.apply(c), rtol=0, atol=1e-13)
    v = np.random.default_rng(4).standard_normal(view.pairs.num_pairs * spec.num_samples)
    np.testing.assert_allclose(view.pairs.apply_transpose(v), ref_sys.pairs.apply_transpose(v), atol=1e-12)
    np.testing.assert_array_equal(view.pairs.offsets, ref_sys.pairs.offsets)
    assert abs(c @ view.Q @ c - c @ ref_sys.Q @ c) <= 1e-9 * abs(c @ ref_sys.Q @ c)


@pytest.mark.gpu
def test_live_reference_objects_solve_to_the_fixture(cuda_ok, swarmtraj):
    from paper_2011_04240_b200 import am_solve
    spec = swarmtraj.problem.generate_random(32, (8, 8, 3), 0.4, 0)
    _, _, ref = load_golden("rand32_s0")
    cache = swarmtraj.FactorCache()
    rep = am_solve(spec, swarmtraj.SolverConfig(), cache=cache)
    assert rep.iterations == int(ref["iterations"])
    assert rel_err(rep.coefficients, ref["coefficients"]) <= coeff_tol(ref)
    st = cache.stats()
    assert st["factorizations"] == 10 and st["solves"] == 3 * rep.iterations and st["entries"] >= 10
    rep2 = am_solve(spec, swarmtraj.SolverConfig(max_iters=20), cache=cache)
    assert cache.stats()["factorizations"] == 10 and cache.stats()["hits"] >= 10
    assert rep2.cache_stats == cache.stats()


@pytest.mark.gpu
def test_reference_test_suite_passes_on_the_dropin(cuda_ok, swarmtraj):
    runner = os.path.join(ROOT, "scripts", "refsuite", "run.py")
    if not os.path.isdir(os.path.join(REF, "ref_tests")):
        pytest.skip("reference tests not staged (scripts/refsuite/run.py prepare)")
    # the suite takes ~10 s here; a hang must fail this test, not stall the GPU run
    res = subprocess.run([sys.executable, runner, "-q", "-rf"], capture_output=True, text=True, timeout=300)
    tail = "\n".join(res.stdout.splitlines()[-25:])
    assert res.returncode == 0, tail
    assert "served by the B200 drop-in" in res.stdout
