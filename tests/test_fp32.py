"""FP32 mode (north star: "an optional FP32 mode with a stated tolerance on final residual and
minimum inter-agent clearance").

FP32 pair state: multipliers and the per-pair-sample arithmetic (projection, d-step,
residual, multiplier update, next right-hand side) in FP32; positions, the S'b sums,
the projection onto the basis and the KKT solve in FP64.  Stated tolerances against
the FP64 reference, checked on the reference's golden fixtures:

    coefficients            <= 1e-4 normwise (||dc|| / ||c||); measured 1e-6 (n=8) .. 2e-5 (n=256).
                            SURVEY A.6's 1e-7..3e-7 rounded only D and lambda to FP32 and kept
                            the pair arithmetic in FP64; here the arithmetic itself is FP32 (a numpy
                            emulation of the same FP32 arithmetic gives 1.2e-6 on rand8_s0, as the
                            device does), so the bar is set from measurement with 5x margin
    iterations, converged   identical
    final residual norm     within 1e-4 relative   (and max-abs within 1e-4 relative)
    min normalized clearance within 1e-4 absolute; violation count identical
"""

import numpy as np
import pytest

from conftest import load_golden, rel_err

pytestmark = pytest.mark.gpu

COEFF_TOL = 1e-4
RES_RTOL = 1e-4
CLEAR_ATOL = 1e-4

# non-chaotic fixtures (the reference's own self-noise is far below the FP32 tolerance)
NAMES = ["rand3_s0", "rand5_s1", "rand8_s0", "rand8_s1", "rand8_s2_sched", "rand20_s0", "circ16j", "sph16j",
         "rand32_s0", "rand32_s1", "rand48_s0", "sph64j", "obs8", "hallway4j", "boundary_derivatives",
         "rand128_s0", "rand256_s0"]


def _solve(name, fp32):
    from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve
    spec, cfg, ref = load_golden(name)
    rep = am_solve(spec, SolverConfig(**cfg, fp32=fp32), cache=FactorCache())
    return rep, ref


@pytest.mark.parametrize("name", NAMES)
def test_fp32_within_stated_tolerance_of_reference(cuda_ok, name):
    rep, ref = _solve(name, True)
    assert rep.iterations == int(ref["iterations"])
    assert rep.converged == bool(ref["converged"])
    err = rel_err(rep.coefficients, ref["coefficients"])
    assert err <= COEFF_TOL, f"fp32 coefficients off by {err:.3e}"
    assert rep.residual_norm == pytest.approx(float(ref["residual_norm_history"][-1]), rel=RES_RTOL)
    assert rep.residual_max_abs == pytest.approx(float(ref["residual_max_history"][-1]), rel=RES_RTOL)
    assert rep.metrics["num_collision_violations"] == int(ref["num_collision_violations"])
    md_ref = float(ref["min_normalized_distance"])
    if np.isfinite(md_ref):
        assert abs(rep.metrics["min_normalized_distance"] - md_ref) <= CLEAR_ATOL


def test_fp32_batch_matches_fp32_single(cuda_ok):
    from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve, am_solve_batch, generate_random
    specs = [generate_random(32, (8.0, 8.0, 3.0), 0.4, s) for s in range(200)]
    cache = FactorCache()
    reps = am_solve_batch(specs, SolverConfig(fp32=True), cache=cache, with_metrics=False)
    for idx in (0, 199):
        one = am_solve_batch([specs[idx]], SolverConfig(fp32=True, cluster_size=2), cache=cache,
                             with_metrics=False)[0]
        assert one.iterations == reps[idx].iterations
        np.testing.assert_array_equal(one.coefficients, reps[idx].coefficients)
    ref0 = am_solve(specs[0], SolverConfig(), cache=cache)
    assert rel_err(reps[0].coefficients, ref0.coefficients) <= COEFF_TOL


def test_fp32_keep_state_exports_reference_layout(cuda_ok):
    from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve
    spec, cfg, ref = load_golden("obs8_state")
    rep = am_solve(spec, SolverConfig(**cfg, fp32=True, keep_state=True), cache=FactorCache())
    st = rep.diagnostics["final_state"]
    lam = np.stack([st.multipliers.lambda_x, st.multipliers.lambda_y, st.multipliers.lambda_z])
    assert lam.shape == ref["lam"].shape
    assert rel_err(lam, ref["lam"]) <= 1e-4
    assert np.all(st.pair_vars.d >= 1.0)


def test_fp32_is_deterministic(cuda_ok):
    a, _ = _solve("rand32_s0", True)
    b, _ = _solve("rand32_s0", True)
    np.testing.assert_array_equal(a.coefficients, b.coefficients)
