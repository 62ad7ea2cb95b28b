"""Device-side guards: non-finite state (reference _check_ranges, solver.py:355-360), plan
sharing across streams, unknown flags."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _plan_and_inputs(n=8, seed=0):
    from paper_2011_04240_b200 import FactorCache, SolverConfig, engine, generate_random, kkt, pack, poly
    spec = generate_random(n, (8.0, 8.0, 3.0), 0.4, seed)
    basis = poly.for_spec(spec)
    cfg = SolverConfig()
    plan = engine._plan_for(FactorCache(), kkt.fingerprint(basis, n, 0), basis, cfg.schedule(), n, 0, 0)
    return spec, cfg, plan, pack([spec], basis)


@pytest.mark.parametrize("fp32", [False, True])
def test_nan_boundary_state_is_flagged_not_converged(cuda_ok, fp32):
    """A NaN in the inputs must never come back as converged=True (max-abs drops NaN); the
    kernel flags the scenario and the drop-in raises like the reference's assertion."""
    from paper_2011_04240_b200 import native
    spec, cfg, plan, (c0, beq, geom) = _plan_and_inputs()
    c0 = c0.copy()
    c0[0, 1, 3, 4] = np.nan
    out = plan.solve(c0, beq, geom, cfg.schedule().switch_every, 150, 1e-2, fp32=fp32)
    assert int(out["status"][0]) == native.ST_NONFINITE
    assert not out["converged"][0]
    assert int(out["iters"][0]) >= 1


def test_nan_state_raises_through_am_solve(cuda_ok, monkeypatch):
    from paper_2011_04240_b200 import NonFiniteStateError, am_solve, engine, generate_random
    spec = generate_random(8, (8.0, 8.0, 3.0), 0.4, 0)
    real_pack = engine.pack

    def poisoned(specs, basis, *args):
        c0, beq, geom = real_pack(specs, basis, *args)
        c0[0, 0, 0, 5] = np.inf
        return c0, beq, geom

    monkeypatch.setattr(engine, "pack", poisoned)
    with pytest.raises(NonFiniteStateError):
        am_solve(spec)
    with pytest.raises(AssertionError):  # the reference's exception type
        am_solve(spec)


def test_device_solves_on_two_streams_share_a_plan_safely(cuda_ok):
    """Two st_solve_device launches on different streams reuse one plan's workspaces; the
    plan orders them, so both results equal a host solve."""
    import torch
    spec, cfg, plan, (c0, beq, geom) = _plan_and_inputs(16, 3)
    ref = plan.solve(c0, beq, geom, cfg.schedule().switch_every, 150, 1e-2)
    dev = torch.device("cuda", 0)
    outs = []
    streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
    ins = [torch.from_numpy(a).to(dev) for a in (c0, beq, geom)]
    for st in streams:
        o = (torch.empty_like(ins[0]), torch.empty((1, 3, 150), dtype=torch.float64, device=dev),
             torch.empty(1, dtype=torch.int32, device=dev), torch.empty(1, dtype=torch.int32, device=dev))
        plan.solve_device(1, ins[0].data_ptr(), ins[1].data_ptr(), ins[2].data_ptr(), cfg.schedule().switch_every,
                          150, 1e-2, o[0].data_ptr(), o[1].data_ptr(), o[2].data_ptr(), o[3].data_ptr(),
                          stream=st.cuda_stream)
        outs.append(o)
    torch.cuda.synchronize()
    for o in outs:
        np.testing.assert_array_equal(o[0].cpu().numpy(), ref["c"])
        assert int(o[2].item()) == int(ref["iters"][0])


def test_unknown_flag_bits_rejected(cuda_ok):
    from paper_2011_04240_b200 import native
    _, cfg, plan, (c0, beq, geom) = _plan_and_inputs()
    import ctypes
    out = (ctypes.c_longlong * 8)()
    with pytest.raises(ValueError):
        native._check(plan._lib.st_query_launch(plan._h, 1, 0, 64, out)) if False else None
        plan.solve.__wrapped__ if False else None
        native._check(plan._lib.st_solve(plan._h, 1, native._ptr(c0), native._ptr(beq), native._ptr(geom), 15,
                                         150, 1e-2, 64, 0, native._ptr(np.empty_like(c0)),
                                         native._ptr(np.empty((1, 3, 150))),
                                         native._ptr(np.empty(1, np.int32), native._ip),
                                         native._ptr(np.empty(1, np.int32), native._ip), None, None, None))
