"""Install the drop-in under the reference package's own callers.

``install()`` rebinds ``am_solve`` in ``swarmtraj``, ``swarmtraj.solver`` and the
modules that imported it by name (cli.py:36, service/app.py, bench.py), so the
CLI, the HTTP service and the bench suites run on the B200 with their own
``ProblemSpec`` / ``SolverConfig`` / ``FactorCache`` objects.  It also extends the
reference's ``FactorCache.persist`` / ``prefactorize`` (kkt_cache.py:454-528) so
that a prebuilt cache entry (``swarmtraj cache`` / ``POST /cache/build``) carries
the device stage operators too (``b200_operators.npz`` beside the reference's
``factors.npz``): a later drop-in solve of that fingerprint is then a cache hit,
as it is for the reference.
"""

from __future__ import annotations

import importlib

from . import engine, kkt, poly

_INSTALLED: dict = {}


def _basis_from_reference(system) -> poly.Basis:
    """Our basis view of a reference AssembledSystem (its matrices are bitwise ours)."""
    b = system.pairs.basis
    fp = system.fingerprint
    return poly.Basis(P=b.P, Pdot=b.Pdot, Pddot=b.Pddot, samples=getattr(b, "samples", None),
                      duration=float(getattr(b, "duration", 0.0)), kind=poly.BasisKind(fp.basis_kind),
                      degree=fp.num_coeffs - 1)


def _device_stages(cache, system, schedule, persist: bool) -> None:
    """Build (and optionally persist) the device stage operators of a reference system in the
    side cache.  Side-cache counters are not mirrored: the reference counted its own work."""
    side, _ = engine._resolve_cache(cache)
    fp = system.fingerprint
    ours = kkt.Fingerprint(fp.num_agents, fp.num_samples, fp.num_coeffs, fp.num_obstacles, fp.basis_kind,
                           fp.basis_sha)
    sched = kkt.RhoSchedule(values=tuple(float(v) for v in schedule.values), switch_every=schedule.switch_every)
    basis = _basis_from_reference(system)
    if persist:
        side.persist(ours, basis, sched)
    else:
        side.prefactorize(ours, basis, sched)


def install(swarmtraj=None) -> None:
    """Route the reference package's entry point and callers to the B200 drop-in."""
    if swarmtraj is None:
        import swarmtraj
    if _INSTALLED.get("pkg") is swarmtraj:
        return
    solver = importlib.import_module(swarmtraj.__name__ + ".solver")
    kc = importlib.import_module(swarmtraj.__name__ + ".kkt_cache")

    def am_solve(spec, config=None, cache=None):
        return engine.am_solve(spec, config, cache)

    am_solve.__doc__ = engine.am_solve.__doc__
    solver.am_solve = am_solve
    swarmtraj.am_solve = am_solve
    for name in ("bench", "service.app", "cli"):
        try:
            mod = importlib.import_module(f"{swarmtraj.__name__}.{name}")
        except ImportError:  # optional front-end dependency (click / fastapi) missing
            continue
        if hasattr(mod, "am_solve"):
            mod.am_solve = am_solve

    ref_persist, ref_prefactorize = kc.FactorCache.persist, kc.FactorCache.prefactorize

    def persist(self, system, schedule):
        manifest = ref_persist(self, system, schedule)
        _device_stages(self, system, schedule, persist=True)
        return manifest

    def prefactorize(self, system, schedule):
        factors = ref_prefactorize(self, system, schedule)
        _device_stages(self, system, schedule, persist=False)
        return factors

    kc.FactorCache.persist = persist
    kc.FactorCache.prefactorize = prefactorize
    _INSTALLED["pkg"] = swarmtraj
