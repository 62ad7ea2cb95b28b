"""Drop-in ``am_solve``: the reference entry point, computed on the B200.

Reference: ``solver.py`` -- ``SolverConfig`` (60-82), ``SolveReport``
(139-172), ``InfeasibleProblemError`` (49-57), ``am_solve`` (363-494).
Same signature, same report layout (trajectories (n,m,3), coefficients
(3,n,n_v), histories of length ``iterations``), same error behaviour
(validation before any work, non-convergence reported not raised), same
``cache_stats`` census (10 factorizations per new fingerprint, 3 solves
per iteration).

The host does only shape work: basis, packing of boundary rows and
straight-line coefficients, the per-stage 17x17 operators (cached), and
the post-loop metrics.  Every iteration of the loop runs in one cluster
kernel on the device (csrc/am_kernel.cuh); there is no CPU path.
``am_solve_batch`` runs many scenarios sharing one fingerprint in one
launch (the reference runs those through a thread pool, bench.py:120-158).
"""

from __future__ import annotations

import gc
import itertools
import logging
import math
import sys
import time
import weakref
from dataclasses import dataclass, field
from operator import attrgetter

import numpy as np

from . import kkt, metrics, native, poly
from .spec import obstacle_axes, validate, validate_batch, validate_positions

log = logging.getLogger(__name__)


class NonFiniteStateError(AssertionError):
    """The pair state left its valid range (NaN/inf), where the reference's ``_check_ranges``
    assertion fires (solver.py:355-360, called every iteration at solver.py:437)."""


class InfeasibleProblemError(ValueError):
    def __init__(self, violations):
        self.violations = list(violations)
        text = "; ".join(str(v) for v in self.violations[:5])
        if len(self.violations) > 5:
            text += f"; ... ({len(self.violations)} total)"
        super().__init__(f"invalid problem instance: {text}")


def _infeasible(violations) -> InfeasibleProblemError:
    """The validation error to raise.  When the reference package is loaded (the drop-in is
    serving its callers, cli.py:186-191 / app.py:70-86 catch ``swarmtraj.InfeasibleProblemError``),
    the error is an instance of both classes so either ``except`` clause catches it."""
    ref = sys.modules.get("swarmtraj.solver")
    ref_cls = getattr(ref, "InfeasibleProblemError", None)
    if isinstance(ref_cls, type) and issubclass(ref_cls, ValueError) and ref_cls is not InfeasibleProblemError:
        both = _COMPAT_ERRORS.get(ref_cls)
        if both is None:
            both = type("InfeasibleProblemError", (InfeasibleProblemError, ref_cls), {})
            _COMPAT_ERRORS[ref_cls] = both
        err = both.__new__(both)
        InfeasibleProblemError.__init__(err, violations)
        return err
    return InfeasibleProblemError(violations)


_COMPAT_ERRORS: dict = {}


def _opt(config, name: str, default):
    """B200 extension fields of SolverConfig; the reference's own config (schemas.py:88-89,
    solver.py:60-82) has none of them and gets the defaults."""
    return getattr(config, name, default)


@dataclass
class SolverConfig:
    max_iters: int = 150
    tolerance: float = 1e-2
    rho_initial: float = 1.0
    rho_growth: float = 2.0
    rho_stages: int = 10
    initialization: str = "straight_line"
    track_descent: bool = False
    keep_state: bool = False
    # B200 extensions (not in the reference): CTAs per scenario (0 = auto), device ordinal,
    # FP32 pair state (multipliers and pair arithmetic in FP32, FP64 solve)
    cluster_size: int = 0
    device: int = 0
    fp32: bool = False

    def __post_init__(self):
        if self.max_iters < 1:
            raise ValueError(f"max_iters must be >= 1, got {self.max_iters}")
        if not self.tolerance > 0:
            raise ValueError(f"tolerance must be positive, got {self.tolerance}")
        if self.initialization != "straight_line":
            raise ValueError(f"unknown initialization mode {self.initialization!r}")

    def schedule(self) -> kkt.RhoSchedule:
        return kkt.build_rho_schedule(self.rho_initial, self.rho_growth, self.rho_stages, self.max_iters)


@dataclass
class PairVariables:
    alpha: np.ndarray
    beta: np.ndarray
    d: np.ndarray


@dataclass
class Multipliers:
    lambda_x: np.ndarray
    lambda_y: np.ndarray
    lambda_z: np.ndarray

    def for_axis(self, axis: int) -> np.ndarray:
        return (self.lambda_x, self.lambda_y, self.lambda_z)[axis]


class PairRows:
    """Host view of the pair incidence of one spec -- the attributes of the reference's
    ``PairwiseBlock`` (kkt_cache.py:104-135) that its state functions read (``apply``,
    ``apply_transpose``, ``offsets``, ``l_xy``, ``l_z``, ``num_pairs``, ``basis``), so the
    reference's ``update_multipliers`` / ``compute_residual`` / ``augmented_cost``
    (solver.py:228-303) run on a ``keep_state`` export.  Rows: agent pairs (i<j,
    lexicographic), then (agent, obstacle) agent-major (kkt_cache.py:197-215).  Diagnostic
    only, never on the solve path."""

    def __init__(self, spec, basis):
        n, n_obs = len(spec.start), len(spec.obstacles)
        self.basis, self.num_agents = basis, n
        self._ii, self._jj = np.triu_indices(n, k=1)
        npair = len(self._ii)
        self.num_pairs = npair + n * n_obs
        self.offsets = np.zeros((self.num_pairs, 3))
        self.l_xy = np.full(self.num_pairs, float(spec.geometry.l_xy))
        self.l_z = np.full(self.num_pairs, float(spec.geometry.l_z))
        self._obs_agent = np.repeat(np.arange(n), n_obs)
        for i in range(n):
            for k, obs in enumerate(spec.obstacles):
                row = npair + i * n_obs + k
                self.offsets[row] = obs.center
                self.l_xy[row], self.l_z[row] = obstacle_axes(spec, obs)

    def apply(self, c_flat: np.ndarray) -> np.ndarray:
        """(n * n_v,) coefficients of one axis -> (p * m,) pair differences, pair-major."""
        X = c_flat.reshape(self.num_agents, -1) @ self.basis.P.T
        return np.concatenate([X[self._ii] - X[self._jj], X[self._obs_agent]]).ravel()

    def apply_transpose(self, v: np.ndarray) -> np.ndarray:
        """(p * m,) -> (n * n_v,): (S' v) P."""
        v = v.reshape(self.num_pairs, -1)
        acc = np.zeros((self.num_agents, v.shape[1]))
        npair = len(self._ii)
        np.add.at(acc, self._ii, v[:npair])
        np.add.at(acc, self._jj, -v[:npair])
        np.add.at(acc, self._obs_agent, v[npair:])
        return (acc @ self.basis.P).ravel()


class SystemView:
    """``state.system`` of a ``keep_state`` export: ``pairs`` and the smoothness Hessian ``Q``
    = I (x) Pdd'Pdd (kkt_cache.py:161-235), sparse."""

    def __init__(self, spec, basis):
        self.pairs = PairRows(spec, basis)
        self._Q = None

    @property
    def Q(self):
        if self._Q is None:
            import scipy.sparse as sp
            H = self.pairs.basis.Pddot.T @ self.pairs.basis.Pddot
            self._Q = sp.kron(sp.identity(self.pairs.num_agents, format="csr"), sp.csr_matrix(H), format="csr")
        return self._Q


@dataclass
class FinalState:
    """Final solver state exported by ``keep_state`` (reference SolverState, solver.py:107-136)."""

    c_x: np.ndarray
    c_y: np.ndarray
    c_z: np.ndarray
    pair_vars: PairVariables
    multipliers: Multipliers
    rho: float
    stage: int
    iteration: int
    residual_norms: list
    residual_max: list
    system: SystemView | None = None

    def coeffs(self, axis: int) -> np.ndarray:
        return (self.c_x, self.c_y, self.c_z)[axis]

    def set_coeffs(self, axis: int, value: np.ndarray) -> None:
        setattr(self, ("c_x", "c_y", "c_z")[axis], value)

    def sampled_positions(self) -> np.ndarray:
        P = self.system.pairs.basis.P
        return np.stack([self.coeffs(a) @ P.T for a in range(3)], axis=-1)


@dataclass
class SolveReport:
    trajectories: np.ndarray
    coefficients: np.ndarray
    converged: bool
    iterations: int
    residual_norm: float
    residual_max_abs: float
    residual_norm_history: list
    residual_max_history: list
    boundary_max_history: list
    timings: dict
    metrics: dict
    cache_stats: dict
    diagnostics: dict = field(default_factory=dict)

    def to_dict(self, include_trajectories: bool = True) -> dict:
        doc = {
            "converged": self.converged,
            "iterations": self.iterations,
            "residual_norm": self.residual_norm,
            "residual_max_abs": self.residual_max_abs,
            "residual_norm_history": list(self.residual_norm_history),
            "residual_max_history": list(self.residual_max_history),
            "boundary_max_history": list(self.boundary_max_history),
            "timings": dict(self.timings),
            "metrics": dict(self.metrics),
            "cache_stats": dict(self.cache_stats),
        }
        if include_trajectories:
            doc["trajectories"] = self.trajectories.tolist()
        return doc


_DEFAULT_CACHE: kkt.FactorCache | None = None


def default_cache() -> kkt.FactorCache:
    global _DEFAULT_CACHE
    if _DEFAULT_CACHE is None:
        _DEFAULT_CACHE = kkt.FactorCache()
    return _DEFAULT_CACHE


# --- host-side packing ---------------------------------------------------------------------


def boundary_arrays(specs) -> np.ndarray:
    """(B, 2, 3, n, 3) boundary states: scenario, start/goal, pos/vel/acc, agent, axis.

    One C-level pass over the state objects (attribute getters feeding ``np.fromiter``):
    the batch entry touches no per-agent Python beyond it."""
    B, n = len(specs), len(specs[0].start)
    chain = itertools.chain.from_iterable
    states = list(chain(side for spec in specs for side in (spec.start, spec.goal)))
    out = np.empty((3, len(states), 3))
    for f, name in enumerate(("position", "velocity", "acceleration")):
        out[f] = np.fromiter(chain(map(attrgetter(name), states)), dtype=float,
                             count=len(states) * 3).reshape(-1, 3)
    # out order: pos/vel/acc, (scenario, start/goal, agent), axis
    return out.reshape(3, B, 2, n, 3).transpose(1, 2, 0, 3, 4)


def pack(specs, basis: poly.Basis, bnd: np.ndarray | None = None, obs_rows: np.ndarray | None = None,
         alloc=np.empty):
    """Scenario batch -> (c0 (B,3,n,nv), b_eq (B,3,n,6), geom (B, 2+5 n_obs)).

    b_eq rows per agent and axis: [pos0, vel0, acc0, posT, velT, accT]
    (kkt_cache.py:174-185); c0 = straight line (solver.py:327-330).
    """
    B = len(specs)
    n = len(specs[0].start)
    n_obs = len(specs[0].obstacles)
    if bnd is None:
        bnd = boundary_arrays(specs)
    # alloc: the output arrays' allocator (page-locked buffers for the pipelined batch path)
    beq = alloc((B, 3, n, 6))
    np.copyto(beq.reshape(B, 3, n, 2, 3), bnd.transpose(0, 4, 3, 1, 2))
    c0 = poly.straight_line(basis, bnd[:, 0, 0].transpose(0, 2, 1), bnd[:, 1, 0].transpose(0, 2, 1),
                            out=alloc((B, 3, n, basis.num_coeffs)))
    geom = alloc((B, 2 + 5 * n_obs))
    geom[:, :2] = [(spec.geometry.l_xy, spec.geometry.l_z) for spec in specs]
    if n_obs:
        if obs_rows is None:  # (B, n_obs, 5): centre, l_xy/2 + R, l_z/2 + R (problem.py:136-141)
            obs_rows = np.array([[[*o.center, *obstacle_axes(spec, o)] for o in spec.obstacles] for spec in specs],
                                dtype=float)
        geom[:, 2:] = obs_rows.reshape(B, 5 * n_obs)
    return c0, beq, geom


def _plan_for(cache: kkt.FactorCache, fp, basis, schedule, n, n_obs, device):
    ops = cache.prefactorize(fp, basis, schedule)
    return cache.plan(fp, schedule, lambda: native.Plan(n, n_obs, basis, ops, device=device), device=device)


# Reference FactorCache objects (kkt_cache.py:385-456) passed in by the reference's callers
# (cli.py:209, bench.py:101, app.py:77): their LU store is useless to the device path, so the
# stage operators and device plans live in a side cache tied to the caller's object, and the
# caller's counters are advanced exactly as the reference would advance them.
_SIDE_CACHES: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_SIDE_LOCK = __import__("threading").Lock()


def _resolve_cache(cache):
    """-> (our FactorCache, foreign reference cache or None)."""
    if cache is None:
        return default_cache(), None
    if isinstance(cache, kkt.FactorCache):
        return cache, None
    if not all(hasattr(cache, a) for a in ("factorizations", "hits", "misses", "solves", "stats")):
        raise TypeError(f"cache must be a FactorCache, got {type(cache).__name__}")
    with _SIDE_LOCK:
        side = _SIDE_CACHES.get(cache)
        if side is None:
            side = kkt.FactorCache(disk_dir=getattr(cache, "disk_dir", None))
            _SIDE_CACHES[cache] = side
            ref_stats = cache.stats
            # reference stats() counts its LU entries; add the device-side stage entries
            cache.stats = lambda: {**ref_stats(), "entries": ref_stats()["entries"] + side.stats()["entries"]}
    return side, cache


def _sync_foreign(side: kkt.FactorCache, foreign, before: dict) -> None:
    """Advance the reference cache's counters by what the side cache just did."""
    if foreign is None:
        return
    after = side.stats()
    lock = getattr(foreign, "_lock", None)
    with (lock if lock is not None else _SIDE_LOCK):
        for k in ("factorizations", "hits", "misses", "solves"):
            setattr(foreign, k, getattr(foreign, k) + after[k] - before[k])


def _check_batch(specs):
    first = specs[0]
    key = (len(first.start), len(first.obstacles), first.num_samples, first.degree, float(first.duration),
           str(getattr(first.basis_kind, "value", first.basis_kind)))
    for s in specs[1:]:
        k2 = (len(s.start), len(s.obstacles), s.num_samples, s.degree, float(s.duration),
              str(getattr(s.basis_kind, "value", s.basis_kind)))
        if k2 != key:
            raise ValueError("all scenarios of a batch must share one fingerprint "
                             f"(agents, obstacles, samples, degree, duration, basis): {k2} != {key}")


def _alpha_beta(diffs, l_xy, l_z):
    """Final-state angles from the final differences (same formula as solver.py:178-195)."""
    planar = np.hypot(diffs[0], diffs[1])
    alpha = np.arctan2(diffs[1], diffs[0])
    beta = np.arctan2(planar / l_xy, diffs[2] / l_z)
    beta = np.where((planar == 0.0) & (diffs[2] == 0.0), np.pi / 2.0, beta)
    return alpha, beta


def _pair_state(spec, coeffs, basis):
    """Pair differences (solver.py:228-236), per-row semi-axes and projected angles of coefficients."""
    n, n_obs, m = len(spec.start), len(spec.obstacles), basis.num_samples
    X = np.einsum("ank,tk->ant", coeffs, basis.P)
    ii, jj = np.triu_indices(n, k=1)
    p = len(ii) + n * n_obs
    diffs = np.empty((3, p, m))
    diffs[:, : len(ii)] = X[:, ii] - X[:, jj]
    lxy = np.full((p, 1), spec.geometry.l_xy)
    lz = np.full((p, 1), spec.geometry.l_z)
    for i in range(n):
        for k, obs in enumerate(spec.obstacles):
            row = len(ii) + i * n_obs + k
            diffs[:, row] = X[:, i] - np.asarray(obs.center)[:, None]
            lxy[row], lz[row] = obstacle_axes(spec, obs)
    alpha, beta = _alpha_beta(diffs, lxy, lz)
    return diffs, lxy, lz, alpha, beta


def _augmented_cost(spec, basis, coeffs, alpha, beta, d, lam, rho) -> float:
    """``augmented_cost`` (solver.py:285-303) of a state whose coefficients are ``coeffs``."""
    diffs, lxy, lz, _, _ = _pair_state(spec, coeffs, basis)
    sb = np.sin(beta)
    target = (lxy * d * sb * np.cos(alpha), lxy * d * sb * np.sin(alpha), lz * d * np.cos(beta))
    H = basis.Pddot.T @ basis.Pddot
    total = 0.0
    for axis in range(3):
        c = coeffs[axis]
        total += 0.5 * float(np.einsum("ik,kl,il->", c, H, c))
        shifted = (diffs[axis] - target[axis]) + lam[axis] / rho
        total += 0.5 * rho * float(np.sum(shifted * shifted))
    return total


def _descent_slack(spec, basis, plan, c0, beq, geom, schedule, config, iterations, final_coeffs) -> list:
    """``descent_slack`` diagnostic (solver.py:413-421): augmented-cost change of every axis step.

    The device loop solves the three axes together (they are independent given the
    pair variables), so the diagnostic is rebuilt from prefix runs: the device state
    after k iterations (``keep_state`` with ``max_iters=k`` and the full run's
    ``switch_every``) is the reference's state entering iteration k, and the
    coefficients after k+1 iterations are that iteration's axis solutions.  Untimed,
    O(iterations^2) device iterations; the cost itself is evaluated on the host.
    """
    slack = []
    states = {}
    for k in range(1, iterations):
        out = plan.solve(c0, beq, geom, schedule.switch_every, k, config.tolerance, keep_state=True,
                         cluster_hint=_opt(config, "cluster_size", 0), fp32=_opt(config, "fp32", False))
        _, _, _, alpha, beta = _pair_state(spec, out["c"][0], basis)
        states[k] = (out["c"][0], alpha, beta, out["d"], out["lam"])
    for k in range(1, iterations):
        c_k, alpha, beta, d, lam = states[k]
        c_next = states[k + 1][0] if k + 1 < iterations else final_coeffs
        rho = schedule.values[schedule.stage_for(k)]
        mixed = c_k.copy()
        before = _augmented_cost(spec, basis, mixed, alpha, beta, d, lam, rho)
        for axis in range(3):
            mixed[axis] = c_next[axis]
            after = _augmented_cost(spec, basis, mixed, alpha, beta, d, lam, rho)
            slack.append(after - before)
            before = after
    return slack


def _make_reports(specs, out, basis, plan, cache, schedule, config, stamps, with_metrics=True,
                  foreign=None) -> list:
    """Device outputs of one launch -> one SolveReport per scenario (reference field layout).

    Whole-batch array work is done once for all scenarios: with the device report pass
    (``st_solve_report``, ``out["traj"]``) the trajectories, arc length / smoothness and the
    collision summary come from the device; otherwise (keep_state, m < 3) the trajectories
    are formed on the host as the reference does (c_axis @ P.T) and the metrics from the
    coefficients.  Single solves take the same path with B = 1, so batch and single solves
    report identical trajectories and metrics."""
    t0, t1, t2, t3 = stamps
    h2d_ms, loop_ms, d2h_ms = out["timings_ms"]
    B = len(specs)
    n = len(specs[0].start)
    nv, m = basis.num_coeffs, basis.num_samples
    c = out["c"]
    tc0 = time.perf_counter()
    if "traj" in out:
        trajs = out["traj"]
    else:
        # trajectories = c_axis @ P.T per axis (solver.py:133-136), all scenarios and axes in one product
        trajs = np.ascontiguousarray((c.reshape(-1, nv) @ basis.P.T).reshape(B, 3, n, m).transpose(0, 2, 3, 1))
    if with_metrics:
        if "min_dist" in out:
            mins, counts = out["min_dist"].tolist(), out["n_viol"].tolist()
            arc, smooth = out["arc"], out["smooth"]
        else:
            cols = metrics.collision_summary_device_batch(trajs, specs, _opt(config, "device", 0))
            mins, counts = [x[0] for x in cols], [x[1] for x in cols]
            arc, smooth = metrics.trajectory_metrics_batch_coeffs(c, basis.P)
        arc_l, smooth_l = arc.tolist(), smooth.tolist()
        # == arc.mean(axis=1) bit for bit (the same add.reduce, then one true division)
        arc_mean = (np.add.reduce(arc, axis=1) / arc.shape[1]).tolist()
        smooth_mean = (np.add.reduce(smooth, axis=1) / smooth.shape[1]).tolist()
    metrics_s = (time.perf_counter() - tc0) / B
    iters = out["iters"].tolist()
    conv = out["converged"].tolist()
    hist = out["hist"]
    common = {"assembly_s": t1 - t0, "factorization_s": t2 - t1, "loop_s": loop_ms / 1e3, "h2d_s": h2d_ms / 1e3,
              "d2h_s": d2h_ms / 1e3, "solve_call_s": t3 - t2, "metrics_s": metrics_s, "batch": B}
    loop_s = loop_ms / 1e3
    stats_obj = foreign if foreign is not None else cache
    reports = []
    for b in range(B):
        it = iters[b]
        before = cache.stats() if foreign is not None else None
        cache.count_solve(3 * it)
        _sync_foreign(cache, foreign, before)
        coeffs = c[b]
        rep_metrics = {}
        if with_metrics:
            md = mins[b]
            rep_metrics = {
                "min_normalized_distance": None if math.isinf(md) else md,
                "num_collision_violations": counts[b],
                "arc_length": arc_l[b],
                "smoothness": smooth_l[b],
                "mean_arc_length": arc_mean[b],
                "mean_smoothness": smooth_mean[b],
            }
        h0, h1, h2 = hist[b, :, :it].tolist()  # only the iterations run become Python floats
        timings = dict(common)
        timings["per_iteration_s"] = loop_s / max(1, it)
        timings["total_s"] = time.perf_counter() - t0
        diagnostics = {}
        if config.keep_state:
            spec = specs[b]
            _, lxy, lz, alpha, beta = _pair_state(spec, coeffs, basis)
            lam = out["lam"]
            stage = schedule.stage_for(it - 1)
            diagnostics["final_state"] = FinalState(
                c_x=coeffs[0].copy(), c_y=coeffs[1].copy(), c_z=coeffs[2].copy(),
                pair_vars=PairVariables(alpha=alpha, beta=beta, d=out["d"]),
                multipliers=Multipliers(lambda_x=lam[0], lambda_y=lam[1], lambda_z=lam[2]),
                rho=schedule.values[stage], stage=stage, iteration=it,
                residual_norms=list(h0), residual_max=list(h1),
                system=SystemView(spec, basis))
        reports.append(SolveReport(
            trajectories=trajs[b],
            coefficients=coeffs,
            converged=bool(conv[b]),
            iterations=it,
            residual_norm=h0[-1] if it else 0.0,
            residual_max_abs=h1[-1] if it else 0.0,
            residual_norm_history=h0,
            residual_max_history=h1,
            boundary_max_history=h2,
            timings=timings,
            metrics=rep_metrics,
            cache_stats=stats_obj.stats(),
            diagnostics=diagnostics,
        ))
    return reports


def am_solve_batch(specs, config: SolverConfig | None = None, cache: kkt.FactorCache | None = None,
                   with_metrics: bool = True) -> list:
    """Solve scenarios sharing one fingerprint in one device launch; one report each.

    The host work builds O(B) small containers (state tuples, history lists, reports) that
    the cyclic garbage collector would otherwise re-traverse many times over; none of them
    forms cycles, so collection is paused for the call (restored on exit)."""
    was_enabled = gc.isenabled()
    gc.disable()
    try:
        return _am_solve_batch(specs, config, cache, with_metrics)
    finally:
        if was_enabled:
            gc.enable()


# Large batches on the device report path run as a pipeline of contiguous chunks: while the
# device solves chunk i (enqueued by st_solve_report_begin, which returns at once), the host
# validates and packs chunk i+1 and builds the reports of chunk i-1, then waits for chunk i with
# st_solve_end.  (Libraries without the begin/end pair fall back to a worker thread that waits in
# st_solve_report.)  Every scenario's result is bitwise the one of the unchunked launch (same
# kernel and cluster shape; see tests).
PIPELINE_MIN_BATCH = 256
_POOL = None
_POOL_LOCK = __import__("threading").Lock()


def _solver_thread():
    global _POOL
    with _POOL_LOCK:
        if _POOL is None:
            from concurrent.futures import ThreadPoolExecutor
            _POOL = ThreadPoolExecutor(max_workers=1, thread_name_prefix="swarm-solve")
        return _POOL


def _pipeline_chunks(B: int) -> int:
    env = __import__("os").environ.get("SWARM_PIPE_CHUNKS")
    if env is not None:
        return max(1, min(B, int(env)))
    return 1 if B < PIPELINE_MIN_BATCH else 4


def _chunk_bounds(B: int, K: int, limit: int = 65535) -> list:
    """Chunk boundaries of a pipelined batch: the first chunk half the size of the others (the
    device starts after packing it, the later chunks are packed while the device runs), none
    larger than ``limit`` scenarios (one report-pass launch)."""
    if K <= 1:
        return [0, B]
    while True:
        w = [0.5] + [1.0] * (K - 1)
        acc = np.cumsum([0.0] + w) / sum(w)
        bounds = [int(B * x + 0.5) for x in acc]
        sizes = [b - a for a, b in zip(bounds, bounds[1:])]
        if min(sizes) < 1:
            bounds = [B * i // K for i in range(K + 1)]  # tiny batches: equal chunks
            sizes = [b - a for a, b in zip(bounds, bounds[1:])]
        if max(sizes) <= limit or K >= B:
            return bounds
        K += 1


def _prep_chunk(specs, basis, n_obs, alloc=np.empty):
    """Validation (raises before this chunk's device work) and packing of one chunk."""
    t0 = time.perf_counter()
    bnd = boundary_arrays(specs)
    # obstacle rows (centre, l_xy/2 + R, l_z/2 + R): validation prefilter, kernel geometry, collision rows
    col_obs = (np.stack([metrics._obstacle_rows(sp.geometry, sp.obstacles) for sp in specs]) if n_obs
               else np.zeros((len(specs), 0, 5)))
    if len(specs) == 1:  # the per-spec check: no batch-vectorization overhead for single solves
        v = validate_positions(specs[0], bnd[0, 0, 0], bnd[0, 1, 0], col_obs[0])
        if v:
            raise _infeasible(v)
    else:
        for v in validate_batch(specs, bnd[:, 0, 0], bnd[:, 1, 0], col_obs):
            if v:
                raise _infeasible(v)
    c0, beq, geom = pack(specs, basis, bnd, col_obs, alloc)
    col_geom = geom[:, :2]
    return t0, time.perf_counter(), c0, beq, geom, col_geom, col_obs


def _check_finite(out, offset: int = 0) -> None:
    flags = out["status"] == native.ST_NONFINITE
    if not flags.any():
        return
    bad = np.flatnonzero(flags)
    if bad.size:
        raise NonFiniteStateError(
            f"non-finite pair state (d/beta out of range) in iteration {int(out['iters'][bad[0]])} of scenario "
            f"{int(bad[0]) + offset}" + (f" and {bad.size - 1} more scenario(s)" if bad.size > 1 else ""))


def _am_solve_batch(specs, config, cache, with_metrics) -> list:
    config = config or SolverConfig()
    specs = list(specs)
    if not specs:
        return []
    if config.track_descent and len(specs) != 1:
        raise ValueError("track_descent is only available for single solves")
    _check_batch(specs)
    if config.keep_state and len(specs) != 1:
        raise ValueError("keep_state is only available for single solves")
    spec0 = specs[0]
    n, n_obs = len(spec0.start), len(spec0.obstacles)
    basis = poly.for_spec(spec0)
    # the device report pass: one warp's (m x 3) positions in shared memory (m <= 2000 here), one
    # launch covers at most 65535 scenarios (grid y of the collision rows)
    report_path = (not config.keep_state and 3 <= basis.num_samples <= 2000 and native.load().swarm_has_report)
    B = len(specs)
    K = max(_pipeline_chunks(B), -(-B // 65535)) if report_path else 1
    bounds = _chunk_bounds(B, K)
    K = len(bounds) - 1
    # the pipelined path enqueues each chunk and returns (st_solve_report_begin): its inputs are
    # packed straight into page-locked buffers so the copies run asynchronously
    pipelined = K > 1 and native.load().swarm_has_async
    alloc = native.pinned_empty if pipelined else np.empty
    prep = _prep_chunk(specs[: bounds[1]], basis, n_obs, alloc)
    fp = kkt.fingerprint(basis, n, n_obs)
    cache, foreign = _resolve_cache(cache)
    schedule = config.schedule()
    before = cache.stats()
    plan = _plan_for(cache, fp, basis, schedule, n, n_obs, _opt(config, "device", 0))
    _sync_foreign(cache, foreign, before)
    hint, fp32 = _opt(config, "cluster_size", 0), _opt(config, "fp32", False)

    def solve(pr):
        _, _, c0, beq, geom, col_geom, col_obs = pr
        t2 = time.perf_counter()
        if report_path:
            # one call: solve + trajectories (+ arc length / smoothness, collision summary) on the device
            out = plan.solve_report(c0, beq, geom, schedule.switch_every, config.max_iters, config.tolerance,
                                    col_geom, col_obs, cluster_hint=hint, fp32=fp32, with_metrics=with_metrics)
        else:
            out = plan.solve(c0, beq, geom, schedule.switch_every, config.max_iters, config.tolerance,
                             keep_state=config.keep_state, cluster_hint=hint, fp32=fp32)
        return out, t2, time.perf_counter()

    def finish(i, pr, res):
        out, t2, t3 = res
        _check_finite(out, bounds[i])
        return _make_reports(specs[bounds[i]: bounds[i + 1]], out, basis, plan, cache, schedule, config,
                             (pr[0], pr[1], t2, t3), with_metrics, foreign=foreign)

    def begin(pr):
        _, _, c0, beq, geom, col_geom, col_obs = pr
        t2 = time.perf_counter()
        pend = plan.solve_report_begin(c0, beq, geom, schedule.switch_every, config.max_iters, config.tolerance,
                                       col_geom, col_obs, cluster_hint=hint, fp32=fp32, with_metrics=with_metrics)
        return pend, t2

    def end(started):
        pend, t2 = started
        out = pend.end()
        return out, t2, time.perf_counter()

    if K == 1:
        res = solve(prep)
        reports = finish(0, prep, res)
    elif pipelined:
        # the device solves chunk i while this thread packs chunk i+1 and builds the reports of
        # chunk i-1: the library enqueues a chunk and returns (st_solve_report_begin), and
        # st_solve_end waits for it, so no Python thread has to win the GIL back to keep the
        # device fed
        reports = []
        started = begin(prep)
        for i in range(1, K):
            try:
                nxt = _prep_chunk(specs[bounds[i]: bounds[i + 1]], basis, n_obs, alloc)
            except BaseException:
                end(started)  # no solve left pending on the plan when the error propagates
                raise
            res = end(started)
            started = begin(nxt)
            try:
                reports += finish(i - 1, prep, res)
            except BaseException:
                end(started)
                raise
            prep = nxt
        reports += finish(K - 1, prep, end(started))
    else:
        pool = _solver_thread()
        reports = []
        fut = pool.submit(solve, prep)
        for i in range(1, K):
            try:
                nxt = _prep_chunk(specs[bounds[i]: bounds[i + 1]], basis, n_obs)
            except BaseException:
                fut.result()  # no solve left running on the plan when the error propagates
                raise
            res = fut.result()
            fut = pool.submit(solve, nxt)
            try:
                reports += finish(i - 1, prep, res)
            except BaseException:
                fut.result()
                raise
            prep = nxt
        reports += finish(K - 1, prep, fut.result())
    if config.track_descent:
        _, _, c0, beq, geom, _, _ = prep
        reports[0].diagnostics["descent_slack"] = _descent_slack(
            spec0, basis, plan, c0, beq, geom, schedule, config, reports[0].iterations, reports[0].coefficients)
    log.info("batch of %d solved on device in %d launch(es)", B, K)
    return reports


def am_solve(spec, config: SolverConfig | None = None, cache: kkt.FactorCache | None = None) -> SolveReport:
    """Run the AM loop end to end on the GPU (reference solver.py:363-494).

    Raises:
        InfeasibleProblemError: if the instance fails validation.
    """
    return am_solve_batch([spec], config, cache)[0]
