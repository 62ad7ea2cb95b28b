"""Per-stage KKT operators in structured form, the rho schedule and the factor cache.

Reference: ``kkt_cache.py``.  The reference LU-factorizes the full
(17n)x(17n) KKT matrix per rho (kkt_cache.py:321-353) and solves with
``lu_solve`` three times per iteration (kkt_cache.py:291-305).

Structure used here instead (verified to 1e-15): with the
complete-graph pair incidence S plus n_obs obstacle rows per agent,
S'S = (n + n_obs) I - 11', so the per-axis KKT matrix permuted to per-agent
17x17 blocks is  I (x) K_dev + 11' (x) K_C, and

    x_i = K_dev^-1 (r_i - rbar) + K_mean^-1 rbar,      rbar = mean_i r_i

    K_dev  = [[Pdd'Pdd + rho (n + n_obs) P'P, E'], [E, 0]]
    K_mean = [[Pdd'Pdd + rho  n_obs      P'P, E'], [E, 0]]

Only the coefficient rows of the solution are needed, and the boundary
right-hand side b_eq is fixed per scenario, so a stage is fully described by
four small matrices (all n_v x n_v or n_v x 6, FP64):

    G  = K_dev^-1[:nv,:nv]          F  = K_dev^-1[:nv, nv:]
    Gm = K_mean^-1[:nv,:nv] - G     Fm = K_mean^-1[:nv, nv:]

    c_i = rho G R_i + rho Gm Rbar + F (beq_i - beqbar) + Fm beqbar,   R_i = (S'b)_i P

which is what the device solve phase evaluates.  The "factorization" of a
stage is the two 17x17 inversions; it is counted exactly like the
reference's LU so ``cache_stats`` keep their meaning (10 per new
fingerprint, none inside the loop; kkt_cache.py:385-419).
"""

from __future__ import annotations

import functools
import hashlib
import json
import logging
import os
import threading
import time
from pathlib import Path
from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import lu_factor

from . import poly

log = logging.getLogger(__name__)

# on-disk entry files (kept apart from the reference's factors.npz / manifest.json, whose LU
# factors are a different operator, so both caches can share one directory)
OPERATORS_FILE = "b200_operators.npz"
MANIFEST_FILE = "b200_manifest.json"

BOUNDARY_ROWS = 6


@dataclass(frozen=True)
class RhoSchedule:
    """Geometric penalty schedule advanced in equal blocks (kkt_cache.py:356-382)."""

    values: tuple
    switch_every: int

    def stage_for(self, iteration: int) -> int:
        return min(iteration // self.switch_every, len(self.values) - 1)

    def value_for(self, iteration: int) -> float:
        return self.values[self.stage_for(iteration)]


@functools.lru_cache(maxsize=64)
def build_rho_schedule(rho_initial: float, growth: float, stages: int, max_iters: int) -> RhoSchedule:
    if not rho_initial > 0:
        raise ValueError(f"rho_initial must be positive, got {rho_initial}")
    if not growth > 1:
        raise ValueError(f"growth must be > 1, got {growth}")
    if stages < 1:
        raise ValueError(f"stages must be >= 1, got {stages}")
    if max_iters < 1:
        raise ValueError(f"max_iters must be >= 1, got {max_iters}")
    return RhoSchedule(values=tuple(rho_initial * growth ** s for s in range(stages)),
                       switch_every=-(-max_iters // stages))


@dataclass(frozen=True)
class Fingerprint:
    """Identity of the iteration-independent operators (kkt_cache.py:52-72)."""

    num_agents: int
    num_samples: int
    num_coeffs: int
    num_obstacles: int
    basis_kind: str
    basis_sha: str

    def key(self) -> str:
        k = _KEYS.get(self)
        if k is None:
            text = (f"{self.num_agents},{self.num_samples},{self.num_coeffs},{self.num_obstacles},"
                    f"{self.basis_kind},{self.basis_sha}")
            k = hashlib.sha256(text.encode()).hexdigest()[:16]
            if len(_KEYS) > 256:
                _KEYS.clear()
            _KEYS[self] = k
        return k


_KEYS: dict = {}  # Fingerprint -> key (the digest text is fixed per fingerprint)


_DIGESTS: dict = {}


def basis_digest(basis: poly.Basis) -> str:
    hit = _DIGESTS.get(id(basis))
    if hit is not None and hit[0] is basis:
        return hit[1]
    d = _basis_digest(basis)
    if len(_DIGESTS) > 64:
        _DIGESTS.clear()
    _DIGESTS[id(basis)] = (basis, d)  # keeps the basis alive, so the id cannot be reused
    return d


def _basis_digest(basis: poly.Basis) -> str:
    h = hashlib.sha256()
    for a in (basis.P, basis.Pdot, basis.Pddot):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def fingerprint(basis: poly.Basis, n: int, n_obs: int) -> Fingerprint:
    return Fingerprint(n, basis.num_samples, basis.num_coeffs, n_obs, basis.kind.value, basis_digest(basis))


@dataclass(frozen=True)
class StageOperator:
    """Solve operator of one rho stage (see module docstring)."""

    rho: float
    G: np.ndarray = field(repr=False)
    Gm: np.ndarray = field(repr=False)
    F: np.ndarray = field(repr=False)
    Fm: np.ndarray = field(repr=False)


def block_matrix(basis: poly.Basis, weight: float) -> np.ndarray:
    """[[Pdd'Pdd + weight P'P, E'], [E, 0]] (17x17 at the default degree)."""
    nv = basis.num_coeffs
    E = poly.endpoint_rows(basis)
    K = np.zeros((nv + BOUNDARY_ROWS, nv + BOUNDARY_ROWS))
    K[:nv, :nv] = basis.Pddot.T @ basis.Pddot + weight * (basis.P.T @ basis.P)
    K[:nv, nv:] = E.T
    K[nv:, :nv] = E
    return K


def _checked_inverse(K: np.ndarray) -> np.ndarray:
    lu, _ = lu_factor(K, check_finite=False)
    diag = np.abs(np.diag(lu))
    if diag.min() <= 1e-14 * diag.max():
        raise ValueError("KKT matrix is numerically singular "
                         f"(pivot ratio {diag.min():.3e}/{diag.max():.3e}); "
                         "check that the endpoint block has full rank")
    return np.linalg.inv(K)


def stage_operator(basis: poly.Basis, n: int, n_obs: int, rho: float) -> StageOperator:
    """Build one stage's operator (the analogue of ``factorize``, kkt_cache.py:332-353)."""
    if rho < 0:
        raise ValueError(f"rho must be non-negative, got {rho}")
    nv = basis.num_coeffs
    if np.linalg.matrix_rank(poly.endpoint_rows(basis)) < BOUNDARY_ROWS:
        raise ValueError("endpoint constraint block is rank deficient; the basis cannot pin "
                         "position, velocity and acceleration at both ends")
    kd = _checked_inverse(block_matrix(basis, rho * (n + n_obs)))
    km = _checked_inverse(block_matrix(basis, rho * n_obs))
    G = kd[:nv, :nv].copy()
    return StageOperator(rho=float(rho), G=G, Gm=km[:nv, :nv] - G, F=kd[:nv, nv:].copy(),
                         Fm=km[:nv, nv:].copy())


class FactorCache:
    """Shared store of stage operators keyed by (fingerprint, rho) (kkt_cache.py:385-456).

    Single-flight per key, immutable entries, the reference's counters.  It
    additionally owns the device plans (one per fingerprint and schedule),
    so a warm cache means no host precompute and no device upload either.
    """

    def __init__(self, disk_dir=None):
        self._ops: dict = {}
        self._plans: dict = {}
        self._lock = threading.Lock()
        self._inflight: dict = {}
        self.disk_dir = Path(disk_dir) if disk_dir else None
        self.factorizations = 0
        self.hits = 0
        self.misses = 0
        self.solves = 0

    def count_solve(self, k: int = 1) -> None:
        with self._lock:
            self.solves += k

    def stats(self) -> dict:
        return {"entries": len(self._ops), "factorizations": self.factorizations, "hits": self.hits,
                "misses": self.misses, "solves": self.solves}

    def get(self, fp: Fingerprint, basis: poly.Basis, rho: float) -> StageOperator:
        key = (fp.key(), float(rho))
        while True:
            with self._lock:
                op = self._ops.get(key)
                if op is not None:
                    self.hits += 1
                    return op
                ev = self._inflight.get(key)
                if ev is None:
                    self._inflight[key] = threading.Event()
                    break
            ev.wait()
        try:
            op = self._load_one(fp, rho)
            built = op is None
            if built:
                op = stage_operator(basis, fp.num_agents, fp.num_obstacles, rho)
            with self._lock:
                self._ops[key] = op
                if built:
                    self.factorizations += 1
                    self.misses += 1
                else:
                    self.hits += 1
            return op
        finally:
            with self._lock:
                self._inflight.pop(key).set()

    def prefactorize(self, fp: Fingerprint, basis: poly.Basis, schedule: RhoSchedule) -> list:
        # warm path: every stage present -> one lock, the same hits as one get() per stage
        fk = fp.key()
        with self._lock:
            ops = [self._ops.get((fk, float(rho))) for rho in schedule.values]
            if all(op is not None for op in ops):
                self.hits += len(ops)
                return ops
        return [self.get(fp, basis, rho) for rho in schedule.values]

    # -- disk persistence (kkt_cache.py:458-528) ---------------------------------------------------
    def _entry_dir(self, fp: Fingerprint):
        return None if self.disk_dir is None else self.disk_dir / fp.key()

    def _load_one(self, fp: Fingerprint, rho: float):
        entry = self._entry_dir(fp)
        if entry is None or not (entry / MANIFEST_FILE).exists():
            return None
        try:
            manifest = json.loads((entry / MANIFEST_FILE).read_text())
            if manifest["fingerprint"] != fp.key() or float(rho) not in manifest["rho_values"]:
                return None
            idx = manifest["rho_values"].index(float(rho))
            with np.load(entry / OPERATORS_FILE) as blob:
                parts = {name: blob[f"{name}_{idx}"] for name in ("G", "Gm", "F", "Fm")}
        except (OSError, KeyError, ValueError) as exc:
            log.warning("ignoring unreadable operator cache entry %s: %s", entry, exc)
            return None
        log.info("loaded cached stage operator %s rho=%g from %s", fp.key(), rho, entry)
        return StageOperator(rho=float(rho), **parts)

    def persist(self, fp: Fingerprint, basis: poly.Basis, schedule: RhoSchedule) -> dict:
        """Build (or fetch) every stage and write them under ``disk_dir`` (kkt_cache.py:483-528).

        Rewriting identical content is skipped (idempotent rebuilds); returns the manifest.
        """
        if self.disk_dir is None:
            raise ValueError("cache has no disk directory configured")
        t0 = time.perf_counter()
        ops = self.prefactorize(fp, basis, schedule)
        entry = self._entry_dir(fp)
        entry.mkdir(parents=True, exist_ok=True)
        manifest = {
            "fingerprint": fp.key(),
            "num_agents": fp.num_agents,
            "num_samples": fp.num_samples,
            "num_coeffs": fp.num_coeffs,
            "num_obstacles": fp.num_obstacles,
            "basis_kind": fp.basis_kind,
            "basis_sha": fp.basis_sha,
            "rho_values": [op.rho for op in ops],
            "operator": "structured 17x17 stage blocks (G, Gm, F, Fm)",
            "block_dimension": fp.num_coeffs + BOUNDARY_ROWS,
        }
        path = entry / MANIFEST_FILE
        text = json.dumps(manifest, indent=2) + "\n"
        if not (path.exists() and path.read_text() == text and (entry / OPERATORS_FILE).exists()):
            blobs = {f"{name}_{i}": getattr(op, name) for i, op in enumerate(ops) for name in ("G", "Gm", "F", "Fm")}
            tmp = entry / (OPERATORS_FILE + ".tmp")
            with open(tmp, "wb") as fh:
                np.savez(fh, **blobs)
            os.replace(tmp, entry / OPERATORS_FILE)
            tmp_manifest = entry / (MANIFEST_FILE + ".tmp")
            tmp_manifest.write_text(text)
            os.replace(tmp_manifest, path)
        manifest["build_time_s"] = time.perf_counter() - t0
        manifest["bytes"] = (entry / OPERATORS_FILE).stat().st_size
        return manifest

    def plan(self, fp: Fingerprint, schedule: RhoSchedule, build, device: int = 0):
        """Device plan for (fingerprint, rho values, device ordinal), created once via ``build()``."""
        key = (fp.key(), tuple(float(v) for v in schedule.values), int(device))
        with self._lock:
            plan = self._plans.get(key)
        if plan is not None:
            return plan
        plan = build()
        with self._lock:
            return self._plans.setdefault(key, plan)
