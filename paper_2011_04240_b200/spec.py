"""Problem description consumed by the drop-in ``am_solve``.

Mirrors the reference's instance types so a caller can hand either a
``swarmtraj.ProblemSpec`` or one of these to :func:`am_solve`; both are read
through the same attribute names (start/goal/geometry/obstacles/num_samples/
degree/duration/basis_kind).  Field meanings, defaults and validation rules
follow reference ``pkg/src/swarmtraj/problem.py``:

* ``AgentGeometry``  -> problem.py:36-60 (pairwise spheroid semi-axes, sphere mode l = 2r)
* ``BoundaryState``  -> problem.py:63-83 (pos/vel/acc pinned at one endpoint)
* ``Obstacle``       -> problem.py:86-96 (circumscribing sphere)
* ``ProblemSpec``    -> problem.py:99-141 (agent-obstacle semi-axes l/2 + R)
* ``validate``       -> problem.py:162-194 (normalized separation >= 1 at both ends)
* JSON schema        -> problem.py:460-553
"""

from __future__ import annotations

import enum
import functools
import json
import math

import numpy as np
import os
from dataclasses import dataclass

DEFAULT_NUM_SAMPLES = 100
DEFAULT_DEGREE = 10
DEFAULT_DURATION = 10.0


class BasisKind(str, enum.Enum):
    """Polynomial family of the per-axis trajectory (reference basis.py:23-27)."""

    BERNSTEIN = "bernstein"
    MONOMIAL = "monomial"


def _vec3(name, value):
    vec = tuple(float(v) for v in value)
    if len(vec) != 3 or not all(math.isfinite(v) for v in vec):
        raise ValueError(f"{name} must be a finite 3-vector, got {value}")
    return vec


@dataclass(frozen=True)
class AgentGeometry:
    l_xy: float
    l_z: float

    def __post_init__(self):
        if not (self.l_xy > 0 and self.l_z > 0):
            raise ValueError(f"spheroid semi-axes must be positive, got ({self.l_xy}, {self.l_z})")

    @property
    def is_sphere(self) -> bool:
        return self.l_xy == self.l_z

    @property
    def agent_radius(self) -> float:
        return self.l_xy / 2.0

    @classmethod
    def sphere_from_radius(cls, radius: float) -> "AgentGeometry":
        if not radius > 0:
            raise ValueError(f"agent radius must be positive, got {radius}")
        return cls(l_xy=2.0 * radius, l_z=2.0 * radius)


@dataclass(frozen=True)
class BoundaryState:
    position: tuple
    velocity: tuple = (0.0, 0.0, 0.0)
    acceleration: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        object.__setattr__(self, "position", _vec3("position", self.position))
        object.__setattr__(self, "velocity", _vec3("velocity", self.velocity))
        object.__setattr__(self, "acceleration", _vec3("acceleration", self.acceleration))

    @classmethod
    def at_rest(cls, position) -> "BoundaryState":
        return cls(position=tuple(position))


@dataclass(frozen=True)
class Obstacle:
    center: tuple
    radius: float

    def __post_init__(self):
        if not self.radius > 0:
            raise ValueError(f"obstacle radius must be positive, got {self.radius}")
        object.__setattr__(self, "center", tuple(float(v) for v in self.center))


@dataclass(frozen=True)
class ProblemSpec:
    start: tuple
    goal: tuple
    geometry: AgentGeometry
    obstacles: tuple = ()
    num_samples: int = DEFAULT_NUM_SAMPLES
    degree: int = DEFAULT_DEGREE
    duration: float = DEFAULT_DURATION
    basis_kind: BasisKind = BasisKind.BERNSTEIN
    seed: int | None = None

    def __post_init__(self):
        if len(self.start) < 1:
            raise ValueError("at least one agent is required")
        if len(self.start) != len(self.goal):
            raise ValueError(
                f"start and goal lists must have equal length, got {len(self.start)} vs {len(self.goal)}"
            )
        object.__setattr__(self, "start", tuple(self.start))
        object.__setattr__(self, "goal", tuple(self.goal))
        object.__setattr__(self, "obstacles", tuple(self.obstacles))
        object.__setattr__(self, "basis_kind", BasisKind(self.basis_kind))

    @property
    def num_agents(self) -> int:
        return len(self.start)

    @property
    def num_obstacles(self) -> int:
        return len(self.obstacles)

    def obstacle_geometry(self, obstacle) -> AgentGeometry:
        return AgentGeometry(l_xy=self.geometry.l_xy / 2.0 + obstacle.radius,
                             l_z=self.geometry.l_z / 2.0 + obstacle.radius)


@dataclass(frozen=True)
class Violation:
    subject: str
    detail: str

    def __str__(self) -> str:
        return f"{self.subject}: {self.detail}"


def _separation(p, q, l_xy, l_z) -> float:
    return math.sqrt(((p[0] - q[0]) / l_xy) ** 2 + ((p[1] - q[1]) / l_xy) ** 2 + ((p[2] - q[2]) / l_z) ** 2)


def obstacle_axes(spec, obstacle) -> tuple[float, float]:
    """Agent-vs-obstacle semi-axes l/2 + R (problem.py:136-141); works on any spec duck type."""
    return spec.geometry.l_xy / 2.0 + obstacle.radius, spec.geometry.l_z / 2.0 + obstacle.radius


@functools.lru_cache(maxsize=16)
def _pairs(n):
    ii, jj = np.triu_indices(n, k=1)
    ii.setflags(write=False)
    jj.setflags(write=False)
    return ii, jj


def _near_pairs(P, l_xy, l_z):
    """Vectorized prefilter: agent pairs (i<j, lexicographic) whose separation may be < 1."""
    ii, jj = _pairs(P.shape[0])
    d = (P[ii] - P[jj]) * np.array([1.0 / l_xy, 1.0 / l_xy, 1.0 / l_z])
    keep = np.einsum("pk,pk->p", d, d) < (1.0 + 1e-9) ** 2
    return zip(ii[keep].tolist(), jj[keep].tolist())


def validate(spec) -> list[Violation]:
    """Every start/goal separation violation (reference problem.py:162-194).

    Same violations, order and text as the reference's O(n^2) scalar loop; a
    vectorized prefilter picks the candidate pairs and the reference's scalar
    expression decides each one, so the O(n^2) part costs no Python per pair.
    """
    out: list[Violation] = []
    g = spec.geometry
    n = len(spec.start)
    for label, states in (("start", spec.start), ("goal", spec.goal)):
        pos = [s.position for s in states]
        if n > 1:
            P = np.asarray(pos, dtype=float).reshape(n, 3)
            for i, j in _near_pairs(P, g.l_xy, g.l_z):
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


def _obstacle_candidates(P, obs_rows):
    """(..., n, 3) positions x (..., k, 5) obstacle rows (centre, l_xy/2 + R, l_z/2 + R) -> (..., n, k)
    mask of the (agent, obstacle) pairs whose normalized separation may be < 1 (loose prefilter)."""
    d = P[..., :, None, :] - obs_rows[..., None, :, :3]
    d[..., :2] /= obs_rows[..., None, :, 3:4]
    d[..., 2] /= obs_rows[..., None, :, 4]
    return np.einsum("...c,...c->...", d, d) < (1.0 + 1e-9) ** 2


def validate_positions(spec, start_pos: np.ndarray, goal_pos: np.ndarray, obs_rows=None) -> list[Violation]:
    """``validate`` of one spec from its (n, 3) start / goal position arrays (``engine.boundary_arrays``)
    and, with obstacles, its (k, 5) obstacle rows: the same violations, order and text; one vectorized
    prefilter over both endpoints, the reference's scalar expression on each candidate."""
    out: list[Violation] = []
    g = spec.geometry
    n = start_pos.shape[0]
    P2 = np.stack([start_pos, goal_pos])
    near = None
    if n > 1:
        ii, jj = _pairs(n)
        d = (P2[:, ii] - P2[:, jj]) * np.array([1.0 / g.l_xy, 1.0 / g.l_xy, 1.0 / g.l_z])
        near = np.einsum("spk,spk->sp", d, d) < (1.0 + 1e-9) ** 2
        if not near.any():
            near = None
    near_o = None
    if spec.obstacles:
        if obs_rows is None:
            obs_rows = np.array([[*o.center, *obstacle_axes(spec, o)] for o in spec.obstacles], dtype=float)
        near_o = _obstacle_candidates(P2, obs_rows)
        if not near_o.any():
            near_o = None
    if near is None and near_o is None:
        return out
    for side, label in enumerate(("start", "goal")):
        P = P2[side]
        if near is not None:
            for p in np.flatnonzero(near[side]).tolist():
                i, j = int(ii[p]), int(jj[p])
                sep = _separation(P[i].tolist(), P[j].tolist(), g.l_xy, g.l_z)
                if sep < 1.0:
                    out.append(Violation(f"{label} pair ({i}, {j})", f"normalized separation {sep:.4f} < 1"))
        if near_o is not None:
            for i, k in zip(*np.nonzero(near_o[side])):
                obs = spec.obstacles[k]
                lxy, lz = obstacle_axes(spec, obs)
                sep = _separation(P[i].tolist(), obs.center, lxy, lz)
                if sep < 1.0:
                    out.append(Violation(f"{label} agent {int(i)} vs obstacle {int(k)}",
                                         f"normalized separation {sep:.4f} < 1"))
    return out


def validate_batch(specs, start_pos: np.ndarray, goal_pos: np.ndarray, obs_rows=None) -> list:
    """``validate`` of B same-shape specs at once: the same violations, order and text per spec.

    start_pos / goal_pos: (B, n, 3) positions (``engine.boundary_arrays``); obs_rows: (B, k, 5)
    obstacle rows (centre, l_xy/2 + R, l_z/2 + R), built here when omitted.  One vectorized
    prefilter over every pair and every (agent, obstacle) row of every spec; only candidates run
    the scalar expression.
    """
    B = len(specs)
    out = [[] for _ in range(B)]
    if B == 0:
        return out
    n = start_pos.shape[1]
    geo = np.array([(s.geometry.l_xy, s.geometry.l_z) for s in specs], dtype=float)
    scale = np.stack([1.0 / geo[:, 0], 1.0 / geo[:, 0], 1.0 / geo[:, 1]], axis=1)[:, None, :]
    upper = np.triu(np.ones((n, n), dtype=bool), 1)
    cand = {}
    for label, P in (("start", start_pos), ("goal", goal_pos)):
        if n < 2:
            continue
        # |pi - pj|^2 = |pi|^2 + |pj|^2 - 2 pi.pj on the scaled positions (batched matmul, in place,
        # over cache-sized slices of the batch); a loose prefilter -- every candidate is re-checked
        # with the exact scalar expression.  np.nonzero walks (b, i, j) in the pair order i < j.
        step = max(1, (1 << 18) // (n * n))
        for b0 in range(0, B, step):
            Ps = P[b0: b0 + step] * scale[b0: b0 + step]
            sq = np.einsum("bnk,bnk->bn", Ps, Ps)
            d2 = np.matmul(Ps, Ps.transpose(0, 2, 1))
            d2 *= -2.0
            tol = sq * (1.0 - 1e-6)  # d2 < 1 + 1e-6 (1 + sq_i + sq_j)
            d2 += tol[:, :, None]
            d2 += tol[:, None, :]
            near = d2 < 1.0 + 1e-6
            near &= upper
            if not near.any():
                continue
            for b, i, j in zip(*np.nonzero(near)):
                cand.setdefault(int(b) + b0, []).append((label, 0, int(i), int(j)))
    k_obs = len(specs[0].obstacles)
    if k_obs:
        if obs_rows is None:
            obs_rows = np.array([[[*o.center, *obstacle_axes(s, o)] for o in s.obstacles] for s in specs],
                                dtype=float)
        step = max(1, (1 << 18) // (n * k_obs))
        for label, P in (("start", start_pos), ("goal", goal_pos)):
            for b0 in range(0, B, step):
                near_o = _obstacle_candidates(P[b0: b0 + step], obs_rows[b0: b0 + step])
                if not near_o.any():
                    continue
                for b, i, k in zip(*np.nonzero(near_o)):  # (b, i, k) in the reference's loop order
                    cand.setdefault(int(b) + b0, []).append((label, 1, int(i), int(k)))
    for b, entries in cand.items():
        spec = specs[b]
        g = spec.geometry
        for label, P in (("start", start_pos), ("goal", goal_pos)):
            for lab, kind, i, j in entries:  # per label: pairs first, then (agent, obstacle) rows
                if lab != label or kind != 0:
                    continue
                sep = _separation(P[b, i], P[b, j], g.l_xy, g.l_z)
                if sep < 1.0:
                    out[b].append(Violation(f"{label} pair ({i}, {j})", f"normalized separation {sep:.4f} < 1"))
            for lab, kind, i, k in entries:
                if lab != label or kind != 1:
                    continue
                obs = spec.obstacles[k]
                lxy, lz = obstacle_axes(spec, obs)
                sep = _separation(P[b, i], obs.center, lxy, lz)
                if sep < 1.0:
                    out[b].append(Violation(f"{label} agent {i} vs obstacle {k}",
                                            f"normalized separation {sep:.4f} < 1"))
    return out


# --- scenario JSON (reference problem.py:460-553) ---------------------------------------------


def spec_to_dict(spec) -> dict:
    doc = {"n": len(spec.start), "duration": spec.duration, "m": spec.num_samples,
           "degree": spec.degree, "basis": BasisKind(spec.basis_kind).value}
    if spec.geometry.l_xy == spec.geometry.l_z:
        doc["radius"] = spec.geometry.l_xy / 2.0
    else:
        doc["l_xy"], doc["l_z"] = spec.geometry.l_xy, spec.geometry.l_z
    for key, states in (("start", spec.start), ("goal", spec.goal)):
        doc[key] = [{"position": list(s.position), "velocity": list(s.velocity),
                     "acceleration": list(s.acceleration)} for s in states]
    doc["obstacles"] = [{"center": list(o.center), "radius": o.radius} for o in spec.obstacles]
    if getattr(spec, "seed", None) is not None:
        doc["seed"] = spec.seed
    return doc


def _state(obj) -> BoundaryState:
    if isinstance(obj, dict):
        return BoundaryState(position=tuple(obj["position"]),
                             velocity=tuple(obj.get("velocity", (0.0, 0.0, 0.0))),
                             acceleration=tuple(obj.get("acceleration", (0.0, 0.0, 0.0))))
    return BoundaryState.at_rest(tuple(obj))


def spec_from_dict(doc: dict) -> ProblemSpec:
    try:
        start = tuple(_state(s) for s in doc["start"])
        goal = tuple(_state(g) for g in doc["goal"])
    except (KeyError, TypeError, IndexError) as exc:
        raise ValueError(f"malformed scenario document: {exc}") from exc
    if "radius" in doc:
        geometry = AgentGeometry.sphere_from_radius(float(doc["radius"]))
    elif "l_xy" in doc and "l_z" in doc:
        geometry = AgentGeometry(l_xy=float(doc["l_xy"]), l_z=float(doc["l_z"]))
    else:
        raise ValueError("scenario must provide either 'radius' or both 'l_xy' and 'l_z'")
    if int(doc.get("n", len(start))) != len(start):
        raise ValueError(f"scenario field n={doc['n']} disagrees with {len(start)} start states")
    obstacles = tuple(Obstacle(center=tuple(o["center"]), radius=float(o["radius"]))
                      for o in doc.get("obstacles", []))
    return ProblemSpec(start=start, goal=goal, geometry=geometry, obstacles=obstacles,
                       num_samples=int(doc.get("m", DEFAULT_NUM_SAMPLES)),
                       degree=int(doc.get("degree", DEFAULT_DEGREE)),
                       duration=float(doc.get("duration", DEFAULT_DURATION)),
                       basis_kind=BasisKind(doc.get("basis", "bernstein")), seed=doc.get("seed"))


def save_scenario(spec, path: str | os.PathLike) -> None:
    with open(path, "w") as fh:
        json.dump(spec_to_dict(spec), fh, indent=2)
        fh.write("\n")


def load_scenario(path: str | os.PathLike) -> ProblemSpec:
    with open(path) as fh:
        return spec_from_dict(json.load(fh))
