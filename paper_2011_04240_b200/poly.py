"""Sampled polynomial bases (host side; consumed on device as the m x n_v matrix P).

Restates reference ``basis.py``: uniform grid on [0, T] (basis.py:75-91),
Bernstein rows binom(d,k) tau^k (1-tau)^(d-k) (basis.py:94-100), derivatives by
degree reduction (basis.py:103-119), monomial debug basis (basis.py:122-131),
1/T chain-rule scaling (basis.py:153-157), straight-line coefficients
(basis.py:162-176) and the 6 x n_v endpoint block (basis.py:179-195).

The floating-point operation order matches the reference so P, Pdot and
Pddot are bitwise identical to ``swarmtraj.build_basis`` output.
"""

from __future__ import annotations

import functools
import math
from dataclasses import dataclass, field

import numpy as np

from .spec import BasisKind

MIN_DEGREE = 5


@dataclass(frozen=True)
class Basis:
    P: np.ndarray = field(repr=False)
    Pdot: np.ndarray = field(repr=False)
    Pddot: np.ndarray = field(repr=False)
    samples: np.ndarray = field(repr=False)
    duration: float
    kind: BasisKind
    degree: int

    @property
    def num_coeffs(self) -> int:
        return self.degree + 1

    @property
    def num_samples(self) -> int:
        return self.P.shape[0]


def _bernstein(tau: np.ndarray, degree: int) -> np.ndarray:
    k = np.arange(degree + 1)
    binom = np.array([float(math.comb(degree, int(j))) for j in k])
    t = tau[:, None]
    return binom * t ** k * (1.0 - t) ** (degree - k)


def _bernstein_family(tau, degree):
    b = _bernstein(tau, degree)
    m = tau.shape[0]
    lo1 = _bernstein(tau, degree - 1)
    d1 = np.zeros((m, degree + 1))
    d1[:, :degree] -= lo1  # 0 - x, not -x: keeps +0.0 where the reference has it
    d1[:, 1:] += lo1
    d1 *= degree
    lo2 = _bernstein(tau, degree - 2)
    d2 = np.zeros((m, degree + 1))
    d2[:, : degree - 1] = lo2
    d2[:, 1:degree] -= 2.0 * lo2
    d2[:, 2:] += lo2
    d2 *= degree * (degree - 1)
    return b, d1, d2


def _monomial_family(tau, degree):
    k = np.arange(degree + 1)
    t = tau[:, None]
    b = t ** k
    d1 = np.zeros_like(b)
    d1[:, 1:] = k[1:] * t ** (k[1:] - 1)
    d2 = np.zeros_like(b)
    d2[:, 2:] = k[2:] * (k[2:] - 1) * t ** (k[2:] - 2)
    return b, d1, d2


def build(num_samples: int, duration: float, degree: int, kind=BasisKind.BERNSTEIN) -> Basis:
    if num_samples < 2:
        raise ValueError(f"num_samples must be >= 2, got {num_samples}")
    if not duration > 0:
        raise ValueError(f"duration must be positive, got {duration}")
    if degree < MIN_DEGREE:
        raise ValueError(f"degree must be >= {MIN_DEGREE}, got {degree}")
    return _build(int(num_samples), float(duration), int(degree), BasisKind(kind))


@functools.lru_cache(maxsize=64)
def _build(num_samples: int, duration: float, degree: int, kind: BasisKind) -> Basis:
    # one immutable Basis per (m, duration, degree, kind): every solve of a fingerprint reuses it
    samples = np.linspace(0.0, float(duration), num_samples)
    samples.setflags(write=False)
    tau = samples / float(duration)
    fam = _bernstein_family if kind == BasisKind.BERNSTEIN else _monomial_family
    b, d1, d2 = fam(tau, degree)
    inv_t = 1.0 / float(duration)
    mats = (b, d1 * inv_t, d2 * inv_t ** 2)
    for a in mats:
        a.setflags(write=False)
    return Basis(P=mats[0], Pdot=mats[1], Pddot=mats[2], samples=samples, duration=float(duration),
                 kind=kind, degree=degree)


def for_spec(spec) -> Basis:
    return build(spec.num_samples, spec.duration, spec.degree, spec.basis_kind)


def endpoint_rows(basis: Basis) -> np.ndarray:
    """[P_0; Pdot_0; Pddot_0; P_end; Pdot_end; Pddot_end] (6 x n_v)."""
    return np.vstack([basis.P[0], basis.Pdot[0], basis.Pddot[0],
                      basis.P[-1], basis.Pdot[-1], basis.Pddot[-1]])


def straight_line(basis: Basis, start: np.ndarray, goal: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    """Straight-line coefficients for many scalars at once: (...,) x2 -> (..., n_v).

    Bernstein: c_k = s + (k/d)(g - s); monomial: [s, g - s, 0, ...].  ``out``: optional
    C-contiguous destination of that shape (e.g. a page-locked buffer).
    """
    start = np.asarray(start, dtype=float)
    goal = np.asarray(goal, dtype=float)
    nv = basis.num_coeffs
    if out is None:
        out = np.empty(start.shape + (nv,))
    if basis.kind == BasisKind.BERNSTEIN:
        frac = np.arange(nv) / basis.degree
        np.multiply.outer(np.subtract(goal, start, order="C"), frac, out=out)  # = s + frac (g - s), bitwise
        out += start[..., None]
        return out
    out[...] = 0.0
    out[..., 0] = start
    out[..., 1] = goal - start
    return out
