"""ORACLE -- test infrastructure only.

CPU restatement (numpy/scipy, FP64) of the reference AM solve path in
``/root/reference/pkg/src/swarmtraj``.  It is the parity checker for the CUDA
path and the "port" CPU baseline timed by ``bench.py``; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs may import it.  The product (``paper_2011_04240_b200``) never
imports or calls anything here.

Pinning: ``tests/golden/*.npz`` were produced by the *real* reference
(``tests/golden/make_golden.py``, run in the build container where the
reference is importable); ``tests/test_oracle.py`` checks this restatement
against them (coefficients within the reference's own self-noise envelope,
identical iteration counts and verdicts).

Algorithm, step by step (each cites the reference line it restates):

* basis: Bernstein/monomial sampled rows, 1/T chain rule        basis.py:94-159
* pairs: agent pairs (i<j) lexicographic, then (agent, obstacle)
  agent-major; signed incidence S, per-pair l_xy/l_z, offsets    kkt_cache.py:195-224
* KKT = [[Q + rho kron(S'S, P'P), A_eq'], [A_eq, 0]], LU          kkt_cache.py:321-353
* rho schedule rho0 g^s, switch_every = ceil(max_iters/stages)    kkt_cache.py:370-382
* init: straight lines; alpha/beta projection; d = max(1, k)      solver.py:309-352
* loop: per axis b = target - lambda/rho + offset, rhs =
  [rho S'b P; b_eq], lu_solve                                      solver.py:414-421, kkt_cache.py:291-305
  diffs = S (c P') - offsets                                       solver.py:228-236
  alpha = atan2(dy, dx), beta = atan2(hypot/l_xy, dz/l_z)          solver.py:178-195
  d = max(1, numer/denom) on g = diffs + lambda/rho                solver.py:204-215, 427-436
  r = diffs - l d trig; lambda += rho r                            solver.py:218-225, 439-442
  (||r||, max|r|), boundary max|A_eq c - b_eq|, stop at tol        solver.py:260-263, 444-457
"""

from __future__ import annotations

import math

import numpy as np
from scipy.linalg import lu_factor, lu_solve


def _bernstein(tau, deg):
    k = np.arange(deg + 1)
    binom = np.array([float(math.comb(deg, int(j))) for j in k])
    t = tau[:, None]
    return binom * t ** k * (1.0 - t) ** (deg - k)


def basis(m: int, duration: float, deg: int, kind: str = "bernstein"):
    """(P, Pdot, Pddot), basis.py:103-159."""
    tau = np.linspace(0.0, float(duration), m) / float(duration)
    if str(kind) in ("bernstein", "BasisKind.BERNSTEIN"):
        b = _bernstein(tau, deg)
        l1 = _bernstein(tau, deg - 1)
        db = np.zeros_like(b)
        db[:, :deg] -= l1
        db[:, 1:] += l1
        db *= deg
        l2 = _bernstein(tau, deg - 2)
        ddb = np.zeros_like(b)
        ddb[:, : deg - 1] += l2
        ddb[:, 1:deg] -= 2.0 * l2
        ddb[:, 2:] += l2
        ddb *= deg * (deg - 1)
    else:
        k = np.arange(deg + 1)
        t = tau[:, None]
        b = t ** k
        db = np.zeros_like(b)
        db[:, 1:] = k[1:] * t ** (k[1:] - 1)
        ddb = np.zeros_like(b)
        ddb[:, 2:] = k[2:] * (k[2:] - 1) * t ** (k[2:] - 2)
    it = 1.0 / float(duration)
    return b, db * it, ddb * it ** 2


def _kind(spec) -> str:
    return str(getattr(spec.basis_kind, "value", spec.basis_kind))


class Problem:
    """Assembled blocks of one instance (kkt_cache.py:161-235)."""

    def __init__(self, spec):
        self.spec = spec
        self.n = n = len(spec.start)
        self.kind = _kind(spec)
        self.P, self.Pd, self.Pdd = basis(spec.num_samples, spec.duration, spec.degree, self.kind)
        self.m, self.nv = self.P.shape
        E = np.vstack([self.P[0], self.Pd[0], self.Pdd[0], self.P[-1], self.Pd[-1], self.Pdd[-1]])
        self.E = E
        self.A_eq = np.kron(np.eye(n), E)
        self.b_eq = np.empty((3, 6 * n))
        for i, (s, g) in enumerate(zip(spec.start, spec.goal)):
            for a in range(3):
                self.b_eq[a, 6 * i:6 * i + 6] = (s.position[a], s.velocity[a], s.acceleration[a],
                                                 g.position[a], g.velocity[a], g.acceleration[a])
        rows, lxy, lz, off = [], [], [], []
        for i in range(n):
            for j in range(i + 1, n):
                r = np.zeros(n)
                r[i], r[j] = 1.0, -1.0
                rows.append(r)
                lxy.append(spec.geometry.l_xy)
                lz.append(spec.geometry.l_z)
                off.append((0.0, 0.0, 0.0))
        for i in range(n):
            for obs in spec.obstacles:
                r = np.zeros(n)
                r[i] = 1.0
                rows.append(r)
                lxy.append(spec.geometry.l_xy / 2.0 + obs.radius)
                lz.append(spec.geometry.l_z / 2.0 + obs.radius)
                off.append(tuple(obs.center))
        self.S = np.array(rows).reshape(len(rows), n)
        self.p = self.S.shape[0]
        self.lxy = np.array(lxy)
        self.lz = np.array(lz)
        self.off = np.array(off).reshape(self.p, 3)
        self.Q = np.kron(np.eye(n), self.Pdd.T @ self.Pdd)

    def kkt(self, rho):
        H = self.Q + rho * np.kron(self.S.T @ self.S, self.P.T @ self.P)
        nc, ne = H.shape[0], self.A_eq.shape[0]
        K = np.zeros((nc + ne, nc + ne))
        K[:nc, :nc] = H
        K[:nc, nc:] = self.A_eq.T
        K[nc:, :nc] = self.A_eq
        return K

    def diffs(self, c):
        out = np.empty((3, self.p, self.m))
        for a in range(3):
            pos = c[a] @ self.P.T
            out[a] = self.S @ pos - self.off[:, a][:, None]
        return out


def project(dx, dy, dz, lxy, lz):
    planar = np.hypot(dx, dy)
    alpha = np.arctan2(dy, dx)
    beta = np.arctan2(planar / lxy, dz / np.asarray(lz, dtype=float))
    deg = (planar == 0.0) & (dz == 0.0)
    if np.any(deg):
        beta = np.where(deg, np.pi / 2.0, beta)
    return alpha, beta


def scale(dx, dy, dz, lxy, lz):
    return np.hypot(np.hypot(dx, dy) / lxy, dz / np.asarray(lz, dtype=float))


def d_step(gx, gy, gz, alpha, beta, lxy, lz):
    sb, cb = np.sin(beta), np.cos(beta)
    numer = lxy * sb * (gx * np.cos(alpha) + gy * np.sin(alpha)) + lz * cb * gz
    denom = np.asarray(lxy, float) ** 2 * sb ** 2 + np.asarray(lz, float) ** 2 * cb ** 2
    return np.maximum(1.0, numer / denom)


def targets(alpha, beta, d, lxy, lz):
    sb = np.sin(beta)
    return np.stack([lxy * d * sb * np.cos(alpha), lxy * d * sb * np.sin(alpha), lz * d * np.cos(beta)])


def schedule(rho0=1.0, growth=2.0, stages=10, max_iters=150):
    return [rho0 * growth ** s for s in range(stages)], -(-max_iters // stages)


def solve(spec, max_iters=150, tol=1e-2, rho0=1.0, growth=2.0, stages=10, keep_state=False,
          factors=None):
    """Full AM solve; returns a dict shaped like SolveReport (no metrics)."""
    pr = Problem(spec)
    n, nv, m, p = pr.n, pr.nv, pr.m, pr.p
    rhos, every = schedule(rho0, growth, stages, max_iters)
    if factors is None:
        factors = [lu_factor(pr.kkt(r), check_finite=False) for r in rhos]
    lxy, lz = pr.lxy[:, None], pr.lz[:, None]
    c = np.empty((3, n, nv))
    frac = np.arange(nv) / spec.degree
    for i, (s, g) in enumerate(zip(spec.start, spec.goal)):
        for a in range(3):
            if pr.kind == "bernstein":
                c[a, i] = s.position[a] + frac * (g.position[a] - s.position[a])
            else:
                c[a, i] = 0.0
                c[a, i, 0] = s.position[a]
                c[a, i, 1] = g.position[a] - s.position[a]
    lam = np.zeros((3, p, m))
    alpha, beta, d = np.zeros((p, m)), np.full((p, m), np.pi / 2), np.ones((p, m))
    if p:
        D = pr.diffs(c)
        alpha, beta = project(D[0], D[1], D[2], lxy, lz)
        d = np.maximum(1.0, scale(D[0], D[1], D[2], lxy, lz))
    hn, hm, hb = [], [], []
    it, conv = 0, False
    nc = n * nv
    for k in range(max_iters):
        stage = min(k // every, len(rhos) - 1)
        rho = rhos[stage]
        tg = targets(alpha, beta, d, lxy, lz)
        for a in range(3):
            b = tg[a] - lam[a] / rho + pr.off[:, a][:, None]
            agg = pr.S.T @ b.reshape(p, m)
            rhs = np.concatenate([rho * (agg @ pr.P).ravel(), pr.b_eq[a]])
            c[a] = lu_solve(factors[stage], rhs, check_finite=False)[:nc].reshape(n, nv)
        D = pr.diffs(c)
        alpha, beta = project(D[0], D[1], D[2], lxy, lz)
        ir = 1.0 / rho
        d = d_step(D[0] + lam[0] * ir, D[1] + lam[1] * ir, D[2] + lam[2] * ir, alpha, beta, lxy, lz)
        r = D - targets(alpha, beta, d, lxy, lz)
        lam += rho * r
        if r.size:
            hn.append(float(np.linalg.norm(r)))
            hm.append(float(np.max(np.abs(r))))
        else:
            hn.append(0.0)
            hm.append(0.0)
        hb.append(max(float(np.max(np.abs(pr.A_eq @ c[a].ravel() - pr.b_eq[a]))) for a in range(3)))
        it = k + 1
        if hm[-1] <= tol:
            conv = True
            break
    traj = np.stack([c[a] @ pr.P.T for a in range(3)], axis=-1)
    out = {"coefficients": c, "trajectories": traj, "iterations": it, "converged": conv,
           "residual_norm_history": np.array(hn), "residual_max_history": np.array(hm),
           "boundary_max_history": np.array(hb)}
    if keep_state:
        out.update(alpha=alpha, beta=beta, d=d, lam=lam)
    return out


def min_normalized_distance(spec, traj) -> tuple[float, int]:
    """(min normalized distance, #samples < 1), validation.py:39-93 semantics."""
    n = traj.shape[0]
    best, bad = math.inf, 0
    if n > 1:
        ii, jj = np.triu_indices(n, 1)
        v = np.sqrt(((traj[ii, :, 0] - traj[jj, :, 0]) / spec.geometry.l_xy) ** 2
                    + ((traj[ii, :, 1] - traj[jj, :, 1]) / spec.geometry.l_xy) ** 2
                    + ((traj[ii, :, 2] - traj[jj, :, 2]) / spec.geometry.l_z) ** 2)
        best, bad = float(v.min()), int((v < 1).sum())
    for obs in spec.obstacles:
        sxy = spec.geometry.l_xy / 2 + obs.radius
        sz = spec.geometry.l_z / 2 + obs.radius
        c = np.asarray(obs.center)
        v = np.sqrt(((traj[..., 0] - c[0]) / sxy) ** 2 + ((traj[..., 1] - c[1]) / sxy) ** 2
                    + ((traj[..., 2] - c[2]) / sz) ** 2)
        best, bad = min(best, float(v.min())), bad + int((v < 1).sum())
    return best, bad


def check_collisions_scalar(traj, l_xy, l_z, obstacles=()):
    """Scalar restatement of validation.py:39-93 (check_collisions), loop for loop.

    Returns (minimum, violations) with violations as
    ((kind, i, j_or_k), sample, value).  Pure Python: small cases only.
    """
    traj = np.asarray(traj, dtype=float)
    n, m, _ = traj.shape
    minimum = math.inf
    viol = []
    for i in range(n):
        for j in range(i + 1, n):
            for r in range(m):
                dx = (float(traj[i, r, 0]) - float(traj[j, r, 0])) / l_xy
                dy = (float(traj[i, r, 1]) - float(traj[j, r, 1])) / l_xy
                dz = (float(traj[i, r, 2]) - float(traj[j, r, 2])) / l_z
                v = math.sqrt(dx * dx + dy * dy + dz * dz)
                minimum = min(minimum, v)
                if v < 1.0:
                    viol.append((("agent", i, j), r, v))
    for i in range(n):
        for k, (center, radius) in enumerate(obstacles):
            sxy = l_xy / 2.0 + radius
            sz = l_z / 2.0 + radius
            for r in range(m):
                dx = (float(traj[i, r, 0]) - center[0]) / sxy
                dy = (float(traj[i, r, 1]) - center[1]) / sxy
                dz = (float(traj[i, r, 2]) - center[2]) / sz
                v = math.sqrt(dx * dx + dy * dy + dz * dz)
                minimum = min(minimum, v)
                if v < 1.0:
                    viol.append((("obstacle", i, k), r, v))
    return minimum, viol
