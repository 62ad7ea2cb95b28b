"""Synthetic scenario families used by the parity tests and ``bench.py``.

The reference's generators (problem.py:197-457) are re-stated so the same
seeds give the same instances (same RNG stream, same draw order):

* ``generate_random``                 problem.py:282-315 (rejection sampling, min separation 4r)
* ``generate_random_with_obstacles``  problem.py:318-380 (agents first, obstacles extend the stream)
* ``generate_square``                 problem.py:210-244 (antipodal points on a square perimeter)
* ``generate_hallway``                problem.py:383-457 (two groups, walls as rows of spheres)

plus the SURVEY.md §8(d) benchmark families the reference lacks: a 3D
antipodal circle swap (``circle_swap``; config 1, "circ16j") and a
Fibonacci-sphere antipodal swap (``sphere_swap``; config 3, "sph64j"), each
optionally symmetry-broken with ``jitter`` (uniform +-amp per coordinate from
``default_rng(seed)``, starts then goals).
"""

from __future__ import annotations

import math
from dataclasses import replace

import numpy as np

from .spec import (DEFAULT_DEGREE, DEFAULT_DURATION, DEFAULT_NUM_SAMPLES, AgentGeometry,
                   BoundaryState, Obstacle, ProblemSpec)

_MAX_REJECTIONS = 10_000


def _disc(num_samples, degree, duration):
    return dict(num_samples=num_samples, degree=degree, duration=duration)


def _rejection_sample(rng, n, box, min_sep, max_rejections):
    bx, by, bz = box
    pts: list[tuple] = []
    misses = 0
    while len(pts) < n:
        c = (float(rng.uniform(-bx / 2.0, bx / 2.0)), float(rng.uniform(-by / 2.0, by / 2.0)),
             float(rng.uniform(0.0, bz)))
        if all(math.dist(c, q) >= min_sep for q in pts):
            pts.append(c)
            continue
        misses += 1
        if misses >= max_rejections:
            raise ValueError(f"failed to place {n} points with separation {min_sep} in box {box} "
                             f"after {max_rejections} rejections")
    return pts


def generate_random(n, box, radius, seed, *, num_samples=DEFAULT_NUM_SAMPLES, degree=DEFAULT_DEGREE,
                    duration=DEFAULT_DURATION, max_rejections=_MAX_REJECTIONS) -> ProblemSpec:
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    if not radius > 0:
        raise ValueError(f"radius must be positive, got {radius}")
    rng = np.random.default_rng(seed)
    starts = _rejection_sample(rng, n, box, 4.0 * radius, max_rejections)
    goals = _rejection_sample(rng, n, box, 4.0 * radius, max_rejections)
    return ProblemSpec(start=tuple(BoundaryState.at_rest(p) for p in starts),
                       goal=tuple(BoundaryState.at_rest(p) for p in goals),
                       geometry=AgentGeometry.sphere_from_radius(radius), seed=seed,
                       **_disc(num_samples, degree, duration))


def generate_random_with_obstacles(n, box, radius, n_obs, obs_radius, seed, *,
                                   num_samples=DEFAULT_NUM_SAMPLES, degree=DEFAULT_DEGREE,
                                   duration=DEFAULT_DURATION,
                                   max_rejections=_MAX_REJECTIONS) -> ProblemSpec:
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    if not radius > 0:
        raise ValueError(f"radius must be positive, got {radius}")
    if n_obs > 0 and not obs_radius > 0:
        raise ValueError(f"obs_radius must be positive, got {obs_radius}")
    rng = np.random.default_rng(seed)
    starts = _rejection_sample(rng, n, box, 4.0 * radius, max_rejections)
    goals = _rejection_sample(rng, n, box, 4.0 * radius, max_rejections)
    spec = ProblemSpec(start=tuple(BoundaryState.at_rest(p) for p in starts),
                       goal=tuple(BoundaryState.at_rest(p) for p in goals),
                       geometry=AgentGeometry.sphere_from_radius(radius), seed=seed,
                       **_disc(num_samples, degree, duration))
    if n_obs == 0:
        return spec
    ends = starts + goals
    clear = obs_radius + 2.0 * radius
    bx, by, bz = box
    obs: list[Obstacle] = []
    misses = 0
    while len(obs) < n_obs:
        c = (float(rng.uniform(-bx / 2.0, bx / 2.0)), float(rng.uniform(-by / 2.0, by / 2.0)),
             float(rng.uniform(0.0, bz)))
        if all(math.dist(c, p) >= clear for p in ends):
            obs.append(Obstacle(center=c, radius=obs_radius))
            continue
        misses += 1
        if misses >= max_rejections:
            raise ValueError(f"failed to place {n_obs} obstacles clear of endpoints after "
                             f"{max_rejections} rejections")
    return replace(spec, obstacles=tuple(obs))


def _perimeter_point(side, s, z):
    s = s % (4.0 * side)
    h = side / 2.0
    if s < side:
        return (-h + s, -h, z)
    if s < 2 * side:
        return (h, -h + (s - side), z)
    if s < 3 * side:
        return (h - (s - 2 * side), h, z)
    return (-h, h - (s - 3 * side), z)


def generate_square(n, side, radius, z_plane=1.0, *, num_samples=DEFAULT_NUM_SAMPLES,
                    degree=DEFAULT_DEGREE, duration=DEFAULT_DURATION) -> ProblemSpec:
    if n < 2:
        raise ValueError(f"square scenario needs n >= 2, got {n}")
    if not (side > 0 and radius > 0):
        raise ValueError(f"side and radius must be positive, got side={side}, radius={radius}")
    per = 4.0 * side
    gap = per / n
    starts = tuple(BoundaryState.at_rest(_perimeter_point(side, i * gap, z_plane)) for i in range(n))
    goals = tuple(BoundaryState.at_rest(_perimeter_point(side, i * gap + per / 2.0, z_plane))
                  for i in range(n))
    return ProblemSpec(start=starts, goal=goals, geometry=AgentGeometry.sphere_from_radius(radius),
                       **_disc(num_samples, degree, duration))


def generate_hallway(n, hallway_length, hallway_width, radius, *, z_plane=1.0,
                     num_samples=DEFAULT_NUM_SAMPLES, degree=DEFAULT_DEGREE,
                     duration=DEFAULT_DURATION) -> ProblemSpec:
    if n % 2 != 0:
        raise ValueError(f"hallway scenario needs an even n, got {n}")
    if n < 2:
        raise ValueError(f"hallway scenario needs n >= 2, got {n}")
    if hallway_width < 4.0 * radius:
        raise ValueError(f"hallway width {hallway_width} cannot admit agent diameter with margin "
                         f"(need >= {4 * radius})")
    if not (hallway_length > 0 and radius > 0):
        raise ValueError("hallway_length and radius must be positive")
    half = n // 2
    spacing = 4.0 * radius
    usable = hallway_width / 2.0 - 2.0 * radius
    cols = min(max(1, int(usable * 2.0 // spacing) + 1), half)
    rows = math.ceil(half / cols)
    depth = (rows - 1) * spacing
    if depth > hallway_length / 2.0 - spacing:
        raise ValueError(f"{n} agents do not fit in the hallway ends (need depth {depth:.2f} per side)")
    ys = np.linspace(-usable, usable, cols) if cols > 1 else np.array([0.0])
    starts, goals = [], []
    for sign in (-1.0, 1.0):
        placed = 0
        for r in range(rows):
            for c in range(cols):
                if placed >= half:
                    break
                x = sign * (hallway_length / 2.0 + r * spacing)
                starts.append(BoundaryState.at_rest((x, float(ys[c]), z_plane)))
                goals.append(BoundaryState.at_rest((-x, float(ys[c]), z_plane)))
                placed += 1
    wall_r = 2.0 * hallway_width
    n_wall = int(hallway_length // (hallway_width / 2.0)) + 1
    xs = np.linspace(-hallway_length / 2.0, hallway_length / 2.0, n_wall)
    walls = tuple(Obstacle(center=(float(x), s * (hallway_width / 2.0 + wall_r), z_plane), radius=wall_r)
                  for s in (-1.0, 1.0) for x in xs)
    return ProblemSpec(start=tuple(starts), goal=tuple(goals),
                       geometry=AgentGeometry.sphere_from_radius(radius), obstacles=walls,
                       **_disc(num_samples, degree, duration))


# --- SURVEY.md §8(d) benchmark families -----------------------------------------------------


def jitter(starts, goals, amp: float, seed: int):
    """Symmetry breaking: uniform(-amp, amp)^3 per agent, all starts first, then all goals."""
    rng = np.random.default_rng(seed)
    js = [tuple(np.asarray(p, float) + rng.uniform(-amp, amp, 3)) for p in starts]
    jg = [tuple(np.asarray(p, float) + rng.uniform(-amp, amp, 3)) for p in goals]
    return js, jg


def _swap_spec(starts, goals, radius, amp, seed, **disc):
    if amp > 0:
        starts, goals = jitter(starts, goals, amp, seed)
    return ProblemSpec(start=tuple(BoundaryState.at_rest(p) for p in starts),
                       goal=tuple(BoundaryState.at_rest(p) for p in goals),
                       geometry=AgentGeometry.sphere_from_radius(radius), **disc)


def circle_swap(n=16, radius=0.4, circle_radius=4.0, jitter_amp=0.05, seed=0, *,
                num_samples=DEFAULT_NUM_SAMPLES, degree=DEFAULT_DEGREE,
                duration=DEFAULT_DURATION) -> ProblemSpec:
    """circ{n}j: theta_i = 2 pi i/n, z alternates 1.5 +- 0.5; goal = (-x, -y, 3 - z)."""
    starts, goals = [], []
    for i in range(n):
        th = 2.0 * math.pi * i / n
        s = (circle_radius * math.cos(th), circle_radius * math.sin(th), 1.5 + 0.5 * (1 if i % 2 == 0 else -1))
        starts.append(s)
        goals.append((-s[0], -s[1], 3.0 - s[2]))
    return _swap_spec(starts, goals, radius, jitter_amp, seed, **_disc(num_samples, degree, duration))


def sphere_swap(n=64, radius=0.4, sphere_radius=4.0, z0=4.0, jitter_amp=0.05, seed=0, *,
                num_samples=DEFAULT_NUM_SAMPLES, degree=DEFAULT_DEGREE,
                duration=DEFAULT_DURATION) -> ProblemSpec:
    """sph{n}j: Fibonacci sphere, goal = (-x, -y, 2 z0 - z)."""
    ga = math.pi * (3.0 - math.sqrt(5.0))
    starts, goals = [], []
    for i in range(n):
        z = 1.0 - 2.0 * (i + 0.5) / n
        r = math.sqrt(1.0 - z * z)
        s = (sphere_radius * r * math.cos(ga * i), sphere_radius * r * math.sin(ga * i), z0 + sphere_radius * z)
        starts.append(s)
        goals.append((-s[0], -s[1], 2.0 * z0 - s[2]))
    return _swap_spec(starts, goals, radius, jitter_amp, seed, **_disc(num_samples, degree, duration))


def named(name: str) -> ProblemSpec:
    """The SURVEY.md §8(d) configs by name: circ16j, circ16, sph16j, sph64j, rand32_s<k>, rand256_s<k>,
    and hall<n>[j]: the reference CLI/service's default corridor (generate_hallway(n, 20, 4, 0.4),
    cli.py:80-83) -- the obstacle-heavy case (two walls of sphere obstacles); "j" jitters the
    boundary positions as for the swaps (the exact corridor is symmetric and chaotic)."""
    if name.startswith("hall"):
        spec = generate_hallway(int(name[4:].rstrip("j")), 20.0, 4.0, 0.4)
        if name.endswith("j"):
            js, jg = jitter([s.position for s in spec.start], [g.position for g in spec.goal], 0.05, 0)
            spec = replace(spec, start=tuple(BoundaryState.at_rest(p) for p in js),
                           goal=tuple(BoundaryState.at_rest(p) for p in jg))
        return spec
    if name.startswith("circ"):
        n = int(name[4:].rstrip("j"))
        return circle_swap(n, jitter_amp=0.05 if name.endswith("j") else 0.0)
    if name.startswith("sph"):
        n = int(name[3:].rstrip("j"))
        return sphere_swap(n, jitter_amp=0.05 if name.endswith("j") else 0.0)
    if name.startswith("rand"):
        n_s, seed_s = name[4:].split("_s")
        n = int(n_s)
        box = (8.0, 8.0, 3.0) if n <= 64 else (20.0, 20.0, 6.0)
        return generate_random(n, box, 0.4, int(seed_s))
    raise ValueError(f"unknown scenario {name!r}")
