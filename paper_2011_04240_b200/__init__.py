"""B200-native drop-in for the reference ``swarmtraj.am_solve`` path (arXiv 2011.04240).

Public surface mirrors the reference package (``swarmtraj/__init__.py``)
for everything on the solve path: problem description in, ``SolveReport``
out.  The AM loop itself runs in hand-written sm_100a CUDA behind the C ABI
in ``include/swarm_am.h``.
"""

from .engine import (FinalState, InfeasibleProblemError, NonFiniteStateError, Multipliers, PairVariables, SolveReport,
                     SolverConfig, am_solve, am_solve_batch, default_cache, pack)
from .kkt import (FactorCache, Fingerprint, RhoSchedule, StageOperator, build_rho_schedule, fingerprint,
                  stage_operator)
from .metrics import CollisionReport, TrajectoryMetrics, arc_length, check_collisions, smoothness, trajectory_metrics
from .poly import Basis
from .poly import build as build_basis
from .scenarios import (circle_swap, generate_hallway, generate_random, generate_random_with_obstacles,
                        generate_square, jitter, named, sphere_swap)
from .spec import (AgentGeometry, BasisKind, BoundaryState, Obstacle, ProblemSpec, Violation, load_scenario,
                   save_scenario, spec_from_dict, spec_to_dict, validate)

__version__ = "0.1.0"
