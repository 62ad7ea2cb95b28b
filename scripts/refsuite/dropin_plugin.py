"""pytest plugin: run the REFERENCE's own test suite with ``swarmtraj.am_solve`` replaced by the drop-in.

Loaded with ``-p dropin_plugin`` before any test module is imported; it calls
``paper_2011_04240_b200.compat.install()`` -- the one line a maintainer adds
 -- so every reference caller (solver.am_solve, cli, service,
bench) receives the reference's own ``ProblemSpec`` / ``SolverConfig`` /
``FactorCache`` objects and solves on the B200.
"""

import swarmtraj

from paper_2011_04240_b200 import compat, engine

CALLS = {"n": 0}
_orig = engine.am_solve


def _counting(spec, config=None, cache=None):
    CALLS["n"] += 1
    return _orig(spec, config, cache)


engine.am_solve = _counting
compat.install(swarmtraj)


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"[dropin] swarmtraj.am_solve calls served by the B200 drop-in: {CALLS['n']}")
