"""Device-loop time of a few single solves (second of two runs) for the library in SWARM_LIB."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import load_golden
from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve
out = []
for name in ["circ16j", "rand32_s0", "sph64j", "rand48_s0", "rand256_s0"]:
    spec, cfg, ref = load_golden(name)
    cache = FactorCache()
    best = 1e9
    for _ in range(3):
        r = am_solve(spec, SolverConfig(), cache=cache)
        best = min(best, r.timings["loop_s"] * 1e3)
    out.append(f"{name}={best:.3f}ms/{r.iterations}")
print(os.environ.get("SWARM_LIB", "current").split("/")[-1], " ".join(out))
