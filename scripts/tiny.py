import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_04240_b200 import SolverConfig, am_solve, generate_random, named
name = sys.argv[1] if len(sys.argv) > 1 else "2"
C = int(sys.argv[2]) if len(sys.argv) > 2 else 0
spec = generate_random(int(name), (8, 8, 3), 0.4, 0) if name.isdigit() else named(name)
r = am_solve(spec, SolverConfig(cluster_size=C))
print("ok", name, C, r.iterations, r.converged)
