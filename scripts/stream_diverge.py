"""Where do the LAM_STREAM kernels diverge from the default ones? (per max_iters)"""
import os, subprocess, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
name = sys.argv[1] if len(sys.argv) > 1 else "rand8_s1"
code = f"""
import sys, json; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np
from conftest import load_golden
from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve
spec, cfg, ref = load_golden('{name}')
out = {{}}
for mi in (1, 2, 3, 4, 8):
    r = am_solve(spec, SolverConfig(max_iters=mi, tolerance=1e-30), cache=FactorCache())
    out[mi] = [np.asarray(r.coefficients).ravel().tolist(), list(r.residual_norm_history), list(r.residual_max_history)]
print(json.dumps(out))
"""
res = {}
for flag in ("0", "1"):
    env = dict(os.environ, SWARM_LAM_STREAM=flag)
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    if p.returncode:
        print(flag, p.stderr[-2000:]); sys.exit(1)
    res[flag] = json.loads(p.stdout.strip().splitlines()[-1])
import numpy as np
for mi in res["0"]:
    a, b = res["0"][mi], res["1"][mi]
    print(mi, "coef maxdiff", float(np.max(np.abs(np.array(a[0]) - np.array(b[0])))),
          "norm hist", a[1], b[1], "max hist", a[2], b[2])
