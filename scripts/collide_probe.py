"""Time st_check_collisions on rand256_s0's reference solution (CUDA events inside the C call are
not exposed, so this reports host wall time per call over many calls; ncu gives the kernel times)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from conftest import load_golden  # noqa: E402

from paper_2011_04240_b200 import metrics, poly  # noqa: E402

spec, _, ref = load_golden("rand256_s0")
traj = np.ascontiguousarray(np.einsum("ank,tk->nta", ref["coefficients"], poly.for_spec(spec).P))
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
metrics.check_collisions_device(traj, spec.geometry, spec.obstacles)
t = time.perf_counter()
for _ in range(reps):
    col = metrics.check_collisions_device(traj, spec.geometry, spec.obstacles)
dev = (time.perf_counter() - t) / reps
t = time.perf_counter()
host = metrics.check_collisions(traj, spec.geometry, spec.obstacles)
ht = time.perf_counter() - t
print(f"rand256_s0 collision verdict: device call {dev * 1e3:.3f} ms, host numpy {ht * 1e3:.1f} ms, "
      f"{len(col.violations)} violations, min {col.min_normalized_distance!r}, equal={col.violations == host.violations}")
