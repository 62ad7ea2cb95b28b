#!/bin/bash
# run each dump_coeffs instance separately under the stream kernels (find hangs / slow cases)
for nm in circ16j rand32_s0 sph64j rand48_s0 obs8 hallway4j rand8_s1 single_agent sph16j rand128_s0 rand256_s0; do
  SWARM_LAM_STREAM=1 timeout 60 python -c "
import sys, time; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
from conftest import load_golden
from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve
spec, cfg, ref = load_golden('$nm')
t=time.time(); r = am_solve(spec, SolverConfig(max_iters=60), cache=FactorCache()); print('$nm', r.iterations, round(time.time()-t,3), flush=True)
" 2>&1 | tail -1
  echo "rc=$?"
done
