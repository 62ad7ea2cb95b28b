#!/bin/bash
# A/B of the LAM_STREAM kernels against the default build (bounded by timeouts)
set -x
SWARM_LAM_STREAM=1 timeout 120 python scripts/one_solve.py rand32_s0 2 2>&1 | tail -2
SWARM_LAM_STREAM=1 timeout 120 python scripts/one_solve.py batch148 2 2>&1 | tail -2
SWARM_LAM_STREAM=1 timeout 300 python scripts/dump_coeffs.py gpurun_out/stream.npz 2>&1 | tail -2
timeout 300 python scripts/dump_coeffs.py gpurun_out/default.npz 2>&1 | tail -1
python scripts/dump_coeffs.py --compare gpurun_out/default.npz gpurun_out/stream.npz
SWARM_LAM_STREAM=1 SWARM_PHASE_TIMERS=1 timeout 120 python scripts/batch_probe.py 1024 2 2>&1 | tail -3
SWARM_LAM_STREAM=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-single 2>&1 | tail -1 | cut -c1-200
