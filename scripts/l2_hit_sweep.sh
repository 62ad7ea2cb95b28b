#!/bin/bash
# L2 persisting-window hit ratio vs DRAM traffic and loop time of the 1024-scenario batch launch
python - <<'PY'
import torch
p = torch.cuda.get_device_properties(0)
print("L2 bytes", p.L2_cache_size)
from cuda.bindings import runtime as rt
for attr in ("cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize"):
    print(attr, rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, attr), 0)[1])
PY
for h in "" 0.95 0.9 0.85 0.8 0.7 0.6; do
  SWARM_PIPE_CHUNKS=1 SWARM_L2_HIT=$h ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:am_cluster -s 1 -c 1 python scripts/one_solve.py batch1024 2 2>&1 | grep -E "dram__|gpu__time" | tr -s ' ' | sed "s#^#hit=${h:-auto} #"
  SWARM_L2_HIT=$h python scripts/batch_probe.py 1024 2 | sed "s#^#hit=${h:-auto} #"
done
