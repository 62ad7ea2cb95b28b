#!/bin/bash
# One full ncu capture (source counters) of the bench's batch kernel; CSV pages into gpurun_out/$1.
set -u
tag=${1:-ncu}
mkdir -p gpurun_out/$tag
python scripts/batch_probe.py 1024 2 > gpurun_out/$tag/probe.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:am_cluster -c 1 -f -o /tmp/$tag \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-single > gpurun_out/$tag/ncu_full.log 2>&1
ncu -i /tmp/$tag.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/$tag/full_raw.csv.gz
ncu -i /tmp/$tag.ncu-rep --page details --csv 2>/dev/null | gzip > gpurun_out/$tag/full_details.csv.gz
ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/$tag/full_src.csv.gz
cp /tmp/$tag.ncu-rep gpurun_out/$tag/ 2>/dev/null
cat gpurun_out/$tag/probe.txt
