#!/bin/bash
# Full ncu capture (source counters) of one am_cluster launch of scripts/one_solve.py <name> <C>.
set -u
tag=$1; shift
mkdir -p gpurun_out/$tag
ncu --set full --import-source on --clock-control none -k regex:"am_(cluster|large)" -s 1 -c 1 -f -o /tmp/$tag \
    python scripts/one_solve.py "$@" > gpurun_out/$tag/ncu.log 2>&1
ncu -i /tmp/$tag.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/$tag/full_raw.csv.gz
ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/$tag/full_src.csv.gz
tail -3 gpurun_out/$tag/ncu.log
