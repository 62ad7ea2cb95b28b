#!/bin/bash
# Round-end measurement pass: bench lines (ours + reference arm), ncu launch list of the bench
# command, one full ncu capture of the AM kernel (summaries exported as CSV, report left on the box).
set -u
OUT=${1:-gpurun_out/final}; mkdir -p $OUT
python bench.py > $OUT/bench.jsonl 2> $OUT/bench.err
python bench.py --impl reference > $OUT/bench_reference.jsonl 2> $OUT/bench_reference.err
python bench.py --steps 2 --warmup 3 --no-cpu --no-single > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-single > $OUT/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:am_cluster -c 1 -f -o /tmp/final_full \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-single > $OUT/ncu_full.log 2>&1
ncu -i /tmp/final_full.ncu-rep --page raw --csv 2>/dev/null | gzip > $OUT/full_raw.csv.gz
ncu -i /tmp/final_full.ncu-rep --page details --csv 2>/dev/null | gzip > $OUT/full_details.csv.gz
ncu -i /tmp/final_full.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $OUT/full_src.csv.gz
ls -la $OUT
