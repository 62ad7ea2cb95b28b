#!/bin/bash
# Round-end measurement pass: bench lines (ours + reference arm), ncu launch list of the bench
# command, one full ncu capture of the AM kernel (summaries exported as CSV, report left on the box).
set -u
mkdir -p gpurun_out/final
python bench.py > gpurun_out/final/bench.jsonl 2> gpurun_out/final/bench.err
python bench.py --impl reference > gpurun_out/final/bench_reference.jsonl 2> gpurun_out/final/bench_reference.err
python bench.py --steps 2 --warmup 3 --no-cpu --no-single > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-single > gpurun_out/final/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:am_cluster -c 1 -o /tmp/final_full \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-single > gpurun_out/final/ncu_full.log 2>&1
ncu -i /tmp/final_full.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/final/full_raw.csv.gz
ncu -i /tmp/final_full.ncu-rep --page details --csv 2>/dev/null | gzip > gpurun_out/final/full_details.csv.gz
ncu -i /tmp/final_full.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/final/full_src.csv.gz
ls -la gpurun_out/final
