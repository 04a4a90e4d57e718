#!/bin/bash
# Round profile: bench line, ncu launch list of the bench command, and one
# `--set full` capture of a c3 transform (per-kernel DRAM traffic).  Output in
# gpurun_out/; summaries are copied into profiles/ by hand.
set -u
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err || exit 1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --c4-images 0 --no-e2e > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    --c4-images 0 --no-e2e > gpurun_out/ncu_launches.log 2>&1
python tools/run_one.py fp32 1 > /dev/null || exit 1
timeout 1500 ncu -f --set full --clock-control none --import-source on -o /tmp/c3_full \
    python tools/run_one.py fp32 1 > gpurun_out/ncu_full.log 2>&1
ncu -i /tmp/c3_full.ncu-rep --page raw --csv > gpurun_out/c3_full_raw.csv
python tools/ncu_summary.py gpurun_out/c3_full_raw.csv --launches --json gpurun_out/kernel_traffic.json \
    > gpurun_out/c3_full_summary.txt
python tools/ncu_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt
