# round evidence: ncu launch list of the bench command (c3 leg), ncu --set full
# of one c3 fp32 transform (per-kernel DRAM traffic -> kernel_traffic.json)
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --legs none --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_bench.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 900 --csv \
    --log-file gpurun_out/bench_launches.csv $CMD > gpurun_out/ncu_bench.log 2>&1
python tools/ncu_summary.py gpurun_out/bench_launches.csv > gpurun_out/bench_launches_summary.txt 2>&1
python tools/run_one.py fp32 1 > gpurun_out/plain_c3.log 2>&1 &&
timeout 1500 ncu -f --set full --clock-control none --import-source on -o /tmp/c3_full \
    python tools/run_one.py fp32 1 > gpurun_out/ncu_full.log 2>&1
ncu -i /tmp/c3_full.ncu-rep --page raw --csv > gpurun_out/c3_full_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/c3_full_raw.csv --launches --json gpurun_out/kernel_traffic_c3.json \
    > gpurun_out/c3_full_summary.txt 2>&1
gzip -f gpurun_out/c3_full_raw.csv gpurun_out/bench_launches.csv
