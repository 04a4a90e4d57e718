# probe: concurrency sweep + per-launch ncu times/DRAM bytes of one c3 transform
set -u
mkdir -p gpurun_out
timeout 600 python tools/concurrency.py fp32 > gpurun_out/conc.txt 2>&1
python tools/run_one.py fp32 1 > /dev/null 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/probe_ncu.csv python tools/run_one.py fp32 1 > gpurun_out/probe_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/probe_ncu.csv --launches > gpurun_out/probe_summary.txt 2>&1
