# parity + per-launch ncu + full ncu captures of selected kernels
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/run_one.py fp32 1 > /dev/null 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/probe_ncu.csv python tools/run_one.py fp32 1 > gpurun_out/probe_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/probe_ncu.csv --launches > gpurun_out/probe_summary.txt 2>&1
for K in ${PROBE_KERNELS:-k_vote_rows k_fftc_cl}; do
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:$K -c 2 -o /tmp/$K \
     python tools/run_one.py fp32 1 > gpurun_out/ncu_$K.log 2>&1
  ncu -i /tmp/$K.ncu-rep --page details --csv > gpurun_out/ncu_${K}_details.csv 2>/dev/null
  ncu -i /tmp/$K.ncu-rep --page source --csv > gpurun_out/ncu_${K}_source.csv 2>/dev/null
  cp /tmp/$K.ncu-rep gpurun_out/ 2>/dev/null
done
timeout 600 python tools/concurrency.py fp32 > gpurun_out/conc.txt 2>&1
if [ -n "${COMPARE_ENV:-}" ]; then env $COMPARE_ENV timeout 600 python tools/concurrency.py fp32 > gpurun_out/conc_compare.txt 2>&1; fi
