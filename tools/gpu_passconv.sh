set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_acceptance_gpu.py tests/test_api_lowlevel.py -m gpu -q -x > gpurun_out/pytest_pc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pc.log
: > gpurun_out/pc_times.txt
for w in c3 c2; do
  timeout 300 python tools/timeline.py fp32 5 $w 2>&1 | head -30 >> gpurun_out/pc_times.txt
  SFFT2D_NO_PASSCONV=1 timeout 300 python tools/timeline.py fp32 5 $w 2>&1 | head -2 | sed 's/^/OFF /' >> gpurun_out/pc_times.txt
done
python tools/concurrency.py > gpurun_out/conc.txt 2>&1
SFFT2D_NO_PASSCONV=1 python tools/concurrency.py 2>&1 | sed 's/^/OFF /' >> gpurun_out/conc.txt
