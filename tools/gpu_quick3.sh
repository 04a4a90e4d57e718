set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_api_lowlevel.py -m gpu -q -x > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
: > gpurun_out/q_times.txt
for w in c3 c2; do timeout 300 python tools/timeline.py fp32 5 $w 2>&1 | grep -v Warn | head -24 >> gpurun_out/q_times.txt; done
SFFT2D_LMAX_DIRECT_MAXB=0 timeout 300 python tools/timeline.py fp32 5 c3 2>&1 | grep -v Warn | head -3 | sed 's/^/NODIRECT /' >> gpurun_out/q_times.txt
python tools/concurrency.py > gpurun_out/conc.txt 2>&1
