set -u
mkdir -p gpurun_out
timeout 300 python tools/pass_host.py fp32 > gpurun_out/pass_host.txt 2>&1; echo "rc=$?" >> gpurun_out/pass_host.txt
SFFT2D_NO_PASS_PIPE=1 timeout 300 python tools/pass_host.py fp32 2>&1 | sed 's/^/OFF /' >> gpurun_out/pass_host.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_api_lowlevel.py tests/test_acceptance_gpu.py -m gpu -q -x > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
: > gpurun_out/q_times.txt
for w in c3 c2; do timeout 300 python tools/timeline.py fp32 5 $w 2>&1 | grep -E "host wall|busy" >> gpurun_out/q_times.txt; done
timeout 300 python tools/concurrency.py > gpurun_out/conc.txt 2>&1
