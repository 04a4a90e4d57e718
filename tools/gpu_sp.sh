set -u
mkdir -p gpurun_out
: > gpurun_out/q_times.txt
for w in c2 c3; do timeout 300 python tools/timeline.py fp32 5 $w 2>&1 | grep -E "host wall|busy|k_small" >> gpurun_out/q_times.txt; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ats or atsfft or c2 or c4 or tuner" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
