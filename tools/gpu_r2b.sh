# round-2 GPU check 2: new GPU tests, per-workload timelines, ncu launch list of one c3 transform
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_harness_verify.py tests/test_acceptance_gpu.py "tests/test_gpu_parity.py::test_count_local_maxima_vs_reference" "tests/test_gpu_parity.py::test_count_local_maxima_random_vs_oracle" -m gpu -q -x -s > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_new.log
WORKS="c3 c1 c3sfft c2 c5" bash tools/gpu_timelines.sh
python tools/run_one.py fp32 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/run_one.py fp32 1 > gpurun_out/ncu_c3.log 2>&1
python tools/ncu_summary.py gpurun_out/c3_launches.csv > gpurun_out/c3_launches_summary.txt 2>&1
