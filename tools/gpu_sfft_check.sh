# SFFT multi-loop fold check: parity tests, then new vs old fold timings
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_api_lowlevel.py tests/test_distributed_gpu.py tests/test_acceptance_gpu.py -m gpu -q -x -k "sfft or SFFT or c05 or loopsplit or c10" > gpurun_out/pytest_sfft.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sfft.log
: > gpurun_out/sfft_times.txt
for args in "4096 100 fp32" "4096 100 fp64" "256 10 fp64" "1024 50 fp32" "16384 64 fp32"; do
  timeout 120 python tools/sfft_time.py $args >> gpurun_out/sfft_times.txt 2>&1
  SFFT2D_OLD_MLFOLD=1 timeout 120 python tools/sfft_time.py $args 2>&1 | head -1 | sed 's/^/OLD /' >> gpurun_out/sfft_times.txt
done
