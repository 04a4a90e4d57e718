# full GPU suite, then c5/c3/c3sfft timelines and a short bench with the c5 / c3_sfft legs
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
WORKS="c5 c3 c3sfft" bash tools/gpu_timelines.sh
timeout 900 python bench.py --steps 50 --warmup 5 --legs c5,c3_sfft,c1 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
