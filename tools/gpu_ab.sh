# A/B of one switch: tests touching the change, then c3 timeline + in-flight
# throughput with and without $AB_ENV (e.g. AB_ENV=SFFT2D_NO_PAIRCOL=1).
# TESTS: pytest -k expression (default: FFT + c3 parity)
set -u
mkdir -p gpurun_out
K=${TESTS:-"large_fft or binned or c3 or c2 or c5_atsfft or c4_bench_images_fp32"}
timeout 1200 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_pytest.log
: > gpurun_out/ab.txt
for side in new old; do
  if [ $side = old ]; then E="env $AB_ENV"; else E="env"; fi
  echo "== $side ($E)" >> gpurun_out/ab.txt
  for w in ${WORKS:-c3}; do
    timeout 300 $E python tools/timeline.py fp32 5 $w > gpurun_out/ab_tl_${side}_$w.txt 2>&1
    grep -E "host wall|busy" gpurun_out/ab_tl_${side}_$w.txt >> gpurun_out/ab.txt
  done
  timeout 300 $E python tools/stress_conc.py 6 4 >> gpurun_out/ab.txt 2>&1
  timeout 300 $E python tools/stress_conc.py 1 2 >> gpurun_out/ab.txt 2>&1
done
