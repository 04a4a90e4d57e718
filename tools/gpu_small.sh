# dense warp sampling of the single-CTA small pass and the B=2048 local-maximum launch
set -u
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
python tools/run_one.py fp32 1 > /dev/null 2>&1 || exit 1
for SPEC in k_small_pass:3 k_lmax_stream:2; do
  K=${SPEC%%:*}; SKIP=${SPEC##*:}
  timeout 600 ncu -f --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:$K --launch-skip $SKIP -c 1 \
     -o /tmp/${K}_$SKIP python tools/run_one.py fp32 1 > gpurun_out/ncu_${K}_$SKIP.log 2>&1
  ncu -i /tmp/${K}_$SKIP.ncu-rep --page details --csv > gpurun_out/ncu_${K}_${SKIP}_details.csv 2>/dev/null
  ncu -i /tmp/${K}_$SKIP.ncu-rep --page source --csv > gpurun_out/ncu_${K}_${SKIP}_source.csv 2>/dev/null
done
timeout 900 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
