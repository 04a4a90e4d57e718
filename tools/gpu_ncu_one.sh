# full ncu capture of chosen launches of one c3 transform: NCU_SPECS="name:skip name:skip ..."
set -u
mkdir -p gpurun_out
python tools/run_one.py fp32 1 > /dev/null 2>&1 || exit 1
for SPEC in $NCU_SPECS; do
  K=${SPEC%%:*}; SKIP=${SPEC##*:}
  timeout 600 ncu -f --set full --warp-sampling-interval 2 --clock-control none --import-source on -k regex:$K --launch-skip $SKIP -c 1 \
     -o /tmp/${K}_$SKIP python tools/run_one.py fp32 1 > gpurun_out/ncu_${K}_$SKIP.log 2>&1
  ncu -i /tmp/${K}_$SKIP.ncu-rep --page details --csv > gpurun_out/ncu_${K}_${SKIP}_details.csv 2>/dev/null
  ncu -i /tmp/${K}_$SKIP.ncu-rep --page source --csv > gpurun_out/ncu_${K}_${SKIP}_source.csv 2>/dev/null
done
