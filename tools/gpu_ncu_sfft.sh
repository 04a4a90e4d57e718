# full ncu capture of the first multi-loop fold of a c3 known-k SFFT
set -u
mkdir -p gpurun_out
python tools/sfft_time.py 4096 100 fp32 > /dev/null 2>&1 || exit 1
timeout 600 ncu -f --set full --warp-sampling-interval 2 --clock-control none --import-source on -k regex:k_fold --launch-skip 0 -c 1 \
   -o /tmp/kfold python tools/sfft_time.py 4096 100 fp32 > gpurun_out/ncu_kfold.log 2>&1
ncu -i /tmp/kfold.ncu-rep --page details --csv > gpurun_out/ncu_kfold_details.csv 2>/dev/null
ncu -i /tmp/kfold.ncu-rep --page source --csv > gpurun_out/ncu_kfold_source.csv 2>/dev/null
