# high-frequency warp sampling of chosen kernels in one c3 fp32 transform
set -u
mkdir -p gpurun_out
python tools/run_one.py fp32 1 > gpurun_out/plain_hot.log 2>&1 &&
timeout 1200 ncu -f --set full --warp-sampling-interval 0 --clock-control none --import-source on \
   -k regex:"k_small_pass|k_fold_ring2|k_lmax_win|k_vote_lazy|k_pass_conv" -c 12 -o /tmp/hot \
   python tools/run_one.py fp32 1 > gpurun_out/ncu_hot.log 2>&1
for k in k_small_pass k_fold_ring2 k_lmax_win k_vote_lazy k_pass_conv; do
  ncu -i /tmp/hot.ncu-rep --page source --csv -k regex:$k --launch-count 1 > gpurun_out/hot_$k.csv 2>/dev/null
done
ncu -i /tmp/hot.ncu-rep --page details --csv > gpurun_out/hot_details.csv 2>/dev/null
gzip -f gpurun_out/hot_*.csv
