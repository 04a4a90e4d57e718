# round-2 ncu evidence: one c3 fp32 transform under --set full (per-launch DRAM
# traffic and durations), the same for the known-k SFFT transform
set -u
mkdir -p gpurun_out
python tools/run_one.py fp32 1 > gpurun_out/plain_c3.log 2>&1 &&
timeout 1500 ncu -f --set full --clock-control none --import-source on -o /tmp/c3_full \
    python tools/run_one.py fp32 1 > gpurun_out/ncu_full.log 2>&1
ncu -i /tmp/c3_full.ncu-rep --page raw --csv > gpurun_out/c3_full_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/c3_full_raw.csv --launches --json gpurun_out/kernel_traffic_c3.json \
    > gpurun_out/c3_full_summary.txt 2>&1
python tools/sfft_time.py 4096 100 fp32 > gpurun_out/plain_sfft.log 2>&1 &&
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_fold_ml -c 2 -o /tmp/sfft_fold \
    python tools/sfft_time.py 4096 100 fp32 > gpurun_out/ncu_sfft.log 2>&1
ncu -i /tmp/sfft_fold.ncu-rep --page raw --csv > gpurun_out/sfft_fold_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/sfft_fold_raw.csv --launches > gpurun_out/sfft_fold_summary.txt 2>&1
ncu -i /tmp/c3_full.ncu-rep --page details --csv > gpurun_out/c3_full_details.csv 2>/dev/null
for k in k_pass_conv k_lmax_win k_vote_lazy k_small_pass k_fold_ring2; do
  ncu -i /tmp/c3_full.ncu-rep --page source --csv -k regex:$k --launch-count 1 > gpurun_out/src_$k.csv 2>/dev/null
done
gzip -f gpurun_out/c3_full_raw.csv gpurun_out/c3_full_details.csv gpurun_out/src_*.csv
du -sh gpurun_out
