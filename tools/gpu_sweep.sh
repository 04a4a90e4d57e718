# fold ring grid sweep: per-launch ncu times of one c3 transform per setting
set -u
mkdir -p gpurun_out
python tools/run_one.py fp32 1 > /dev/null 2>&1 || exit 1
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/sweep_$tag.csv python tools/run_one.py fp32 1 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/sweep_$tag.csv --launches > gpurun_out/sweep_$tag.txt 2>&1
  env "$@" python tools/concurrency.py fp32 > gpurun_out/sweep_conc_$tag.txt 2>&1
}
run base X=1
run onewave SFFT2D_FOLD_ONEWAVE=1
run t444 SFFT2D_FOLD_TARGET=444
run t592 SFFT2D_FOLD_TARGET=592
