# sweep of the L2 prefetch distance of the TMA rings (SFFT2D_PF rows ahead):
# per-pass host times of one c3 transform, in-flight throughput, fold bandwidth
set -u
mkdir -p gpurun_out
: > gpurun_out/pf.txt
for pf in ${PFS:-0 2 4 8}; do
  echo "== SFFT2D_PF=$pf" >> gpurun_out/pf.txt
  SFFT2D_PF=$pf timeout 300 python tools/pass_host.py fp32 >> gpurun_out/pf.txt 2>&1
  SFFT2D_PF=$pf timeout 300 python tools/stress_conc.py 6 3 >> gpurun_out/pf.txt 2>&1
  SFFT2D_PF=$pf timeout 300 python tools/fold_bw.py 2>&1 | grep "B=" >> gpurun_out/pf.txt
done
