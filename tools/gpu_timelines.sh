# per-workload CUPTI timelines (busy / idle / per-kernel) -> gpurun_out/timelines.txt
set -u
mkdir -p gpurun_out
: > gpurun_out/timelines.txt
for w in ${WORKS:-c3 c1 c3sfft c2 c5}; do
  timeout 300 python tools/timeline.py ${PREC:-fp32} 5 $w >> gpurun_out/timelines.txt 2>&1
  echo "---- rc=$? $w" >> gpurun_out/timelines.txt
done
