# A/B of two builds of the library: the in-tree one, then $ALT copied over it
# (per-pass host times, in-flight throughput, warm per-kernel times of c3)
set -u
mkdir -p gpurun_out
L=paper_1908_02461_b200/libsfft2d_b200.so
: > gpurun_out/lib_ab.txt
for side in new alt; do
  if [ $side = alt ]; then cp ${ALT:-paper_1908_02461_b200/lib_nohints.so} $L; fi
  echo "== $side" >> gpurun_out/lib_ab.txt
  for i in 1 2; do timeout 300 python tools/pass_host.py fp32 2>&1 | tail -7 >> gpurun_out/lib_ab.txt; done
  timeout 300 python tools/stress_conc.py 6 3 >> gpurun_out/lib_ab.txt 2>&1
  timeout 300 python tools/timeline.py fp32 5 c3 2>&1 | grep -E "host wall|busy|k_fft|k_pass_conv|k_lmax_stream" >> gpurun_out/lib_ab.txt
done
