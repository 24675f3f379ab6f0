CMD="python tools/opbench.py 10"
timeout 600 $CMD > gpurun_out/n26_plain.log 2>&1 || exit 1
for K in gb_phase1 probe_kernel filter_kernel rle_kernel expand_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/p26_$K $CMD > gpurun_out/n26_$K.log 2>&1
done
