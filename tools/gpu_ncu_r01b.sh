set -x
CMD="python tools/opbench.py 10"
timeout 600 $CMD > gpurun_out/n8_plain.log 2>&1 || exit 1
for K in gb_phase1 probe_kernel intersect_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/n8_$K.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:onesweep -s 8 -c 2 -o gpurun_out/prof_onesweep $CMD > gpurun_out/n8_onesweep.log 2>&1
