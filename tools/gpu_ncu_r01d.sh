set -x
CMD="python tools/opbench.py 10"
timeout 600 $CMD > gpurun_out/n13_plain.log 2>&1 || exit 1
# sort_probe (60M) runs 2 warmup + 5 reps after sort_build: skip sort_build's 28 onesweep launches + 1 pass
timeout 900 ncu --set full --clock-control none --import-source on -k regex:onesweep -s 29 -c 2 -o gpurun_out/prof_os60 $CMD > gpurun_out/n13_os.log 2>&1
for K in expand_kernel rle_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/n13_$K.log 2>&1
done
