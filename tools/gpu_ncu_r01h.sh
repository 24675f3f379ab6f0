CMD="python tools/opbench.py 10 q6_sum,q6_filter"
timeout 600 $CMD > gpurun_out/n41_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gb_phase1 -c 1 -o gpurun_out/p41_q6 $CMD > gpurun_out/n41_q6.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:filter_kernel -c 1 -o gpurun_out/p41_filter $CMD > gpurun_out/n41_f.log 2>&1
