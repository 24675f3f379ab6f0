CMD="python tools/opbench.py 10 q1_groupby"
timeout 600 $CMD > gpurun_out/n45_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gb_phase1 -c 1 -o gpurun_out/p45_q1 $CMD > gpurun_out/n45_q1.log 2>&1
