set -x
PYTEST_K="sort or filter or groupby or smoke" bash tools/gpu_quick.sh
CMD="python tools/opbench.py 10"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gb_phase1 -s 7 -c 1 -o gpurun_out/prof_gb_q6 $CMD > gpurun_out/n11_gbq6.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gb_phase1 -c 1 -o gpurun_out/prof_gb_q1 $CMD > gpurun_out/n11_gbq1.log 2>&1
