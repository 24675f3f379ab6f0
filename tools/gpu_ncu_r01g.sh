CMD="python tools/opbench.py 10"
timeout 600 $CMD > gpurun_out/n32_plain.log 2>&1 || exit 1
# sort_probe: sort_build runs 7 x 3 scatter launches first
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scatter_tma -s 22 -c 1 -o gpurun_out/p32_scatter $CMD > gpurun_out/n32_sc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gb_phase1 -c 1 -o gpurun_out/p32_gbq1 $CMD > gpurun_out/n32_gb.log 2>&1
