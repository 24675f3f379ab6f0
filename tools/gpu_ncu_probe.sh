CMD="python tools/opbench.py 10 pkfk_small_build,pkfk_join"
timeout 600 $CMD > gpurun_out/n61_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:probe_kernel -c 1 -o gpurun_out/p61_small $CMD > gpurun_out/n61_s.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:probe_kernel -s 8 -c 1 -o gpurun_out/p61_full $CMD > gpurun_out/n61_f.log 2>&1
