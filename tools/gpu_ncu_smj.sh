CMD="python tools/opbench.py 10 smj_join"
timeout 600 $CMD > gpurun_out/n76_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"intersect_kernel|common_kernel|tile_bounds" -c 3 -o gpurun_out/p76_int $CMD > gpurun_out/n76_i.log 2>&1
