CMD="python tools/opbench.py 10 smj_join"
timeout 600 $CMD > gpurun_out/n68_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rle_kernel -s 3 -c 1 -o gpurun_out/p68_rle $CMD > gpurun_out/n68_r.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:intersect_kernel -c 1 -o gpurun_out/p68_int $CMD > gpurun_out/n68_i.log 2>&1
