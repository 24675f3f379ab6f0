CMD="python tools/opbench.py 10"
timeout 600 $CMD > gpurun_out/n19_plain.log 2>&1 || exit 1
# sort_probe: skip sort_build (7 calls x 4 passes = 28 scatter launches) + 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scatter_kernel -s 29 -c 1 -o gpurun_out/prof_scatter $CMD > gpurun_out/n19_sc.log 2>&1
