CMD="python tools/opbench.py 10 sort_probe"
timeout 600 $CMD > gpurun_out/n59_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scatter -s 1 -c 1 -o gpurun_out/p59_scatter $CMD > gpurun_out/n59_s.log 2>&1
