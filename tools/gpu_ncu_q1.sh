CMD="python tools/opbench.py 10 q1_groupby"
timeout 600 $CMD > gpurun_out/n53_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gb_dense_kernel -c 1 -o gpurun_out/p53_dense $CMD > gpurun_out/n53_d.log 2>&1
