for NT in 128 256; do for NS in 1 2 3; do
  echo "NT=$NT NS=$NS" >> gpurun_out/ns.log
  TQP_DENSE_NT=$NT TQP_DENSE_NS=$NS timeout 300 python tools/opbench.py 10 q1_groupby 2>&1 | grep "^q1" | cut -c1-130 >> gpurun_out/ns.log
done; done
echo "auto" >> gpurun_out/ns.log
timeout 300 python tools/opbench.py 10 q1_groupby 2>&1 | grep "^q1" | cut -c1-130 >> gpurun_out/ns.log
timeout 600 python -m pytest tests -m gpu -q -x -k "groupby or q1" > gpurun_out/ns_tests.log 2>&1
