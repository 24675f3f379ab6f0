for W in 1 0; do
  echo "L2W=$W" >> gpurun_out/l2.log
  TQP_L2_WINDOW=$W timeout 300 python tools/opbench.py 10 pkfk_join,smj_join,q1_groupby 2>&1 | grep -E "^(pkfk|smj|q1)" | cut -c1-160 >> gpurun_out/l2.log
  TQP_L2_WINDOW=$W timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python tools/show.py | head -2 >> gpurun_out/l2.log
done
timeout 600 python -m pytest tests -m gpu -q -x -k "pkfk or smoke" > gpurun_out/l2_tests.log 2>&1
