set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests3.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests3.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke3.log 2>&1; echo rc=$? >> gpurun_out/smoke3.log
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_launch3.log 2>&1; echo rc=$? >> gpurun_out/ncu_launch3.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gb_phase1|onesweep|probe_kernel|filter_kernel|expand_kernel" -s 2 -c 6 -o gpurun_out/prof_r01 $CMD > gpurun_out/ncu_full3.log 2>&1; echo rc=$? >> gpurun_out/ncu_full3.log
