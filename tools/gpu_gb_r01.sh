set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "groupby or smoke or launch" > gpurun_out/gpu_tests4.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests4.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo rc=$? >> gpurun_out/bench4.err
