# quick GPU check: parity subset + bench + per-operator timings
set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/q_tests.log 2>&1; echo rc=$? >> gpurun_out/q_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo rc=$? >> gpurun_out/q_bench.err
timeout 600 python tools/opbench.py 10 > gpurun_out/q_opbench.log 2>&1; echo rc=$? >> gpurun_out/q_opbench.log
