# A/B of compile-time variants with a parity check of each: builds the variant, runs the
# selected GPU tests, then opbench on one scale factor; restores the default build.
#   bash tools/ab_tests.sh <sf> <ops> "<pytest -k expr>" "<flags 1>" "<flags 2>" ...
SF=$1; OPS=$2; K=$3; shift 3
B='import importlib.util as u; s=u.spec_from_file_location("b","paper_2203_01877_b200/build.py"); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)'
for V in "$@"; do
  TQP_NVCC_EXTRA="$V" python -c "$B" || exit 1
  echo "== $V sf=$SF" >> gpurun_out/ab.log
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" 2>&1 | tail -2 >> gpurun_out/ab.log
  timeout 600 python tools/opbench.py $SF $OPS 2>&1 | grep -v "^{" | cut -c1-400 >> gpurun_out/ab.log
done
python -c "$B"
