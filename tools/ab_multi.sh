# A/B of several compile-time variants on one scale factor:
#   bash tools/ab_multi.sh <sf> <ops> "<flags 1>" "<flags 2>" ...
SF=$1; OPS=$2; shift 2
for V in "$@"; do
  TQP_NVCC_EXTRA="$V" python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_2203_01877_b200/build.py'); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)" || exit 1
  echo "== $V sf=$SF" >> gpurun_out/ab.log
  timeout 600 python tools/opbench.py $SF $OPS 2>&1 | grep -v "^{" | cut -c1-400 >> gpurun_out/ab.log
done
# restore the default build
python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_2203_01877_b200/build.py'); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)"
