# A/B of a compile-time switch on the sort ops: bash tools/ab_sort.sh "<flags A>" "<flags B>" [ops]
OPS=${3:-sort_build,sort_probe,smj_join}
for V in "$1" "$2"; do
  TQP_NVCC_EXTRA="$V" python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_2203_01877_b200/build.py'); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)" || exit 1
  echo "== $V" >> gpurun_out/ab.log
  timeout 600 python tools/opbench.py 10 $OPS 2>&1 | grep -v "^{" | cut -c1-300 >> gpurun_out/ab.log
done
# restore the default build (the stamp would also force it on the next build())
python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_2203_01877_b200/build.py'); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)"
