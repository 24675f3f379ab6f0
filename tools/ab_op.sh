# A/B of a compile-time switch on one scale factor: bash tools/ab_op.sh "<flags A>" "<flags B>" <sf> <ops>
for V in "$1" "$2"; do
  TQP_NVCC_EXTRA="$V" python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_2203_01877_b200/build.py'); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)" || exit 1
  echo "== $V sf=$3" >> gpurun_out/ab.log
  timeout 600 python tools/opbench.py $3 $4 2>&1 | grep -v "^{" | cut -c1-300 >> gpurun_out/ab.log
done
