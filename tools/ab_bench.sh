# A/B of compile-time variants on the whole bench step (2 streams, SF10):
#   bash tools/ab_bench.sh "<flags 1>" "<flags 2>" ...   (each variant twice, interleaved)
B='import importlib.util as u; s=u.spec_from_file_location("b","paper_2203_01877_b200/build.py"); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)'
for R in 1 2; do
for V in "$@"; do
  TQP_NVCC_EXTRA="$V" python -c "$B" > /dev/null || exit 1
  L=$(timeout 600 python bench.py --steps 20 --warmup 3 --no-sf100 --no-cpu-baseline 2>/dev/null | tail -1)
  echo "== $V run $R: $(echo "$L" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), d["operators_ms"])')" >> gpurun_out/ab_bench.log
done
done
python -c "$B" > /dev/null
