# build libtqp here; print ptxas errors and stop non-zero on failure
python - <<'PY'
import importlib.util, sys
spec = importlib.util.spec_from_file_location("_tqp_build", "paper_2203_01877_b200/build.py")
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
try:
    b.build(verbose=False)
except Exception as e:
    print("BUILD FAILED:", str(e)[-3000:]); sys.exit(1)
print("build ok")
PY
