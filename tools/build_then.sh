# build libtqp here; print ptxas errors and stop non-zero on failure
python - <<'PY'
import subprocess, sys
import paper_2203_01877_b200.build as b
try:
    b.build(verbose=False)
except Exception as e:
    print("BUILD FAILED:", str(e)[-3000:]); sys.exit(1)
print("build ok")
PY
