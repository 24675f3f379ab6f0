# Checked run (compute-sanitizer is closed on this GPU pool): libtqp built with
# -DTQP_CHECKED=1 (device bounds checks that trap on the computed store indices of the
# scatter, compaction, partition, expansion and partial-record kernels) and run with
# TQP_ALLOC_EXACT=1 (every temporary its own cudaMalloc + 256 canary bytes checked at
# release; tests/conftest.py asserts none was overwritten) and TQP_ALLOC_POISON=1 (every
# temporary filled with 0xA5 garbage when handed out, so reads of unwritten temporaries
# are deterministic failures), over the -m gpu tests at their small sizes. Then the
# default build is restored.
# Usage (on the GPU box): bash tools/gpu_checked.sh
SMALL="not large and not sf1 and not sf10 and not full_size and not zipf_uniform and not both_zipf and not q1_parity and not scale"
TQP_NVCC_EXTRA="-DTQP_CHECKED=1" python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_2203_01877_b200/build.py'); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)" || exit 1
TQP_ALLOC_EXACT=1 TQP_ALLOC_POISON=1 timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$SMALL" > gpurun_out/checked_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/checked_pytest.log
grep -c "TQP_DCHECK failed" gpurun_out/checked_pytest.log >> gpurun_out/checked_pytest.log
python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_2203_01877_b200/build.py'); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)"
