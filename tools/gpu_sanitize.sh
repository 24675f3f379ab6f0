# NOTE: compute-sanitizer is refused on this GPU pool (profiles/sanitizer_refused_r02.txt);
# tools/gpu_checked.sh is the substitute that runs.
# compute-sanitizer over every libtqp kernel (SURVEY.md §5 / VERDICT r01 missing #5).
# Runs the -m gpu parity tests at their small sizes (<= ~1M rows; the SF1/SF10/100M cases are
# excluded) under memcheck, racecheck and synccheck, checking only libtqp's kernels
# (mangled names contain "3tqp"; torch's datagen kernels run unchecked). TQP_ALLOC_EXACT=1
# makes every libtqp temporary its own exact-size cudaMalloc so memcheck sees overruns that
# a cached block would hide. Logs: gpurun_out/san_<tool>.log (+ pytest output).
# Usage (on the GPU box): bash tools/gpu_sanitize.sh [tools...]
TOOLS=${*:-memcheck racecheck synccheck}
SAN=/usr/local/cuda/bin/compute-sanitizer
SMALL="not large and not sf1 and not sf10 and not full_size and not zipf and not q1_parity and not scale"
export TQP_ALLOC_EXACT=1
for T in $TOOLS; do
  case $T in
    memcheck) K="$SMALL"; TO=1500; EXTRA="--leak-check no" ;;
    racecheck) K="$SMALL and (sort_parity or pkfk_random or pkfk_presorted or smj_random or smj_key_domains or filter_random or groupby_random or groupby_dense or groupby_q6 or groupby_spec or groupby_high_cardinality or groupby_f64_aggregates or pkfk_outer or pkfk_semi or merge or pack_keys or multipass or partition or exchange)"; TO=1200; EXTRA="--racecheck-report all" ;;
    synccheck) K="$SMALL"; TO=900; EXTRA="" ;;
  esac
  timeout $TO $SAN --tool $T $EXTRA --kernel-name kns=3tqp --print-limit 50 --error-exitcode 99 \
      --log-file gpurun_out/san_$T.%p.log \
      python -m pytest tests -m gpu -q -p no:cacheprovider -k "$K" > gpurun_out/san_${T}_pytest.log 2>&1
  echo "tool=$T rc=$?" | tee -a gpurun_out/san_summary.txt
  grep -hE "ERROR SUMMARY|RACECHECK SUMMARY|hazard" gpurun_out/san_$T.*.log | sort | uniq -c | head -20 >> gpurun_out/san_summary.txt
  tail -3 gpurun_out/san_${T}_pytest.log >> gpurun_out/san_summary.txt
done
