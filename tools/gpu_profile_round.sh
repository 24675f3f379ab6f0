# Round profiling: full bench line, reference line, ncu launch list, ncu --set full of the
# top kernels, summarised on the box (gpurun_out/ copies back at most 64 MiB: the big
# .ncu-rep files are reduced to their summaries and deleted).
# Usage (on the GPU box via gpurun): bash tools/gpu_profile_round.sh <tag>
TAG=${1:-r01}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2>> gpurun_out/${TAG}_bench.err
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-sf100"
timeout 600 $CMD > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
for K in tqp_groupby_dense_jit gb_phase1 scatter_tma probe_sector expand_kernel filter_mask bucket_r rank_bitmap andor_hist0 tile_hist; do
  C=2; S=0
  if [ $K = scatter_tma ]; then C=9; S=0; fi   # every scatter launch of one step (the bench averages them all)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C -o gpurun_out/${TAG}_full_$K $CMD > gpurun_out/${TAG}_ncu_full_$K.log 2>&1
done
python tools/profile_summary.py ${TAG} gpurun_out/${TAG}_summary
mkdir -p gpurun_out/${TAG}_reps
for K in tqp_groupby_dense_jit scatter_tma probe_sector expand_kernel; do
  ncu -i gpurun_out/${TAG}_full_$K.ncu-rep --page raw --csv > gpurun_out/${TAG}_reps/${K}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_full_$K.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_reps/${K}_source.csv 2>/dev/null
done
rm -f gpurun_out/${TAG}_full_*.ncu-rep
du -sh gpurun_out
echo done
