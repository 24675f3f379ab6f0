# One ncu --set full capture of one kernel while running one opbench operator.
# usage (on the GPU box via gpurun): bash tools/gpu_ncu_kernel.sh <op> <kernel-regex> <tag> [skip] [count]
#   e.g. bash tools/gpu_ncu_kernel.sh q1_groupby gb_dense_kernel q1dense
OP=$1; K=$2; TAG=$3; SKIP=${4:-0}; CNT=${5:-1}
CMD="python tools/opbench.py 10 $OP"
timeout 600 $CMD > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $SKIP -c $CNT \
    -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
