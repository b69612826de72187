# ncu --set full of chosen kernels at config 1 (serial streams), source-level
#   bash scripts/gpu_ncu_kernels.sh <tag> <kernel regex> <count> [prof_step args...]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=$1; RX=$2; CNT=$3; shift 3
DMK_SERIAL=1 timeout 900 ncu --set full --clock-control none --import-source on \
    -k "regex:$RX" -c $CNT -o gpurun_out/ncu_$TAG python scripts/prof_step.py --reps 1 "$@" > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
