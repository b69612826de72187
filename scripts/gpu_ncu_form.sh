# ncu --set full of one near-field form at config 1 (one launch)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
FORM=$1; TAG=$2
DMK_P2P_FORM=$FORM DMK_SERIAL=1 timeout 900 ncu --set full --clock-control none --import-source on \
    -k "regex:k_p2p32" -c 1 -o gpurun_out/ncu_$TAG python scripts/prof_step.py --reps 1 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
