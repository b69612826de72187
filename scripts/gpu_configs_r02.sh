# r02 measurement of the other configs (tag $1): per-stage roofline at eps = 1e-9 (bench),
# ncu launch lists and --set full captures of configs 2 (1e7 clusters), 3 (2D log, 1e7
# noisy circle, eps 1e-9) and 4 (Yukawa, 1e8 uniform, one GPU); every ncu command after
# the same command exited 0 without ncu
set -e
T=${1:-v1}
if [ -z "$SKIP_BENCH" ]; then
python bench.py --eps 1e-9 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_eps1e-9_$T.json 2> gpurun_out/r02_bench_eps1e-9_$T.err
fi
K2="regex:k_p2p32s|k_p2p_psum|k_p2p32q|k_anterp32|k_pwshift|k_pw2poly32|k_eval_tc|k_prox2pw32"
K3="regex:k_p2p2|k_anterp2|k_pwlocal2|k_eval2|k_prox2pw2"
K4=$K2
C2="scripts/prof_step.py --reps 1 --n 10000000 --kind clusters"
C3="scripts/prof_step.py --reps 1 --n 10000000 --kind circle2d --kernel log --eps 1e-9"
C4="scripts/prof_step.py --reps 1 --n 100000000 --kind uniform --kernel yukawa --lam 10"
for c in ${CONFIGS:-2 3 4}; do
  eval CMD=\$C$c
  python $CMD > gpurun_out/r02_plain_c${c}_$T.log 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c${c}_$T.csv python $CMD > gpurun_out/r02_ncu_launch_c${c}_$T.log 2>&1
  eval KRX=\$K$c
  DMK_SERIAL=1 ncu --set full --clock-control none -k "$KRX" -c 12 \
      -o /tmp/r02_prof_c${c}_$T python $CMD > gpurun_out/r02_ncu_full_c${c}_$T.log 2>&1
  # summaries only (the reports exceed gpurun's copy-back limit)
  python scripts/ncu_metrics.py /tmp/r02_prof_c${c}_$T.ncu-rep > gpurun_out/r02_ncu_c${c}_$T.txt 2>&1
  python scripts/traffic_json.py /tmp/r02_prof_c${c}_$T.ncu-rep gpurun_out/r02_traffic_c${c}_$T.json "config $c, r02 $T" > /dev/null 2>&1
  rm -f /tmp/r02_prof_c${c}_$T.ncu-rep
done
tail -2 gpurun_out/r02_bench_eps1e-9_$T.err
