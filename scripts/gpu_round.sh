# scratch helper for one gpurun call (edited per experiment): launch lists of the
# eps = 1e-9 (p = 28) tier and of config 2 (1e7 clustered points)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_p28_v9.csv \
    python scripts/prof_step.py --reps 2 --eps 1e-9 > gpurun_out/ncu_p28.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_v9.csv \
    python scripts/prof_step.py --reps 2 --n 10000000 --kind clusters > gpurun_out/ncu_c2.log 2>&1
tail -1 gpurun_out/ncu_p28.log; tail -1 gpurun_out/ncu_c2.log
