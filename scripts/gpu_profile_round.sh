# one profiling round: bench line, per-config timings, ncu launch list, ncu --set full of
# the top kernels (each under its own command, after the plain run exited 0)
set -e
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_v6.json 2> gpurun_out/bench_v6.err
python scripts/configs_timing.py --reps 3 > gpurun_out/configs_v6.jsonl 2> gpurun_out/configs_v6.err || true
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v6.csv \
    python scripts/prof_step.py --reps 2 > gpurun_out/ncu_launch_v6.log 2>&1
DMK_SERIAL=1 ncu --set full --clock-control none --import-source on \
    -k "regex:k_p2p32|k_anterp32|k_eval32|k_pwshift|k_pw2poly32|k_prox2pw32|k_c2p_grp|k_p2c_grp" -c 16 \
    -o gpurun_out/prof_v6 python scripts/prof_step.py --reps 1 > gpurun_out/ncu_full_v6.log 2>&1
tail -3 gpurun_out/bench_v6.err
