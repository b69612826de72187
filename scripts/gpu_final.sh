# final round check: all GPU tests, smoke, bench, per-config timings, launch list
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; tail -2 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -3 gpurun_out/final_smoke.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_v9.json 2> gpurun_out/bench_v9.err; tail -2 gpurun_out/bench_v9.err
python scripts/configs_timing.py --reps 3 > gpurun_out/configs_v9.jsonl 2> gpurun_out/configs_v9.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v9.csv \
    python scripts/prof_step.py --reps 2 > gpurun_out/ncu_launch_v9.log 2>&1
DMK_SERIAL=1 ncu --set full --clock-control none --import-source on \
    -k "regex:k_p2p32|k_anterp32|k_eval32|k_pwshift|k_pw2poly32|k_prox2pw32|k_c2p_grp|k_p2c_grp" -c 16 \
    -o gpurun_out/prof_v9 python scripts/prof_step.py --reps 1 > gpurun_out/ncu_full_v9.log 2>&1
