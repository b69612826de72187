# final round check: all GPU tests, smoke, bench, per-config timings, launch list
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; tail -2 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -3 gpurun_out/final_smoke.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_v8.json 2> gpurun_out/bench_v8.err; tail -2 gpurun_out/bench_v8.err
python scripts/configs_timing.py --reps 3 > gpurun_out/configs_v8.jsonl 2> gpurun_out/configs_v8.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v8.csv \
    python scripts/prof_step.py --reps 2 > gpurun_out/ncu_launch_v8.log 2>&1
