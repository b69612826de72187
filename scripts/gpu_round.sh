timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
python scripts/tree_prof.py 2>&1 | tail -1
python scripts/tree_prof.py 1000000 uniform 1e-9 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r26.json 2> gpurun_out/bench_r26.err; tail -2 gpurun_out/bench_r26.err
python scripts/configs_timing.py --only config2 --reps 3
