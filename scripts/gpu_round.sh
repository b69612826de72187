set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_yukawa.py -x -q 2>&1 | tail -5
python scripts/near_err.py 2>&1 | tail -8
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_pws.json 2> gpurun_out/bench_pws.err; tail -3 gpurun_out/bench_pws.err
