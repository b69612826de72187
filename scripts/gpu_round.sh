timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_yukawa.py -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
python scripts/near_err.py 2>&1 | tail -5
python scripts/tree_prof.py 2>&1 | tail -1
DMK_ANTERP_SIMT=1 python scripts/tree_prof.py 2>&1 | tail -1
