timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "octant or far_and_near or deterministic" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
python scripts/tree_prof.py 10000000 clusters 2>&1 | tail -1
DMK_P2P_FORM=leaf python scripts/tree_prof.py 10000000 clusters 2>&1 | tail -1
python scripts/configs_timing.py --only config2 --reps 3
python scripts/tree_prof.py 2>&1 | tail -1
