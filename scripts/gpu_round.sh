timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
python scripts/tree_prof.py 2>&1 | tail -1
python scripts/tree_prof.py 10000000 clusters 2>&1 | tail -1
