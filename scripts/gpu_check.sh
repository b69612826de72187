# parity tests (the given -k filter) + serial stage timings at config 1 and eps=1e-9
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_yukawa.py -x -q ${1:+-k "$1"} 2>&1 | tail -2
timeout 300 python scripts/tree_prof.py 1000000 uniform 1e-6 2>&1 | tail -1
timeout 300 python scripts/tree_prof.py 1000000 uniform 1e-9 2>&1 | tail -1
