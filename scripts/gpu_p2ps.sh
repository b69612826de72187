cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "p2p or determin or far_and_near or config1" 2>&1 | tail -3
timeout 300 python scripts/p2p_forms.py --forms sym,queue --cases uniform:1000000:1e-6,clusters:10000000:1e-6 2>&1 | cut -c1-200
