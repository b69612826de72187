# prox2pw<28> register-blocked sweeps against the independent-tile form: parity at
# eps = 1e-9 (every stage), then serial stage times of config 1 at eps = 1e-9 per form
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "1e-09" 2>&1 | tail -2
for f in tiles sweep; do
  DMK_PROX2PW=$f python scripts/stage_times.py uniform 1e6 1e-9 laplace 3 2>&1 | tail -2 | sed "s/^{/{\"DMK_PROX2PW\": \"$f\", /" | tee -a gpurun_out/prox2pw_rb.jsonl
done
