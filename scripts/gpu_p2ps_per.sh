# overlapped step time against the number of resident symmetric-P2P CTAs per SM
# (DMK_P2PS_PER: 64 = all that fit (4), 0 = one task per warp, non-persistent grid)
mkdir -p gpurun_out
for per in 64 3 2 1 0; do
  echo "== DMK_P2PS_PER=$per"
  DMK_P2PS_PER=$per python scripts/configs_timing.py --reps 6 --only "config1 laplace uniform 1e6 eps1e-6|config1 laplace uniform 1e6 eps1e-3|config2" 2>&1 | \
    sed "s/^{/{\"DMK_P2PS_PER\": $per, /" | tee -a gpurun_out/p2ps_per.jsonl
done
