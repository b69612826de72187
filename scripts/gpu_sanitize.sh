# compute-sanitizer (memcheck, racecheck) over one small step of each tier / kernel
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck; do
  for cfg in "--n 30000 --eps 1e-9" "--n 30000 --eps 1e-6" "--n 30000 --eps 1e-3 --kind clusters" "--n 20000 --eps 1e-6 --kernel yukawa --kind clusters" "--n 20000 --eps 1e-9 --kernel log --kind circle2d"; do
    echo "== $tool $cfg"
    timeout 600 $S --tool $tool --print-limit 5 python scripts/prof_step.py --reps 1 --ns 60 $cfg 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Invalid|hazard|rep 0" | head -8
  done
done 2>&1 | tee gpurun_out/sanitize.log
