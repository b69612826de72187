# r02 (late) state check + profiling round (tag $1): GPU tests, smoke, bench line,
# per-config timings, ncu launch list, ncu --set full of the step's kernels (serial
# stages), each ncu run after the plain run exited 0.
T=${1:-v7}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest_$T.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02_gputest_$T.log
tail -3 gpurun_out/r02_gputest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_$T.log 2>&1; echo "smoke exit $?"
set -e
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_$T.json 2> gpurun_out/r02_bench_$T.err
python scripts/configs_timing.py --reps 3 > gpurun_out/r02_configs_$T.jsonl 2> gpurun_out/r02_configs_$T.err || true
python scripts/prof_step.py --reps 2 > gpurun_out/r02_plain_$T.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_$T.csv \
    python scripts/prof_step.py --reps 2 > gpurun_out/r02_ncu_launch_$T.log 2>&1
DMK_SERIAL=1 ncu --set full --clock-control none --import-source on \
    -k "regex:k_p2p32|k_p2p_psum|k_anterp|k_eval|k_pwshift|k_pw2poly32|k_prox2pw32|k_c2p_grp|k_p2c_grp" -c 24 \
    -o gpurun_out/r02_prof_$T python scripts/prof_step.py --reps 1 > gpurun_out/r02_ncu_full_$T.log 2>&1
tail -3 gpurun_out/r02_bench_$T.err
