# translation / back-transform forms: parity tests, then serial stage times at config 1
# (eps = 1e-9: DMK_PW64 = box | group | staged; fp32 tier: DMK_PWS = reg | staged)
T=${1:-v1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pw64 or pws_staged" > gpurun_out/r02_pwforms_test_$T.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02_pwforms_test_$T.log
tail -3 gpurun_out/r02_pwforms_test_$T.log
timeout 600 python scripts/stage_forms.py DMK_PW64 box,group,staged --eps 1e-9 --no-err > gpurun_out/r02_pw64_forms_$T.jsonl 2>&1
timeout 600 python scripts/stage_forms.py DMK_PWS reg,staged --eps 1e-6,1e-3 --no-err > gpurun_out/r02_pws_forms_$T.jsonl 2>&1
cat gpurun_out/r02_pw64_forms_$T.jsonl gpurun_out/r02_pws_forms_$T.jsonl | cut -c1-600
if [ -n "$NCU" ]; then
  DMK_SERIAL=1 ncu --set full --clock-control none --import-source on -k "regex:k_pwshift_s|k_pw2poly64|k_prox2pw" -c 4 \
      -o gpurun_out/r02_prof_pw64_$T python scripts/prof_step.py --eps 1e-9 --reps 1 > gpurun_out/r02_ncu_pw64_$T.log 2>&1
  tail -2 gpurun_out/r02_ncu_pw64_$T.log
fi
