# A/B of the symmetric near field's tail handling (libdmk_base: none, libdmk: skip
# records past a chunk's tail, libdmk_rs: + skip records with no in-ball pair):
# parity tests with the default library, serial stage times per library
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "p2p or near or config0 or direct" 2>&1 | tail -2
for v in base "" rs; do
  L=paper_2308_00292_b200/libdmk${v:+_$v}.so
  [ -f $L ] || continue
  echo "== $L"
  DMK_LIB=$PWD/$L python scripts/stage_times.py uniform 1e6 1e-6 laplace 4 2>&1 | tail -2 | tee -a gpurun_out/p2p_tail_${v:-tail}.jsonl
  DMK_LIB=$PWD/$L python scripts/stage_times.py clusters 1e7 1e-6 laplace 3 2>&1 | tail -1 | tee -a gpurun_out/p2p_tail_${v:-tail}.jsonl
done
