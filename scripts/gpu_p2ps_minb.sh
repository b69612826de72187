# symmetric P2P register caps (min blocks per SM 5, 6: 96, 80 registers, spilling)
# against the default (128 registers, 4 CTAs per SM): serial stage times
mkdir -p gpurun_out
for v in "" mb5 mb6; do
  L=paper_2308_00292_b200/libdmk${v:+_$v}.so
  [ -f $L ] || continue
  DMK_LIB=$PWD/$L python scripts/stage_times.py uniform 1e6 1e-6 laplace 4 2>&1 | tail -2 | sed "s/^{/{\"lib\": \"${v:-default}\", /" | tee -a gpurun_out/p2ps_minb.jsonl
  DMK_LIB=$PWD/$L python scripts/stage_times.py clusters 1e7 1e-6 laplace 3 2>&1 | tail -1 | sed "s/^{/{\"lib\": \"${v:-default}\", /" | tee -a gpurun_out/p2ps_minb.jsonl
done
