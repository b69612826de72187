# symmetric P2P: blocks of DMK_P2PS_BL consecutive tasks per warp visit (L1 locality of a
# leaf's entries) against the round-robin single-task deal: serial stage times
mkdir -p gpurun_out
for v in "" bl4 bl8 bl16; do
  L=paper_2308_00292_b200/libdmk${v:+_$v}.so
  [ -f $L ] || continue
  DMK_LIB=$PWD/$L python scripts/stage_times.py uniform 1e6 1e-6 laplace 4 2>&1 | tail -2 | sed "s/^{/{\"lib\": \"${v:-bl1}\", /" | tee -a gpurun_out/p2ps_bl.jsonl
  DMK_LIB=$PWD/$L python scripts/stage_times.py clusters 1e7 1e-6 laplace 3 2>&1 | tail -1 | sed "s/^{/{\"lib\": \"${v:-bl1}\", /" | tee -a gpurun_out/p2ps_bl.jsonl
done
