# session-5: isolated chain builder at HEAD (cycles per table) and its per-phase split (-DPROF build)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r5g; mkdir -p $D
timeout 180 ./scripts/ubench_chain > $D/ubench_chain.log 2>&1; echo "chain rc $?"; grep -E "cycles per table|TOTAL" $D/ubench_chain.log | head
timeout 180 ./scripts/ubench_chain_prof > $D/ubench_chain_prof.log 2>&1; echo "prof rc $?"; grep -E "cycles" $D/ubench_chain_prof.log | tail -32
