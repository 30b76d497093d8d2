# session-5: in-situ decoder ablations at C2 (what bounds k_decode2): Phi replaced by a linear stub (ABL_NOPHI), deficit selection skipped (ABL_NOSEL); garbage decodes, timing only
cd $GRAFT_REPO_ROOT
D=gpurun_out/r5e; mkdir -p $D
for rep in 1 2; do
  timeout 300 python scripts/dec_time_abl.py kaiming 2 2>&1 | tail -2
  LPIC_LIB=paper_2212_01185_b200/ab/nophi.so timeout 300 python scripts/dec_time_abl.py kaiming 2 2>&1 | tail -2
  LPIC_LIB=paper_2212_01185_b200/ab/nosel.so timeout 300 python scripts/dec_time_abl.py kaiming 2 2>&1 | tail -2
done | tee $D/dec_ablation.txt
