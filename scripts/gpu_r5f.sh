# session-5: Phi ablation with a logistic stub (-DABL_NOPHI, Kaiming-like table shapes, no fp64 polynomial); timing only
cd $GRAFT_REPO_ROOT
D=gpurun_out/r5f; mkdir -p $D
for rep in 1 2; do
  timeout 300 python scripts/dec_time_abl.py kaiming 2 2>&1 | tail -2
  LPIC_LIB=paper_2212_01185_b200/ab/nophi2.so timeout 300 python scripts/dec_time_abl.py kaiming 2 2>&1 | tail -2
done | tee $D/dec_ablation_phi.txt
