# tc2 diagnostics: time without epilogue work / without MMAs (garbage outputs; timing only)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r3f; mkdir -p $D
for v in main noepi nomma; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 600 python scripts/net_time.py 2>&1 | tail -1
done | tee $D/tc2_diag.txt
