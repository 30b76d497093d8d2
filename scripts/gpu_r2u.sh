# iteration u: A/B early target, aux-warp poll interval
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2u; mkdir -p $D
for v in main tgte sleep1k main tgte sleep1k; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/dec_time.py kaiming 3 2>&1 | tail -1
done | tee $D/dec_ab.txt
