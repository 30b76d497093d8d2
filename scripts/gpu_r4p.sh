# FAST float32 table kernel at 4 blocks/SM (A/B)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4p; mkdir -p $D
for v in main f32m4 main f32m4; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/enc_time.py kaiming 3 fast 2>&1 | tail -1
done | tee $D/enc_fast_ab.txt
