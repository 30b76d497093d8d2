# Table kernel occupancy A/B (Phi chains per step QC, blocks per SM MINB);
# parity suite on the main build (FAST restored to two accumulators)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4h; mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -x > $D/pytest_parity.log 2>&1; echo "tests rc $?"; tail -2 $D/pytest_parity.log
timeout 300 python scripts/net_time.py 2>&1 | tail -1 | tee $D/net_time.txt
for rep in 1 2; do
for v in main prev qc4m3 qc8m3 qc2m3 qc4m2; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/enc_time.py kaiming 3 2>&1 | tail -1
done; done | tee $D/enc_ab.txt
for v in main qc4m3 qc8m3; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/enc_time.py fitted 3 2>&1 | tail -1
done | tee $D/enc_ab_fitted.txt
