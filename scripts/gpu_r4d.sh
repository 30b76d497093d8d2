# Raster-order gather in both encoder networks (compat k_enc_net, FAST k_enc_net_tc2):
# parity suite, then A/B vs the previous build
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4d; mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -x > $D/pytest_parity.log 2>&1; echo "tests rc $?"; tail -2 $D/pytest_parity.log
for v in main prev main prev; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/net_time.py 2>&1 | tail -1
  env $LIB timeout 300 python scripts/enc_time.py kaiming 3 2>&1 | tail -1
done | tee $D/enc_ab.txt
