# iteration x: table kernel software pipeline (next pixel's loads); A/B vs session-start build
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2x; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $D/pytest_parity.log 2>&1; echo "tests rc $?"; tail -2 $D/pytest_parity.log
for v in main base main base; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/enc_time.py kaiming 5 2>&1 | tail -1
  env $LIB timeout 300 python scripts/enc_time.py fitted 5 2>&1 | tail -1
done | tee $D/enc_ab.txt
