# crowded pick by one warp (A/B vs all four warps)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r3a; mkdir -p $D
timeout 180 ./scripts/ubench_chain > $D/ubench_chain.log 2>&1; echo "chain rc $?"; grep -E "cycles per table|TOTAL" $D/ubench_chain.log
timeout 180 ./scripts/ubench_chain_prof > $D/prof.log 2>&1; grep -E "flat S|flat: " $D/prof.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $D/pytest_parity.log 2>&1; echo "tests rc $?"; tail -2 $D/pytest_parity.log
for v in main allw main allw; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/dec_time.py kaiming 3 2>&1 | tail -1
done | tee $D/dec_ab.txt
for v in main allw; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/dec_time.py flat 2 2>&1 | tail -1
  env $LIB timeout 300 python scripts/dec_time.py fitted 2 2>&1 | tail -1
done | tee $D/misc_ab.txt
