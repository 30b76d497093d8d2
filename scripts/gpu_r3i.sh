# reciprocal-free near-one scale: exhaustive-ish check, parity suite, A/B vs HEAD (prev)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r3i; mkdir -p $D
timeout 300 ./scripts/check_scale > $D/check_scale.log 2>&1; echo "check rc $?"; cat $D/check_scale.log
timeout 180 ./scripts/ubench_chain > $D/ubench_chain.log 2>&1; echo "chain rc $?"; grep -E "K=3: |TOTAL" $D/ubench_chain.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -x > $D/pytest_parity.log 2>&1; echo "tests rc $?"; tail -2 $D/pytest_parity.log
for v in main prev main prev; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/dec_time.py kaiming 3 2>&1 | tail -1
done | tee $D/dec_ab.txt
for v in main prev; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/enc_time.py kaiming 3 2>&1 | tail -1
done | tee $D/enc_ab.txt
