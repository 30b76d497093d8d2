# iteration z: crowded pick inlined (A/B), vs main (noinline) 
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2z; mkdir -p $D
timeout 180 ./scripts/ubench_chain_prof > $D/prof.log 2>&1; grep -E "flat S|flat: |K=3: " $D/prof.log
timeout 180 ./scripts/ubench_chain_prof_inl > $D/prof_inl.log 2>&1; grep -E "flat S|flat: |K=3: |TOTAL" $D/prof_inl.log
for v in main cinl main cinl; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/dec_time.py kaiming 3 2>&1 | tail -1
done | tee $D/dec_ab.txt
for v in main cinl; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/enc_time.py kaiming 5 2>&1 | tail -1
  env $LIB timeout 300 python scripts/dec_time.py flat 2 2>&1 | tail -1
done | tee $D/misc_ab.txt
LPIC_LIB=paper_2212_01185_b200/ab/cinl.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $D/pytest_parity_cinl.log 2>&1; echo "tests cinl rc $?"; tail -2 $D/pytest_parity_cinl.log
