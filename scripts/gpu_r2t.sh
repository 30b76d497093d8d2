# iteration t: quotient back in the chain search, red search A/B (multiply vs quotient),
# no per-pixel timeline code in production, lazy back-pressure; in-situ profile
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2t; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $D/pytest_parity.log 2>&1; echo "tests rc $?"; tail -2 $D/pytest_parity.log
for v in main redq main redq; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/dec_time.py kaiming 3 2>&1 | tail -1
done | tee $D/dec_ab.txt
LPIC_LIB=paper_2212_01185_b200/ab/prof.so timeout 600 python scripts/dec_timeline.py 512 768 24 > $D/timeline_prof_c2.log 2>&1; echo "rc $?"; head -5 $D/timeline_prof_c2.log; grep -A15 "in-situ" $D/timeline_prof_c2.log
