cd $GRAFT_REPO_ROOT
D=gpurun_out/r3h; mkdir -p $D
for v in main tcp main tcp; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 600 python scripts/net_time.py 2>&1 | tail -1
done | tee $D/tc2_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fast or FAST or tc" > $D/pytest_fast.log 2>&1; echo "tests rc $?"; tail -2 $D/pytest_fast.log
