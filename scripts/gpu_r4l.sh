# gather A/B on one box: byte loads (HEAD) vs word-loaded runs (FAST only / FAST + compat)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4l; mkdir -p $D
for rep in 1 2; do
for v in main tcruns bytes; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/net_time.py 2>&1 | tail -1
  env $LIB timeout 300 python scripts/enc_time.py kaiming 3 2>&1 | tail -1
done; done | tee $D/gather_ab.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > $D/pytest_parity.log 2>&1; echo "tests rc $?"; tail -2 $D/pytest_parity.log
