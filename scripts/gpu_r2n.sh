# iteration n: encoder A/B (tail skip, list ranking), FAST tc2 with paired
# TMEM loads (time + ncu full capture).
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2n; mkdir -p $D
for k in kaiming fitted; do
  for v in main notail oldexact both; do
    if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
    env $LIB timeout 300 python scripts/enc_time.py $k 5 2>&1 | tail -1
  done
done | tee $D/enc_ab.txt
timeout 300 python scripts/enc_time.py kaiming 5 fast 2>&1 | tail -1 | tee $D/enc_fast.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fast" > $D/pytest_fast.log 2>&1; echo "fast tests rc $?"; tail -2 $D/pytest_fast.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_net_tc2 -c 1 -o $D/encnet_tc2 python scripts/enc_fast.py 8 > $D/ncu_tc2.log 2>&1; echo "ncu tc2 rc $?"
