# FAST tc2: next pair's layer-0 operand gathered during the last layer (A/B vs base)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r3d; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fast or FAST or tc" > $D/pytest_fast.log 2>&1; echo "tests rc $?"; tail -2 $D/pytest_fast.log
for v in main base main base; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 600 python bench.py --precision fast --steps 2 --no-cpu-baseline --parity-images 0 --e2e-steps 1 > $D/bench_fast_$v.log 2>&1
  grep '^{' $D/bench_fast_$v.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'dec', round(d['value'],2), 'enc', round(d['encode']['value'],1), 'net ms', round(d['encode_network']['ms'],3), 'TF', round(d['encode_network']['model_tflops'],1))"
done | tee $D/fast_ab.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_net_tc2 -c 1 -o $D/encnet_tc2 python scripts/enc_fast.py 8 > $D/ncu_tc2.log 2>&1; echo "ncu tc2 rc $?"
