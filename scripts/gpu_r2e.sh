# Round 2 iteration e: pipelined tcgen05 FAST encoder network (k_enc_net_tc2).
# FAST tests first (bitwise enc/dec agreement), then the FAST bench (A/B vs
# the serial tile kernel), ncu of k_enc_net_tc2 and of the unfused table kernel.
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2e; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fast" > $D/pytest_fast.log 2>&1; echo "fast tests rc $?"; tail -3 $D/pytest_fast.log
timeout 900 python bench.py --precision fast --steps 3 --no-cpu-baseline --parity-images 0 > $D/bench_fast.log 2>&1; echo "fast bench rc $?"; grep '^{' $D/bench_fast.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'net', d['encode_network'])"
LPIC_TC_V1=1 timeout 900 python bench.py --precision fast --steps 3 --no-cpu-baseline --parity-images 0 > $D/bench_fast_v1.log 2>&1; echo "fast v1 bench rc $?"; grep '^{' $D/bench_fast_v1.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'net', d['encode_network'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_net_tc2 -c 1 -o $D/encnet_tc2_c2 python scripts/enc_fast.py > $D/ncu_tc2.log 2>&1; echo "ncu tc2 rc $?"; tail -2 $D/ncu_tc2.log
LPIC_RC_UNFUSED=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_tables -c 1 -o $D/enctab_c2_unfused python scripts/enc_c2.py 24 > $D/ncu_enctab.log 2>&1; echo "ncu enctab rc $?"
timeout 2400 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $D/pytest_gpu.log
