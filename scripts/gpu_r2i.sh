# Round 2 iteration i: common-path histogram without match (revert), crowded
# buckets via per-warp radix in the chain; tc2 with smem bias, 16-col chunks.
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2i; mkdir -p $D
timeout 180 ./scripts/ubench_chain > $D/ubench_chain.log 2>&1; echo "chain rc $?"; grep -E "cycles per table|TOTAL" $D/ubench_chain.log
timeout 180 ./scripts/ubench_chain_prof > $D/ubench_chain_prof.log 2>&1; echo "prof rc $?"; grep -E "flat S|flat Q" $D/ubench_chain_prof.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fast or flat or seam" > $D/pytest_sel.log 2>&1; echo "sel tests rc $?"; tail -3 $D/pytest_sel.log
timeout 900 python bench.py --steps 3 > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'chain', d.get('chain',{}).get('frac'), 'parity', d.get('parity',{}).get('byte_identical'), 'cpu', d.get('cpu_baseline',{}).get('value'))"
timeout 900 python bench.py --weights flat --steps 2 --no-cpu-baseline --parity-images 1 > $D/bench_flat.log 2>&1; echo "flat bench rc $?"; grep '^{' $D/bench_flat.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'bpsp', d['bpsp'])"
timeout 900 python bench.py --precision fast --steps 3 --no-cpu-baseline --parity-images 0 > $D/bench_fast.log 2>&1; echo "fast bench rc $?"; grep '^{' $D/bench_fast.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'net', d['encode_network']['ms'], d['encode_network']['model_tflops'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_net_tc2 -c 1 -o $D/encnet_tc2_c2 python scripts/enc_fast.py > $D/ncu_tc2.log 2>&1; echo "ncu tc2 rc $?"
