# iteration o: digits 0 and 255 counted by a packed REDUX (no same-address
# shared atomics on near-uniform PMFs), tail skip dropped, warp builder keeps
# member ranking.
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2o; mkdir -p $D
timeout 180 ./scripts/ubench_chain > $D/ubench_chain.log 2>&1; echo "chain rc $?"; grep -E "cycles per table|TOTAL" $D/ubench_chain.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > $D/pytest_parity.log 2>&1; echo "parity tests rc $?"; tail -2 $D/pytest_parity.log
timeout 900 python bench.py --steps 3 --no-cpu-baseline --parity-images 1 > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'chain', d.get('chain',{}).get('frac'), 'parity', d.get('parity',{}).get('byte_identical'))"
timeout 900 python bench.py --weights flat --steps 2 --no-cpu-baseline --parity-images 1 > $D/bench_flat.log 2>&1; echo "flat bench rc $?"; grep '^{' $D/bench_flat.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'bpsp', d['bpsp'])"
timeout 900 python bench.py --weights fitted --steps 2 --no-cpu-baseline --parity-images 1 > $D/bench_fitted.log 2>&1; echo "fitted bench rc $?"; grep '^{' $D/bench_fitted.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'bpsp', d['bpsp'], 'parity', d.get('parity',{}).get('byte_identical'))"
