# FAST network with one accumulator (scale-input-d fold of the split terms):
# parity suite (FAST raw budget, round trips, encoder/decoder raw equality), timing
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4g; mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -x > $D/pytest_parity.log 2>&1; echo "tests rc $?"; tail -2 $D/pytest_parity.log
for i in 1 2; do timeout 300 python scripts/net_time.py 2>&1 | tail -1; done | tee $D/net_time.txt
timeout 900 python bench.py --precision fast --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 0 > $D/bench_fast.log 2>&1; echo "bench fast rc $?"
grep '^{' $D/bench_fast.log | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'net', d['encode_network'])"
