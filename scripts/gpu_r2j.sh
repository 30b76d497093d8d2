# Round 2 session 2 baseline at HEAD: chain ubench, full GPU suite (with the
# reference suite), default / flat / FAST benches.
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2j; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/smi.txt 2>&1
timeout 180 ./scripts/ubench_chain > $D/ubench_chain.log 2>&1; echo "chain rc $?"; grep -E "cycles per table|TOTAL" $D/ubench_chain.log
timeout 180 ./scripts/ubench_chain_prof > $D/ubench_chain_prof.log 2>&1; echo "prof rc $?"
timeout 900 python bench.py --steps 3 > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'chain', d.get('chain',{}).get('frac'), 'parity', d.get('parity',{}).get('byte_identical'), 'cpu', d.get('cpu_baseline',{}).get('value'))"
timeout 900 python bench.py --weights flat --steps 2 --no-cpu-baseline --parity-images 1 > $D/bench_flat.log 2>&1; echo "flat bench rc $?"; grep '^{' $D/bench_flat.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'bpsp', d['bpsp'])"
timeout 900 python bench.py --precision fast --steps 3 --no-cpu-baseline --parity-images 0 > $D/bench_fast.log 2>&1; echo "fast bench rc $?"; grep '^{' $D/bench_fast.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'net', d['encode_network']['ms'], d['encode_network']['model_tflops'])"
LPIC_PARITY_OUT=$D/parity timeout 2700 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $D/pytest_gpu.log
