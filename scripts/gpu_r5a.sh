# session-5 check at HEAD from a fresh container build: GPU suite, smoke, default + FAST + reference bench, launch lists
cd $GRAFT_REPO_ROOT
D=gpurun_out/r5a; mkdir -p $D
timeout 2400 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 $D/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc $?"; tail -1 $D/smoke.log
timeout 900 python bench.py > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'e2e', d['e2e']['value'], 'enc', d['encode']['value'], d['encode']['e2e'], 'tc', d.get('encode_network_tcgen05',{}).get('model_tflops'), 'tab', d.get('encode_tables',{}).get('phi_frac'), 'parity', d.get('parity',{}).get('byte_identical'), 'clk', d['clocks'])"
timeout 900 python bench.py --precision fast > $D/bench_fast.log 2>&1; echo "bench fast rc $?"; grep '^{' $D/bench_fast.log | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], d['encode']['e2e'], 'net', d['encode_network']['model_tflops'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $D/ncu_smoke.log 2>&1; echo "ncu smoke rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $D/launches_bench_c2.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 0 > $D/ncu_launches.log 2>&1; echo "launches rc $?"
timeout 900 python bench.py --impl reference > $D/bench_ref.log 2>&1; echo "ref rc $?"; grep '^{' $D/bench_ref.log | tail -1 | cut -c1-300
