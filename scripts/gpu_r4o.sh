# bench line with the encode_tables key (encoder Phi roofline)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4o; mkdir -p $D
timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 1 > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'tables', d.get('encode_tables'))"
timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --gray --config c5-64 --no-cpu-baseline > $D/bench_gray.log 2>&1; echo "bench gray rc $?"; grep '^{' $D/bench_gray.log | tail -1 | cut -c1-300
