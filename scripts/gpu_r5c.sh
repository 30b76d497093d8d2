# session-5: remaining per-config rows at HEAD (FAST C3, C5-512, FAST C5-4096)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r5c; mkdir -p $D
summ() { grep '^{' $1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); e=d.get('encode') or {}; print('$2', 'dec', round(d['value'],2), 'enc', round(e.get('value',0) or 0,1), 'bpsp', d.get('bpsp'), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
timeout 1200 python bench.py --config c3 --precision fast --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 0 > $D/bench_c3_fast.log 2>&1; echo "c3 fast rc $?"; summ $D/bench_c3_fast.log c3-fast
timeout 900 python bench.py --config c5-512 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $D/bench_c5-512.log 2>&1; echo "c5-512 rc $?"; summ $D/bench_c5-512.log c5-512
timeout 900 python bench.py --config c5-4096 --precision fast --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 0 > $D/bench_c5-4096_fast.log 2>&1; echo "c5-4096 fast rc $?"; summ $D/bench_c5-4096_fast.log c5-4096-fast
