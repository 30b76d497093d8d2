# session-5 refresh of the per-config table at HEAD: C3 (strong, 256 images on one GPU), C4 tiles, C5, fitted and flat C2, gray
cd $GRAFT_REPO_ROOT
D=gpurun_out/r5b; mkdir -p $D
summ() { grep '^{' $1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); e=d.get('encode') or {}; print('$2', 'dec', round(d['value'],2), 'enc', round(e.get('value',0) or 0,1), 'bpsp', d.get('bpsp'), 'parity', (d.get('parity') or {}).get('byte_identical'), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for c in c3 c4 c5-64 c5-4096; do
  timeout 1200 python bench.py --config $c --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $D/bench_$c.log 2>&1; echo "$c rc $?"; summ $D/bench_$c.log $c
done
for wt in fitted flat; do
  timeout 900 python bench.py --weights $wt --steps 5 --e2e-steps 1 --no-cpu-baseline > $D/bench_c2_$wt.log 2>&1; echo "$wt rc $?"; summ $D/bench_c2_$wt.log c2-$wt
done
timeout 900 python bench.py --gray --steps 5 --e2e-steps 1 --no-cpu-baseline > $D/bench_c2_gray.log 2>&1; echo "gray rc $?"; summ $D/bench_c2_gray.log c2-gray
