# Round 2 iteration h: match-aggregated histogram adds (crowded buckets),
# float64 training path + finite_difference_check; flat and default benches,
# chain phase profile on flat tables, full GPU suite with the reference suite.
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2h; mkdir -p $D
timeout 180 ./scripts/ubench_chain > $D/ubench_chain.log 2>&1; echo "chain rc $?"; grep -E "cycles per table|TOTAL" $D/ubench_chain.log
timeout 180 ./scripts/ubench_chain_prof > $D/ubench_chain_prof.log 2>&1; echo "prof rc $?"; grep -E "flat" $D/ubench_chain_prof.log
timeout 900 python bench.py --weights flat --steps 2 --no-cpu-baseline --parity-images 1 > $D/bench_flat.log 2>&1; echo "flat bench rc $?"; grep '^{' $D/bench_flat.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'bpsp', d['bpsp'])"
timeout 900 python bench.py --steps 3 > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'chain', d.get('chain',{}).get('frac'), 'parity', d.get('parity',{}).get('byte_identical'), 'cpu', d.get('cpu_baseline',{}).get('value'))"
LPIC_PARITY_OUT=$D/parity timeout 2400 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $D/pytest_gpu.log; for f in $D/parity/reference_suite_*.txt; do echo "$f: $(grep -E 'passed|failed|error' $f | tail -1)"; done
