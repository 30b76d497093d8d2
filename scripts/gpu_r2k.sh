# Round 2 session 2, iteration k: adaptive-digit crowded-bucket selection;
# exact selection test; flat / default benches; ncu source capture of k_decode2 (C2).
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2k; mkdir -p $D
timeout 180 ./scripts/ubench_chain > $D/ubench_chain.log 2>&1; echo "chain rc $?"; grep -E "cycles per table|TOTAL" $D/ubench_chain.log
timeout 180 ./scripts/ubench_chain_prof > $D/ubench_chain_prof.log 2>&1; echo "prof rc $?"; grep -E "flat S|cycles per table" $D/ubench_chain_prof.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "flat or selection or seam or cdfs" > $D/pytest_sel.log 2>&1; echo "sel tests rc $?"; tail -3 $D/pytest_sel.log
timeout 900 python bench.py --weights flat --steps 2 --no-cpu-baseline --parity-images 1 > $D/bench_flat.log 2>&1; echo "flat bench rc $?"; grep '^{' $D/bench_flat.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'bpsp', d['bpsp'])"
timeout 900 python bench.py --steps 3 --no-cpu-baseline > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'chain', d.get('chain',{}).get('frac'), 'parity', d.get('parity',{}).get('byte_identical'))"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_decode2 -c 1 -o $D/dec_c2 python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 0 > $D/ncu_dec.log 2>&1; echo "ncu dec rc $?"
