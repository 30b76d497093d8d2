# iteration p: red search by multiply-compare, digit-255 REDUX reverted; in-situ timeline at C2.
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2p; mkdir -p $D
timeout 180 ./scripts/ubench_chain > $D/ubench_chain.log 2>&1; echo "chain rc $?"; grep -E "cycles per table|TOTAL" $D/ubench_chain.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "container or golden or decode or flat or selection" > $D/pytest_sel.log 2>&1; echo "tests rc $?"; tail -2 $D/pytest_sel.log
timeout 600 python scripts/dec_timeline.py 512 768 24 > $D/timeline_c2.log 2>&1; echo "timeline rc $?"; head -5 $D/timeline_c2.log
timeout 900 python bench.py --steps 3 --no-cpu-baseline --parity-images 1 > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'chain', d.get('chain',{}).get('frac'), 'parity', d.get('parity',{}).get('byte_identical'))"
