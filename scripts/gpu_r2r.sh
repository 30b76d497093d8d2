# iteration r: payload bytes prefetched one advance ahead; in-situ profile + bench + selected tests
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2r; mkdir -p $D
timeout 180 ./scripts/ubench_chain > $D/ubench_chain.log 2>&1; echo "chain rc $?"; grep -E "cycles per table|TOTAL" $D/ubench_chain.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $D/pytest_parity.log 2>&1; echo "tests rc $?"; tail -2 $D/pytest_parity.log
LPIC_LIB=paper_2212_01185_b200/ab/prof.so timeout 600 python scripts/dec_timeline.py 512 768 24 > $D/timeline_prof_c2.log 2>&1; echo "rc $?"; head -5 $D/timeline_prof_c2.log; grep -A15 "in-situ" $D/timeline_prof_c2.log
timeout 900 python bench.py --steps 3 --no-cpu-baseline --parity-images 1 > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'chain', d.get('chain',{}).get('frac'), 'parity', d.get('parity',{}).get('byte_identical'))"
