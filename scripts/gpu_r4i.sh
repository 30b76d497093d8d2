# Session 3 verification at the table-occupancy commit: full GPU suite, default
# and FAST bench, reference arm, table A/B (4 blocks/SM), smoke + bench launch lists
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4i; mkdir -p $D
timeout 2400 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $D/pytest_gpu.log
timeout 900 python bench.py > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'e2e', d['e2e']['value'], 'enc', d['encode']['value'], 'tc', d.get('encode_network_tcgen05',{}).get('model_tflops'), 'parity', d.get('parity',{}).get('byte_identical'), 'clk', d['clocks'])"
timeout 900 python bench.py --precision fast --steps 3 --warmup 3 --no-cpu-baseline --parity-images 0 > $D/bench_fast.log 2>&1; echo "bench fast rc $?"; grep '^{' $D/bench_fast.log | tail -1 | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.log 2>&1; echo "ref rc $?"; grep '^{' $D/bench_ref.log | tail -1 | cut -c1-300
for v in main qc2m4 qc1m4 main qc2m4 qc1m4; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/enc_time.py kaiming 3 2>&1 | tail -1
done | tee $D/enc_ab.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $D/ncu_smoke.log 2>&1; echo "ncu smoke rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $D/launches_bench_c2.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 0 > $D/ncu_launches.log 2>&1; echo "launches rc $?"
