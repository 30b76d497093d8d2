# Session 3 final verification at HEAD: full GPU suite, smoke, default / FAST /
# reference bench lines, C3 strong, launch lists, ncu of the FAST network,
# then the full-scale parity run (all C2 images, C3/C4/C5-64, fitted, >= 10 M tables)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4n; mkdir -p $D; R=/tmp/r4n_reps; mkdir -p $R
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $D/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 $D/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc $?"; tail -1 $D/smoke.log
timeout 900 python bench.py > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'e2e', d['e2e']['value'], 'enc', d['encode']['value'], 'tc', d.get('encode_network_tcgen05',{}).get('model_tflops'), 'parity', d.get('parity',{}).get('byte_identical'), 'clk', d['clocks'])"
timeout 900 python bench.py --precision fast > $D/bench_fast.log 2>&1; echo "bench fast rc $?"; grep '^{' $D/bench_fast.log | tail -1 | cut -c1-200
timeout 900 python bench.py --impl reference > $D/bench_ref.log 2>&1; echo "ref rc $?"; grep '^{' $D/bench_ref.log | tail -1 | cut -c1-200
timeout 1200 python bench.py --config c3 --steps 3 --warmup 3 --e2e-steps 1 --parity-images 0 --no-cpu-baseline > $D/bench_c3.log 2>&1; echo "c3 rc $?"; grep '^{' $D/bench_c3.log | tail -1 | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $D/ncu_smoke.log 2>&1; echo "ncu smoke rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $D/launches_bench_c2.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 0 > $D/ncu_launches.log 2>&1; echo "launches rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_net_tc2 -c 1 -o $R/tc2_c2 python scripts/enc_fast.py 24 > $D/ncu_tc2_c2.log 2>&1; echo "ncu tc2 rc $?"
ncu -i $R/tc2_c2.ncu-rep --page raw --csv > $D/tc2_c2_raw.csv 2>/dev/null; python scripts/ncu_lines.py $R/tc2_c2.ncu-rep regex:k_enc_net_tc2 45 > $D/tc2_c2_lines.txt 2>&1
LPIC_PARITY_FULL=1 LPIC_PARITY_OUT=$D/parity_full timeout 3000 python -m pytest tests/test_gpu_scale_parity.py -q -x -rA > $D/pytest_parity_full.log 2>&1; echo "full parity rc $?"; tail -2 $D/pytest_parity_full.log
