# Session 3 baseline at HEAD: full GPU suite, default bench, reference arm,
# smoke under ncu (launch list), bench launch list.
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4a; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $D/pytest_gpu.log
timeout 900 python bench.py > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | tail -1 | cut -c1-600
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.log 2>&1; echo "ref rc $?"; grep '^{' $D/bench_ref.log | tail -1 | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $D/ncu_smoke.log 2>&1; echo "ncu smoke rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $D/launches_bench_c2.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 0 > $D/ncu_launches.log 2>&1; echo "launches rc $?"
