# Round 2 iteration b: peaks (Phi throughput, isolated chain), GPU suite with
# the scale-parity tests, default bench line (new keys), C3 strong on 1 GPU,
# C4 / C5-4096 / C5-64.
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2b; mkdir -p $D
timeout 120 ./scripts/ubench_phi_peak > $D/ubench_phi_peak.json 2>&1; echo "phi rc $?"; cat $D/ubench_phi_peak.json
timeout 180 ./scripts/ubench_chain > $D/ubench_chain.log 2>&1; echo "chain rc $?"; grep -E "cycles per table|TOTAL" $D/ubench_chain.log
LPIC_PARITY_OUT=$D/parity timeout 2400 python -m pytest tests -m gpu -q -x -rA > $D/pytest_gpu.log 2>&1; echo "pytest rc $?"; grep -E "passed|failed|^containers|^table" $D/pytest_gpu.log | tail -12
timeout 900 python bench.py > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | tail -1
for c in c4 c5-4096 c5-64; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 2 > $D/compat_$c.log 2>&1; echo "$c rc $?"; grep '^{' $D/compat_$c.log | cut -c 1-300
done
timeout 1500 python bench.py --config c3 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 1 > $D/compat_c3.log 2>&1; echo "c3 rc $?"; grep '^{' $D/compat_c3.log | cut -c 1-400
