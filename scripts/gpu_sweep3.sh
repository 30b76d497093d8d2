# Round-1 final sweep: tests, default bench (+ CPU baseline), every config,
# FAST precision, grayscale, reference arm, launch list and ncu captures.
cd $GRAFT_REPO_ROOT
D=gpurun_out/sweep3; mkdir -p $D
python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; tail -1 $D/pytest_gpu.log
timeout 900 python bench.py > $D/bench_default.log 2>&1; echo "default rc $?"
for c in c1 c3 c4 c5-1 c5-8 c5-64 c5-512 c5-4096; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $D/compat_$c.log 2>&1; echo "$c rc $?"
done
for c in c2 c4 c5-512; do
  timeout 900 python bench.py --config $c --precision fast --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $D/fast_$c.log 2>&1; echo "fast $c rc $?"
done
timeout 600 python bench.py --config c5-64 --gray --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $D/compat_c5-64_gray.log 2>&1; echo "gray rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $D/reference_c2.log 2>&1; echo "ref rc $?"
# ncu serialises kernels: the encoder's chasing plan is switched off (LPIC_NO_CHASE=1)
LPIC_NO_CHASE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_bench_c2.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $D/ncu_launches.log 2>&1; echo "launches rc $?"
LPIC_NO_CHASE=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_decode2 -c 1 -o $D/dec_c5-64 python bench.py --config c5-64 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $D/ncu_dec.log 2>&1; echo "ncu dec rc $?"
LPIC_NO_CHASE=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_tables -c 1 -o $D/enctab_c2 python scripts/enc_c2.py 4 > $D/ncu_enctab.log 2>&1; echo "ncu enctab rc $?"
LPIC_NO_CHASE=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_net -c 1 -o $D/encnet_c2 python scripts/enc_c2.py 4 > $D/ncu_encnet.log 2>&1; echo "ncu encnet rc $?"
