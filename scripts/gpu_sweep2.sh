cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sweep2
python -m pytest tests -m gpu -q > gpurun_out/sweep2/pytest_gpu.log 2>&1; tail -1 gpurun_out/sweep2/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/sweep2/bench_default.log 2>&1; echo "default rc $?"
for c in c1 c2 c3 c4 c5-1 c5-8 c5-64 c5-512 c5-4096; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep2/compat_$c.log 2>&1; echo "$c rc $?"
done
for c in c2 c4 c5-512; do
  timeout 900 python bench.py --config $c --precision fast --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep2/fast_$c.log 2>&1; echo "fast $c rc $?"
done
timeout 600 python bench.py --config c5-64 --gray --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep2/compat_c5-64_gray.log 2>&1; echo "gray rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/sweep2/reference_c2.log 2>&1; echo "ref rc $?"
