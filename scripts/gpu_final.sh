# Round-1 closing measurements at HEAD: GPU suite, smoke, default bench (with
# the CPU baseline), FAST C2, the many-stream configs, the reference arm.
cd $GRAFT_REPO_ROOT
D=gpurun_out/final; mkdir -p $D
python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; tail -1 $D/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > $D/bench_default.log 2>&1; echo "default rc $?"
timeout 900 python bench.py --precision fast --steps 3 --warmup 3 --no-cpu-baseline > $D/fast_c2.log 2>&1; echo "fast rc $?"
for c in c3 c4 c5-64 c5-512 c5-4096; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $D/compat_$c.log 2>&1; echo "$c rc $?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $D/reference_c2.log 2>&1; echo "ref rc $?"
