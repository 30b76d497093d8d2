cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python scripts/dec_timeline.py 256 256 512 > gpurun_out/tl_c5.log 2>&1; echo "tl5 rc $?"; head -6 gpurun_out/tl_c5.log
timeout 300 python scripts/dec_timeline.py 512 768 24 > gpurun_out/tl_c2_24.log 2>&1; echo "tl2 rc $?"; head -6 gpurun_out/tl_c2_24.log
for c in c2 c5-512; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc $?"; tail -n 1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('e2e'), d.get('extra', {}))"; done
