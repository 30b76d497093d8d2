cd $GRAFT_REPO_ROOT
timeout 120 ./scripts/ubench_chain > gpurun_out/ubench_chain.log 2>&1; echo "ubench rc $?"; cat gpurun_out/ubench_chain.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python scripts/dec_timeline.py 512 768 > gpurun_out/tl_c2.log 2>&1; echo "tl rc $?"; head -4 gpurun_out/tl_c2.log
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc $?"; tail -c 1500 gpurun_out/bench.log
