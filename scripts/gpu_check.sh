cd $GRAFT_REPO_ROOT
nvidia-smi -L
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --sample-px 4096 > gpurun_out/bench.log 2>&1; echo "bench rc $?"
tail -5 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log
