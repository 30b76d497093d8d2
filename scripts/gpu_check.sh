cd $GRAFT_REPO_ROOT
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 300 python scripts/dec_timeline.py 512 768 > gpurun_out/tl_c2.log 2>&1; echo "tl rc $?"
timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --sample-px 4096 > gpurun_out/bench.log 2>&1; echo "bench rc $?"
tail -n 5 gpurun_out/pytest_gpu.log; head -4 gpurun_out/tl_c2.log; tail -c 2500 gpurun_out/bench.log
