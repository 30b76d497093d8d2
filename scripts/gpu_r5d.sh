# session-5: full GPU suite at HEAD with the reference's own tests present (baseline/_ref_tests)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r5d; mkdir -p $D
timeout 2400 python -m pytest tests -m gpu -q -rs > $D/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $D/pytest_gpu.log
