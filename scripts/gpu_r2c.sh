# Round 2 iteration c: chain phase profile, the reference's own test suite
# against this build, the FULL scale-parity set (>= 10 M tables), GPU tests.
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2c; mkdir -p $D
timeout 180 ./scripts/ubench_chain_prof > $D/ubench_chain_prof.log 2>&1; echo "prof rc $?"; grep -E "cycles" $D/ubench_chain_prof.log | head -40
LPIC_PARITY_OUT=$D/parity timeout 2400 python -m pytest tests -m gpu -q -x -rA > $D/pytest_gpu.log 2>&1; echo "pytest rc $?"; grep -E "passed|failed" $D/pytest_gpu.log | tail -3; tail -30 $D/parity/reference_suite.txt
LPIC_PARITY_FULL=1 LPIC_PARITY_OUT=$D/parity_full timeout 3000 python -m pytest tests/test_gpu_scale_parity.py -q -x -rA > $D/pytest_parity_full.log 2>&1; echo "full parity rc $?"; grep -E "^containers|^table|passed|failed" $D/pytest_parity_full.log | cut -c 1-300
