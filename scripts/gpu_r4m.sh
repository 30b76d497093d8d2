# FAST network: hi.hi and hi.lo in one N=2N MMA (A/B vs prev3): parity + timing
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4m; mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -x > $D/pytest_parity.log 2>&1; echo "tests rc $?"; tail -2 $D/pytest_parity.log
for i in 1 2; do timeout 300 python scripts/net_time.py 2>&1 | tail -1; done | tee $D/net_time.txt
for i in 1 2; do LPIC_LIB=paper_2212_01185_b200/ab/prev3.so timeout 300 python scripts/net_time.py 2>&1 | tail -1; done | tee -a $D/net_time.txt
