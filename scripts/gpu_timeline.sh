cd $GRAFT_REPO_ROOT
timeout 300 python scripts/dec_timeline.py 128 128 > gpurun_out/tl_128.log 2>&1; echo "rc $?"
timeout 300 python scripts/dec_timeline.py 512 768 > gpurun_out/tl_c2.log 2>&1; echo "rc $?"
cat gpurun_out/tl_128.log gpurun_out/tl_c2.log
