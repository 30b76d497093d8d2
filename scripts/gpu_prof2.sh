cd $GRAFT_REPO_ROOT
timeout 300 python scripts/prof_small.py 256 8 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_small.csv python scripts/prof_small.py 256 8 > gpurun_out/ncu_launch.log 2>&1
echo "launch rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_encode -c 1 -o gpurun_out/prof_encode2 python scripts/prof_small.py 256 8 > gpurun_out/ncu_enc.log 2>&1
echo "enc rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode2 -c 1 -o gpurun_out/prof_decode2 python scripts/prof_small.py 128 1 > gpurun_out/ncu_dec.log 2>&1
echo "dec rc $?"
