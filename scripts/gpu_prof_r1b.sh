cd $GRAFT_REPO_ROOT
B="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $B > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $B > gpurun_out/ncu_bench.log 2>&1
echo "launch rc $?"
S="python scripts/prof_small.py 128 2"
timeout 300 $S > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_decode2|k_enc_net|k_enc_tables|k_rc_plan|k_rc_chunks" -c 5 -o gpurun_out/prof_r1b $S > gpurun_out/ncu_full.log 2>&1
echo "full rc $?"
