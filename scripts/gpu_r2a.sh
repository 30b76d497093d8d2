# Round 2, first iteration: fused cooperative range-coder plan, FAST tags,
# decoder acquire fences.  GPU suite, smoke, default bench, then the smoke
# under ncu (launch list) and compute-sanitizer (memcheck / racecheck /
# synccheck) -- the serialised-launch cases that broke the round-1 chase.
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2a; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; tail -3 $D/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py --steps 3 --warmup 3 > $D/bench_default.log 2>&1; echo "bench rc $?"; tail -c 3000 $D/bench_default.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/smoke_launches.csv \
   python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke_ncu.log 2>&1; echo "ncu smoke rc $?"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" \
     > $D/sanitizer_$tool.log 2>&1; echo "sanitizer $tool rc $?"; tail -3 $D/sanitizer_$tool.log
done
