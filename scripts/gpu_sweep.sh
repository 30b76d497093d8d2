cd $GRAFT_REPO_ROOT
# every BASELINE config on one B200 (C2 is the driver's default bench line)
for c in c1 c2 c5-1 c5-8 c5-64 c5-512 c4 c3 c5-4096; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep_$c.log 2>&1
  echo "$c rc $?"; grep '^{' gpurun_out/sweep_$c.log | head -c 400; echo
done
timeout 600 python bench.py --config c5-64 --gray --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep_c5-64_gray.log 2>&1
echo "gray rc $?"; grep '^{' gpurun_out/sweep_c5-64_gray.log | head -c 400; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref_c2.log 2>&1; echo "ref rc $?"; tail -c 600 gpurun_out/ref_c2.log
