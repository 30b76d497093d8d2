cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 120 ./scripts/ubench_chain > gpurun_out/ubench_chain.log 2>&1; echo "ubench rc $?"; tail -5 gpurun_out/ubench_chain.log
python scripts/enc_c2.py 4 && ncu --set full --import-source on --clock-control none -k regex:k_enc_tables -c 1 -o gpurun_out/enctab_$1 python scripts/enc_c2.py 4 > gpurun_out/ncu_enctab.log 2>&1; echo "ncu rc $?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench rc $?"; tail -n 1 gpurun_out/bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'e2e', d['e2e']['value'], 'enc', d['encode'], 'net', d['encode_network']['ms'])"
