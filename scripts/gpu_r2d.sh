# Round 2 iteration d: transposed-Phi table builder + packed compat network.
# GPU suite (bitwise network/table checks), default bench, launch list,
# ncu --set full of the encoder kernels (4 C2 images) and the decoder (C2).
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2d; mkdir -p $D
timeout 2400 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $D/pytest_gpu.log
timeout 900 python bench.py --steps 3 > $D/bench_default.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_default.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], 'net ms', d['encode_network']['ms'], 'parity', d.get('parity',{}).get('byte_identical'))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $D/launches_bench_c2.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 0 > $D/ncu_launches.log 2>&1; echo "launches rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_tables -c 1 -o $D/enctab_c2 python scripts/enc_c2.py 4 > $D/ncu_enctab.log 2>&1; echo "ncu enctab rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_net -c 1 -o $D/encnet_c2 python scripts/enc_c2.py 4 > $D/ncu_encnet.log 2>&1; echo "ncu encnet rc $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_decode2 -c 1 -o $D/dec_c2 python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 0 > $D/ncu_dec.log 2>&1; echo "ncu dec rc $?"
