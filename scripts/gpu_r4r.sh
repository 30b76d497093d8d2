# Overlapped encode A/B (LPIC_ENC_OVERLAP=1: half 1's network on a side stream beside half 0's tables)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4r; mkdir -p $D
for rep in 1 2; do
  timeout 300 python scripts/enc_time.py kaiming 3 2>&1 | tail -1
  LPIC_ENC_OVERLAP=1 timeout 300 python scripts/enc_time.py kaiming 3 2>&1 | tail -1 | sed 's/^/overlap /'
done | tee $D/enc_overlap_ab.txt
LPIC_ENC_OVERLAP=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -x > $D/pytest_parity_overlap.log 2>&1; echo "tests (overlap) rc $?"; tail -2 $D/pytest_parity_overlap.log
LPIC_ENC_OVERLAP=1 timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 1 > $D/bench_overlap.log 2>&1; echo "bench rc $?"; grep '^{' $D/bench_overlap.log | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec', d['value'], 'enc', d['encode']['value'], d['encode']['e2e'], 'parity', d.get('parity'))"
