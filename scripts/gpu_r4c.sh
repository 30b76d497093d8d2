# Many-stream decode diagnosis: compat vs FAST network in the producer, 1 vs 2 streams per cluster
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4c; mkdir -p $D
run() { tag=$1; shift; timeout 900 env "$@" > $D/$tag.log 2>&1; echo "$tag rc $?"; grep '^{' $D/$tag.log | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('  dec', round(d['value'],2), 'ms', round(d['ms_per_step'],1), 'enc', round(d['encode']['value'],1))"; }
B="python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline --parity-images 0"
run c5_compat_s2 $B --config c5-4096
run c5_fast_s2 $B --config c5-4096 --precision fast
run c5_compat_s1 LPIC_DEC_STREAMS_PER_CLUSTER=1 $B --config c5-4096
run c5_512_compat $B --config c5-512
run c5_512_fast $B --config c5-512 --precision fast
run c3_fast $B --config c3 --precision fast
