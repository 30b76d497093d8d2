# ncu --set full captures at the current commit, exported on the box to CSV
# (raw metrics + per-source-line stall summary); the .ncu-rep files stay behind
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4f; mkdir -p $D; R=/tmp/r4f_reps; mkdir -p $R
cap() {  # tag kernel-regex timeout cmd...
  tag=$1; k=$2; to=$3; shift 3
  timeout $to ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $R/$tag "$@" > $D/ncu_$tag.log 2>&1; echo "ncu $tag rc $?"
  ncu -i $R/$tag.ncu-rep --page raw --csv > $D/${tag}_raw.csv 2>/dev/null
  python scripts/ncu_lines.py $R/$tag.ncu-rep regex:$k 45 > $D/${tag}_lines.txt 2>&1
}
cap tc2_c2 k_enc_net_tc2 900 python scripts/enc_fast.py 24
cap enctab_c2 k_enc_tables 900 python scripts/enc_c2.py 24
cap encnet_c2 'k_enc_net<' 900 python scripts/enc_c2.py 24
cap dec_c2 k_decode2 1500 python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 0
ls -la $R
