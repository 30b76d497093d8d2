cd $GRAFT_REPO_ROOT
D=gpurun_out/r3g; mkdir -p $D
LPIC_LIB=paper_2212_01185_b200/ab/nomma.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_net_tc2 -c 1 -o $D/nomma python scripts/enc_fast.py 8 > $D/ncu.log 2>&1; echo "ncu rc $?"
