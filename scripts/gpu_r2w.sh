# ncu source captures of the compat encoder kernels (4 C2 images, unfused plan) at HEAD
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2w; mkdir -p $D
LPIC_RC_UNFUSED=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_tables -c 1 -o $D/enctab python scripts/enc_c2.py 4 > $D/ncu_enctab.log 2>&1; echo "ncu enctab rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_enc_net<" -c 1 -o $D/encnet python scripts/enc_c2.py 4 > $D/ncu_encnet.log 2>&1; echo "ncu encnet rc $?"
