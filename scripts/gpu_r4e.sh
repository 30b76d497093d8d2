# ncu --set full captures at the current commit: FAST network (raster tiles),
# compat network, table kernel (24 C2 images), decoder (C2)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r4e; mkdir -p $D
timeout 600 python scripts/net_time.py > $D/net_time.log 2>&1; tail -1 $D/net_time.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_net_tc2 -c 1 -o $D/tc2_c2 python scripts/enc_fast.py 24 > $D/ncu_tc2.log 2>&1; echo "ncu tc2 rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_tables -c 1 -o $D/enctab_c2 python scripts/enc_c2.py 24 > $D/ncu_enctab.log 2>&1; echo "ncu enctab rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_net -c 1 -o $D/encnet_c2 python scripts/enc_c2.py 24 > $D/ncu_encnet.log 2>&1; echo "ncu encnet rc $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_decode2 -c 1 -o $D/dec_c2 python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --parity-images 0 > $D/ncu_dec.log 2>&1; echo "ncu dec rc $?"
