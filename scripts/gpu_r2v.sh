# iteration v: aux poll interval A/B (256 main, 200, 64, 1000), with clocks
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2v; mkdir -p $D
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $D/smi.txt
for v in main s200 s64 sleep1k main s200 s64 sleep1k; do
  if [ $v = main ]; then LIB=""; else LIB="LPIC_LIB=paper_2212_01185_b200/ab/$v.so"; fi
  env $LIB timeout 300 python scripts/dec_time.py kaiming 3 2>&1 | tail -1
done | tee $D/dec_ab.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv >> $D/smi.txt; cat $D/smi.txt
