# in-situ chain phase profile at C2 (A/B build with -DLPIC_DEC_PROF)
cd $GRAFT_REPO_ROOT
D=gpurun_out/r2q; mkdir -p $D
LPIC_LIB=paper_2212_01185_b200/ab/prof.so timeout 600 python scripts/dec_timeline.py 512 768 24 > $D/timeline_prof_c2.log 2>&1; echo "rc $?"; head -5 $D/timeline_prof_c2.log; grep -A15 "in-situ" $D/timeline_prof_c2.log
