cd $GRAFT_REPO_ROOT
timeout 900 python tools/schur_ab.py --n 32768 --b 128 --p 144 --reps 2 --variants ws,lower_ws,lower_pp > gpurun_out/g6_ab_c3.log 2>&1; echo "ab c3 exit $?"
tail -4 gpurun_out/g6_ab_c3.log
