cd $GRAFT_REPO_ROOT
timeout 600 python tools/schur_ab.py --n 32768 --b 128 --p 144 --reps 2 > gpurun_out/g4_ab_c3.log 2>&1; echo "ab c3 exit $?"
tail -3 gpurun_out/g4_ab_c3.log
