cd $GRAFT_REPO_ROOT
timeout 600 python tools/schur_ab.py --n 32768 --b 128 --p 144 --reps 2 --variants full > gpurun_out/g8_c3.log 2>&1; echo "c3 exit $?"; tail -2 gpurun_out/g8_c3.log
timeout 600 python tools/schur_ab.py --n 8192 --b 64 --p 74 --reps 3 --variants full > gpurun_out/g8_c2.log 2>&1; echo "c2 exit $?"; tail -2 gpurun_out/g8_c2.log
