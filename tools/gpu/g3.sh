cd $GRAFT_REPO_ROOT
timeout 300 python tools/schur_ab.py --n 2500 --b 64 --p 74 --reps 1 > gpurun_out/g3_ab_small.log 2>&1; echo "ab small exit $?"
tail -3 gpurun_out/g3_ab_small.log
timeout 600 python tools/schur_ab.py --n 32768 --b 128 --p 144 --reps 2 > gpurun_out/g3_ab_c3.log 2>&1; echo "ab c3 exit $?"
tail -3 gpurun_out/g3_ab_c3.log
timeout 1200 python -m pytest tests -m gpu -x -q -s > gpurun_out/g3_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/g3_tests.log
tail -n 5 gpurun_out/g3_tests.log
grep "C2:\|C4:\|C3:" gpurun_out/g3_tests.log
