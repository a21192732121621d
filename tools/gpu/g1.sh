cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/g1_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -s > gpurun_out/g1_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/g1_tests.log
tail -n 5 gpurun_out/g1_tests.log
grep "C2:\|C4:\|C3:" gpurun_out/g1_tests.log
timeout 300 python tools/solve_timing.py --n 32768 > gpurun_out/g1_solve.log 2>&1
timeout 300 python tools/solve_timing.py --n 32768 --nrhs 4 >> gpurun_out/g1_solve.log 2>&1
timeout 300 python tools/solve_timing.py --n 8191 --b 64 --p 74 --nrhs 3 >> gpurun_out/g1_solve.log 2>&1
cat gpurun_out/g1_solve.log | tail -5
cat gpurun_out/g1_smi.txt
