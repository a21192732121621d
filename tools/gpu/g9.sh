cd $GRAFT_REPO_ROOT
timeout 300 python tools/solve_timing.py --n 32768 > gpurun_out/g9_solve.log 2>&1
timeout 300 python tools/solve_timing.py --n 32768 --nrhs 3 >> gpurun_out/g9_solve.log 2>&1
timeout 300 python tools/solve_timing.py --n 8191 --b 64 --p 74 --nrhs 2 >> gpurun_out/g9_solve.log 2>&1
timeout 300 python tools/solve_timing.py --n 1000 --b 32 --p 42 --nrhs 1 >> gpurun_out/g9_solve.log 2>&1
cat gpurun_out/g9_solve.log | grep solve
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/g9_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/g9_tests.log
tail -n 4 gpurun_out/g9_tests.log
