cd $GRAFT_REPO_ROOT
timeout 300 python tools/solve_timing.py --n 32768 > gpurun_out/g10_solve.log 2>&1
timeout 300 python tools/solve_timing.py --n 32768 --nrhs 3 >> gpurun_out/g10_solve.log 2>&1
timeout 300 python tools/solve_timing.py --n 8191 --b 64 --p 74 --nrhs 2 >> gpurun_out/g10_solve.log 2>&1
timeout 300 python tools/solve_timing.py --n 1000 --b 32 --p 42 --nrhs 1 >> gpurun_out/g10_solve.log 2>&1
cat gpurun_out/g10_solve.log | grep solve
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_api_edges_gpu.py tests/test_full_size.py::test_c2_full_size -x -q > gpurun_out/g10_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/g10_tests.log
