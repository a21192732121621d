cd $GRAFT_REPO_ROOT
free -g > gpurun_out/g2_host.txt; nproc >> gpurun_out/g2_host.txt; grep "model name" /proc/cpuinfo | head -1 >> gpurun_out/g2_host.txt
timeout 900 python -m pytest tests -m gpu -x -q -s > gpurun_out/g2_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/g2_tests.log
tail -n 5 gpurun_out/g2_tests.log
grep "C2:\|C4:\|C3:" gpurun_out/g2_tests.log
timeout 300 python tools/solve_timing.py --n 32768 > gpurun_out/g2_solve.log 2>&1
timeout 300 python tools/solve_timing.py --n 32768 --nrhs 3 >> gpurun_out/g2_solve.log 2>&1
timeout 300 python tools/solve_timing.py --n 8191 --b 64 --p 74 --nrhs 2 >> gpurun_out/g2_solve.log 2>&1
cat gpurun_out/g2_solve.log | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/g2_bench.log 2>&1; echo "bench exit $?"
tail -c 3000 gpurun_out/g2_bench.log
cat gpurun_out/g2_host.txt
