# round-2 closing measurements: full GPU test suite, bench lines (C3 default, C2, C4, C5), launch list of the
# C3 bench command.  Outputs under gpurun_out/ (copied into profiles/ by hand).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02_gpu_tests_final.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r02_gpu_tests_final.log
timeout 1200 python bench.py --steps 20 --warmup 3 > gpurun_out/r02_bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench c3 exit $?"
timeout 600 python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 exit $?"
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 exit $?"
timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 exit $?"
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 5406 -c 1802 --csv --log-file gpurun_out/r02_launches_c3.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?"
