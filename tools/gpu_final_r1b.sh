# Round-1 final validation: GPU tests, smoke, C3 + C5 bench lines, launch list of one C3 factorization.
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/final_tests.log
python __graft_entry__.py smoke > gpurun_out/final_smoke.log 2>&1
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --workload c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
  python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_launch.log 2>&1
tail -n 2 gpurun_out/final_tests.log; cat gpurun_out/final_smoke.log
