# Round-1 final measurement: C3 bench line, C5 bench line, launch list of one C3 factorization.
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --workload c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
  python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_launch.log 2>&1
tail -n 2 gpurun_out/bench_c3.err gpurun_out/bench_c5.err
