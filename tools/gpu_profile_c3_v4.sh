# Round-1 measurement pass: bench line (C3), launch list of one C3 factorization (device times,
# serialised: compare SHARES), full ncu captures of the panel and Schur kernels at panel 20.
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
tail -n 3 gpurun_out/bench_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
  python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:schur_ws -s 20 -c 1 -o gpurun_out/ncu_schur \
  python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_schur.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 20 -c 1 -o gpurun_out/ncu_panel \
  python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_panel.log 2>&1
ls -la gpurun_out/
