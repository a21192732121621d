# launch list of the bench command (device times, cold-cache + serialised: compare SHARES) and
# one full capture each of the dominant kernels at C3.
set -x
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 5406 -c 1802 --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:schur_update -s 40 -c 1 -o gpurun_out/prof_schur_c3 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_s.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 40 -c 1 -o gpurun_out/prof_panel_c3 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_p.log 2>&1
ls -la gpurun_out | tail
