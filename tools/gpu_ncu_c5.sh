# C5 launch list of the bench command and one full capture of the batched kernel (16384 matrices:
# ncu saves/restores the kernel's outputs between replay passes, so the full-size 34 GB L is avoided).
CMD="python bench.py --workload c5 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/c5n_plain.json 2> gpurun_out/c5n_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv $CMD > gpurun_out/c5n_launch.log 2>&1
echo "launch list exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:batched_factor_kernel -s 3 -c 1 -o gpurun_out/prof_batched_c5 python bench.py --workload c5 --count 16384 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/c5n_full.log 2>&1
echo "full exit $?"
tail -3 gpurun_out/c5n_full.log
