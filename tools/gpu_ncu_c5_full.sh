timeout 1200 ncu --set full --clock-control none --import-source on -k regex:batched_factor_kernel -s 3 -c 1 -o gpurun_out/prof_batched_c5_v11 python bench.py --workload c5 --count 16384 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/c5full11.log 2>&1
echo "full exit $?"
