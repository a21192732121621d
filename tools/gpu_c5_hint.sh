timeout 600 python -m pytest tests/test_batched.py -x -q > gpurun_out/hint_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/hint_tests.log; tail -2 gpurun_out/hint_tests.log
timeout 600 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/hint_bench_c5.json 2> gpurun_out/hint_bench_c5.err; echo "bench exit $?"
python -c "import json;d=json.load(open('gpurun_out/hint_bench_c5.json'));print(d['value'], d['ms_per_step'], d['e2e']['value'])"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:batched_factor_kernel -s 3 -c 1 python bench.py --workload c5 --count 16384 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/hint_ncu.log 2>&1
grep -E "dram__bytes|gpu__time" gpurun_out/hint_ncu.log
