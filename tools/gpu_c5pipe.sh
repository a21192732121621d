tag=${1:-c5p}
timeout 600 python -m pytest tests/test_batched.py -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/${tag}_tests.log
tail -n 15 gpurun_out/${tag}_tests.log
for ch in 148 296 592; do
timeout 600 python bench.py --workload c5 --no-cpu-baseline --e2e-chunk $ch > gpurun_out/${tag}_bench_c5_$ch.json 2> gpurun_out/${tag}_bench_c5_$ch.err; echo "bench c5 $ch exit $?"
python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_c5_$ch.json'));print($ch, d['value'], d['e2e'])"
done
