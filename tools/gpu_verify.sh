# Round-end style verification: parity tests, smoke, the default bench line (C3) and the C5 line.
tag=${1:-v12}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/${tag}_tests.log
tail -n 3 gpurun_out/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${tag}_smoke.log 2>&1; tail -n 2 gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench_c3.json 2> gpurun_out/${tag}_bench_c3.err; echo "bench exit $?"
cut -c1-400 gpurun_out/${tag}_bench_c3.json
timeout 600 python bench.py --workload c5 > gpurun_out/${tag}_bench_c5.json 2> gpurun_out/${tag}_bench_c5.err; echo "bench c5 exit $?"
cut -c1-300 gpurun_out/${tag}_bench_c5.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err; echo "bench ref exit $?"
cut -c1-300 gpurun_out/${tag}_bench_ref.json
