cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/g13_smi.txt
/usr/bin/time -v timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/g13_ref.log 2> gpurun_out/g13_ref.err; echo "ref exit $?"
tail -c 1500 gpurun_out/g13_ref.log; grep "Elapsed\|Maximum resident" gpurun_out/g13_ref.err
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/g13_bench.log 2>&1; echo "bench exit $?"
tail -c 3500 gpurun_out/g13_bench.log
