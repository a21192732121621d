cd $GRAFT_REPO_ROOT
t0=$(date +%s)
timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/g14_ref.log 2> gpurun_out/g14_ref.err; echo "ref exit $? wall $(( $(date +%s) - t0 )) s"
tail -c 1800 gpurun_out/g14_ref.log
t0=$(date +%s)
timeout 1700 python bench.py --impl reference --workload c5 --gpus 1 --steps 3 --warmup 1 > gpurun_out/g14_ref_c5.log 2>&1; echo "ref c5 exit $? wall $(( $(date +%s) - t0 )) s"
tail -c 800 gpurun_out/g14_ref_c5.log
