cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 > gpurun_out/g7_bench_c2.log 2>&1; echo "c2 exit $?"; tail -c 600 gpurun_out/g7_bench_c2.log
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/g7_bench_c4.log 2>&1; echo "c4 exit $?"; tail -c 600 gpurun_out/g7_bench_c4.log
RCP_B200_LIB=paper_1710_00125_b200/librcp_prof.so timeout 300 python tools/profile_factor.py --n 8192 --b 64 --p 74 --reps 2 > gpurun_out/g7_prof_c2.log 2>&1
RCP_B200_LIB=paper_1710_00125_b200/librcp_prof.so timeout 300 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/g7_prof_c3.log 2>&1
tail -1 gpurun_out/g7_prof_c2.log; tail -1 gpurun_out/g7_prof_c3.log
python tools/profile_factor.py --n 8192 --b 64 --p 74 --reps 1 > gpurun_out/g7_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"schur_ws|dmma_gemm" -s 20 -c 2 -o gpurun_out/g7_c2 python tools/profile_factor.py --n 8192 --b 64 --p 74 --reps 1 > gpurun_out/g7_ncu.log 2>&1
echo "ncu exit $?"
