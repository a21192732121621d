cd $GRAFT_REPO_ROOT
timeout 300 python tools/solve_timing.py --n 32768 2>&1 | grep solve
timeout 300 python tools/solve_timing.py --n 32768 --nrhs 3 2>&1 | grep solve
python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/g12_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:schur_ws -s 20 -c 1 -o gpurun_out/g12_c3 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/g12_ncu.log 2>&1
echo "ncu exit $?"
