cd $GRAFT_REPO_ROOT
python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/g5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:schur_pp -s 20 -c 1 -o gpurun_out/g5_pp python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/g5_ncu.log 2>&1
echo "exit $?"; tail -3 gpurun_out/g5_ncu.log
