timeout 300 python tools/profile_factor.py --n 16384 --b 128 --p 144 --reps 1 > gpurun_out/plain_s.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:schur_update -s 10 -c 1 -o gpurun_out/prof_schur2 python tools/profile_factor.py --n 16384 --b 128 --p 144 --reps 1 > gpurun_out/ncu_schur2.log 2>&1
tail -3 gpurun_out/ncu_schur2.log
