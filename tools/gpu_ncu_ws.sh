timeout 300 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:schur_ws -s 40 -c 1 -o gpurun_out/prof_ws_c3 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_ws.log 2>&1
tail -2 gpurun_out/ncu_ws.log
