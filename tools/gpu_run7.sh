timeout 300 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/plain7.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 20 -c 1 -o gpurun_out/prof_panel_c3 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_panel_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:SchurEpi -s 20 -c 1 -o gpurun_out/prof_schur_c3 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_schur_c3.log 2>&1
ls -la gpurun_out/*.ncu-rep
