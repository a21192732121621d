# Full ncu captures (with source) of one panel_kernel and one schur_ws_kernel launch at C3 (m ~ 30k).
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 20 -c 1 -o gpurun_out/ncu_panel python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_panel.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:schur_ws -s 20 -c 1 -o gpurun_out/ncu_schur python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_schur.log 2>&1
ls -la gpurun_out/*.ncu-rep
