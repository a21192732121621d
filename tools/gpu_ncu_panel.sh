# Full ncu capture (with source) of one panel_kernel launch at C3 (panel 20, m ~ 30k).
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 20 -c 1 -o gpurun_out/ncu_panel python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_panel.log 2>&1
ls -la gpurun_out/*.ncu-rep
