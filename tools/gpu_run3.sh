set -x
timeout 300 python tools/profile_factor.py --n 8192 --b 64 --p 74 --reps 2
timeout 300 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 2
timeout 300 python tools/profile_factor.py --n 8192 --b 64 --p 74 --reps 1 > /dev/null && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dmma_gemm_kernel -s 20 -c 2 -o gpurun_out/prof_gemm python tools/profile_factor.py --n 8192 --b 64 --p 74 --reps 1 > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 10 -c 1 -o gpurun_out/prof_panel python tools/profile_factor.py --n 8192 --b 64 --p 74 --reps 1 > gpurun_out/ncu_panel.log 2>&1
ls -la gpurun_out
