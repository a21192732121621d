cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 20 -c 1 -f -o gpurun_out/g29_panel python tools/schur_ab.py c3 0 > gpurun_out/ncu_panel.log 2>&1
echo "ncu panel exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batched_factor -s 1 -c 1 -f -o gpurun_out/g29_c5 python tools/c5_timing.py 4096 > gpurun_out/ncu_c5.log 2>&1
echo "ncu c5 exit $?"
