cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export RCP_SCHUR_HINTS=${HINTS:-0}
timeout 300 python tools/schur_ab.py c3 0 > gpurun_out/g17_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:schur_ws2 -s 20 -c 1 -f -o gpurun_out/${OUT:-g17_ws2_c3} python tools/schur_ab.py c3 0 > gpurun_out/g17_ncu.log 2>&1
echo "ncu exit $?"; tail -2 gpurun_out/g17_ncu.log
