cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/schur_ab.py c3 1 2>&1 | tail -1
timeout 300 python tools/schur_ab.py c3 0 > gpurun_out/g17_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:schur_ws2 -s 20 -c 1 -f -o gpurun_out/g27_ws2 python tools/schur_ab.py c3 0 > gpurun_out/g17_ncu.log 2>&1
echo "ncu exit $?"
