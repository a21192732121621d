cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
for t in 1 0; do echo "TMA=$t"; RCP_SCHUR_TMA=$t timeout 300 python tools/schur_ab.py c3 2 2>&1 | tail -1; done
for t in 1 0; do echo "c2 TMA=$t"; RCP_SCHUR_TMA=$t timeout 300 python tools/schur_ab.py c2 3 2>&1 | tail -1; done
timeout 300 python tools/schur_ab.py c3 0 > gpurun_out/g17_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:schur_ws2 -s 20 -c 1 -f -o gpurun_out/g24_ws2 python tools/schur_ab.py c3 0 > gpurun_out/g17_ncu.log 2>&1
echo "ncu exit $?"
