cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export RCP_SCHUR_HINTS=0
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
echo "V=2 prefetch + setmaxnreg 208/88"; timeout 300 python tools/schur_ab.py c3 2 2>&1 | tail -1
echo "V=2 prefetch, no setmaxnreg"; RCP_B200_LIB=$PWD/paper_1710_00125_b200/librcp_nosmr.so timeout 300 python tools/schur_ab.py c3 2 2>&1 | tail -1
echo "c2"
timeout 300 python tools/schur_ab.py c2 3 2>&1 | tail -1
timeout 300 python tools/schur_ab.py c3 0 > gpurun_out/g17_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:schur_ws2 -s 20 -c 1 -f -o gpurun_out/g21_ws2 python tools/schur_ab.py c3 0 > gpurun_out/g17_ncu.log 2>&1
echo "ncu exit $?"
