cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
echo "group 16 (default)"; timeout 300 python tools/schur_ab.py c3 2 2>&1 | tail -1
for g in 1 8 32; do echo "group $g"; RCP_B200_LIB=$PWD/paper_1710_00125_b200/librcp_g$g.so timeout 300 python tools/schur_ab.py c3 2 2>&1 | tail -1; done
timeout 300 python tools/schur_ab.py c2 3 2>&1 | tail -1
timeout 300 python tools/schur_ab.py c4 2 2>&1 | tail -1
