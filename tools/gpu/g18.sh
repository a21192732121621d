cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
echo "V=1"; RCP_SCHUR_V=1 timeout 300 python tools/schur_ab.py c3 2 2>&1 | tail -1
echo "V=2 hints"; timeout 300 python tools/schur_ab.py c3 2 2>&1 | tail -1
echo "V=2 nohints"; RCP_SCHUR_HINTS=0 timeout 300 python tools/schur_ab.py c3 2 2>&1 | tail -1
echo "c2: V=1, V=2 hints, V=2 nohints"
RCP_SCHUR_V=1 timeout 300 python tools/schur_ab.py c2 3 2>&1 | tail -1
timeout 300 python tools/schur_ab.py c2 3 2>&1 | tail -1
RCP_SCHUR_HINTS=0 timeout 300 python tools/schur_ab.py c2 3 2>&1 | tail -1
