cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_diagnostics.py tests/test_dist_gpu.py -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/schur_ab.py c3 2 2>&1 | tail -1
timeout 300 python tools/schur_ab.py c2 3 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_full_size.py -x -q -m gpu 2>&1 | tail -3
