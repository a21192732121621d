cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for h in 0 1 2; do echo "hints=$h"; RCP_SCHUR_HINTS=$h timeout 300 python tools/schur_ab.py c3 2 2>&1 | tail -1; done
for h in 0 1; do echo "c2 hints=$h"; RCP_SCHUR_HINTS=$h timeout 300 python tools/schur_ab.py c2 3 2>&1 | tail -1; done
