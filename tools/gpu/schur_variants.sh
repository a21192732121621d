# A/B of the trailing-update kernels on one box (device time per factorization, checksums):
#   RCP_SCHUR_V=1 first-generation kernel; RCP_SCHUR_TMA=0 cp.async producer; RCP_SCHUR_HINTS=0|1|2 L2 policies;
#   RCP_B200_LIB=<variant .so built with python -m paper_1710_00125_b200.build --variant NAME -D...>
cd $GRAFT_REPO_ROOT
for env in "" "RCP_SCHUR_TMA=0" "RCP_SCHUR_V=1" "RCP_SCHUR_HINTS=0" "RCP_SCHUR_HINTS=2"; do
  echo "== ${env:-default}"; env $env timeout 300 python tools/schur_ab.py ${WL:-c3} 2 2>&1 | tail -1
done
