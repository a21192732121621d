# SM-partition model for lookahead: the panel kernel on a reserved partition of S SMs
# (RCP_PANEL_SMS=S) and the trailing update on the remaining 148 - S (RCP_SCHUR_SMS), each measured alone over a
# whole C3 factorization (device stamps).  With perfect overlap a panel step costs max(panel(S), schur(148 - S)).
cd $GRAFT_REPO_ROOT
echo "baseline"; timeout 300 python tools/schur_ab.py c3 1 2>&1 | tail -1
for s in 16 32 74 111; do
  echo "panel on $s SMs"; RCP_PANEL_SMS=$s timeout 600 python tools/schur_ab.py c3 1 2>&1 | tail -1
  echo "schur on $((148 - s)) SMs"; RCP_SCHUR_SMS=$((148 - s)) timeout 600 python tools/schur_ab.py c3 1 2>&1 | tail -1
done
