cd $GRAFT_REPO_ROOT
for m in 2 1; do echo "MINB=$m"; RCP_BATCH_MINB=$m timeout 300 python tools/c5_timing.py 16384 2>&1 | tail -1; done
