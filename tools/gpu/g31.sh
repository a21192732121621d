cd $GRAFT_REPO_ROOT
for w in c1 c2 c4 c3; do timeout 300 python tools/schur_ab.py $w 3 2>&1 | tail -1; done
