cd $GRAFT_REPO_ROOT
for lib in librcp_b200.so librcp_u4.so; do
  echo "== $lib"
  RCP_B200_LIB=paper_1710_00125_b200/$lib timeout 300 python tools/solve_timing.py --n 32768 2>&1 | grep solve
  RCP_B200_LIB=paper_1710_00125_b200/$lib timeout 300 python tools/solve_timing.py --n 32768 --nrhs 3 2>&1 | grep solve
  RCP_B200_LIB=paper_1710_00125_b200/$lib timeout 300 python tools/solve_timing.py --n 8191 --b 64 --p 74 --nrhs 2 2>&1 | grep solve
done
