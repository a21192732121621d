# One full ncu capture of the single-GPU trailing-update kernel (launch 20 of a factorization):
#   WL=c3|c2 OUT=name bash tools/gpu/ncu_schur.sh      (run under gpurun; report -> gpurun_out/$OUT.ncu-rep)
# Read it here with: ncu -i gpurun_out/$OUT.ncu-rep --page raw --csv / --page source --csv --print-source sass
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
WL=${WL:-c3}
timeout 300 python tools/schur_ab.py $WL 0 > gpurun_out/ncu_schur_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:schur_ws2 -s 20 -c 1 -f \
  -o gpurun_out/${OUT:-ncu_schur_$WL} python tools/schur_ab.py $WL 0 > gpurun_out/ncu_schur.log 2>&1
echo "ncu exit $?"
