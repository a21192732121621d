# One iteration on the GPU box: parity tests, C3 timing (normal build) and the per-phase
# panel profile (RCP_PANEL_PROF build).  Usage: bash tools/gpu_iter.sh [tag]
tag=${1:-it}
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/${tag}_tests.log
tail -n 2 gpurun_out/${tag}_tests.log
timeout 300 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 2 > gpurun_out/${tag}_c3.log 2>&1
cat gpurun_out/${tag}_c3.log | cut -c1-200
if [ -f paper_1710_00125_b200/librcp_prof.so ]; then
  RCP_B200_LIB=paper_1710_00125_b200/librcp_prof.so timeout 300 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/${tag}_prof.log 2>&1
  cat gpurun_out/${tag}_prof.log
fi
for v in ${VARIANTS}; do
  echo "== variant $v"
  RCP_B200_LIB=paper_1710_00125_b200/librcp_$v.so timeout 300 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 2 | cut -c1-120
done
