cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# compute-sanitizer passes over small parity cases (memcheck: global/shared OOB and misaligned; racecheck: shared-memory hazards; synccheck)
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --target-processes all --error-exitcode 7 \
    python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "test_factor_matches_oracle_live or test_q1_mode_matches_oracle_live or test_solve_many" \
    > gpurun_out/sanitizer_$tool.log 2>&1
  echo "exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitizer_$tool.log | tail -4
done
