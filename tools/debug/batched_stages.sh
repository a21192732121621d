#!/bin/bash
# run the small batched case stopping after each debug stage
for s in 1 2 3 4 5 6 0; do
  echo "== stage $s"
  RCP_BATCH_DBG=$s timeout 60 python tools/debug/batched_small.py 64 2 2>&1 | tail -2
done
