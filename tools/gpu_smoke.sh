set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 300 python __graft_entry__.py smoke
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
