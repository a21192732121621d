set -x
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python bench.py --n 8192 --b 64 --p 74 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1
