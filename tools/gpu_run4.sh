timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/profile_factor.py --n 8192 --b 64 --p 74 --reps 2
timeout 300 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 2
