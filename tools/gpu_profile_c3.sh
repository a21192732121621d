#!/bin/bash
# C3 bench line + reference arm, then (after the plain runs exited 0) the ncu launch list of one
# full factorization (device times; cold-cache, serialised: compare SHARES) and one full capture
# of the Schur kernel.
set -x
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err || exit 1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_c3_ref.json 2> gpurun_out/bench_c3_ref.err
NL=$(timeout 300 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['n_launches'])")
echo "launches per factorization: $NL"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s $NL -c $NL --csv --log-file gpurun_out/launches_c3.csv python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 2 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:schur_ws -s 40 -c 1 -o gpurun_out/prof_schur_c3 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 > gpurun_out/ncu_s.log 2>&1
ls -la gpurun_out | tail
