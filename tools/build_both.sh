# build the product library and the per-phase profile variant in parallel
cd "$(dirname "$0")/.."
python -m paper_1710_00125_b200.build --force > /tmp/build_main.log 2>&1 &
nvcc -shared -Xcompiler -fPIC -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -DRCP_PANEL_PROF=1 \
  -o paper_1710_00125_b200/librcp_prof.so paper_1710_00125_b200/csrc/*.cu > /tmp/build_prof.log 2>&1
wait
tail -n 2 /tmp/build_main.log; tail -n 2 /tmp/build_prof.log
