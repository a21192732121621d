for v in "$@"; do
  echo "== $v"
  RCP_B200_LIB=paper_1710_00125_b200/librcp_$v.so timeout 300 python tools/profile_factor.py --n 32768 --b 128 --p 144 --reps 1 | cut -c1-120
done
