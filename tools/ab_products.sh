#!/bin/bash
# tools/ab_products.sh N ROUNDS VARIANT... -- alternate the in-tree library and
# each tools/_bin/VARIANT build over ROUNDS rounds of tools/profile_products.py
# (m = 65536, r = 64, n = N); prints one line per run.
N=${1:-65536}; R=${2:-3}; shift 2
for i in $(seq "$R"); do
  echo -n "base  "; python tools/profile_products.py --n "$N" --reps 5
  for v in "$@"; do
    echo -n "$v  "; MLNMF_B200_LIB=tools/_bin/$v/libmlnmf_b200.so python tools/profile_products.py --n "$N" --reps 5
  done
done
