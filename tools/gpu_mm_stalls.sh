#!/bin/bash
# matmul stall captures (development aid): full ncu sets with source for n = 8192 and n = 2048
D=gpurun_out/${OUT:-mmstall}
mkdir -p $D
for n in 8192 2048; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_matmul_tma -c 1 -s 1 -f \
      -o $D/mm$n python tools/profile_one.py matmul "{\"n\": $n, \"B0\": 128, \"ub1\": 8, \"s\": 16}" 2 > $D/mm$n.log 2>&1
  echo "ncu $n rc=$?"
done
