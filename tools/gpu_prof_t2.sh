#!/bin/bash
D=gpurun_out/pt2
mkdir -p $D
ncu --set full --clock-control none --import-source on -k regex:k_jacobi2d_temporal -s 1 -c 1 -o $D/t2 -f \
    python tools/profile_one.py jacobi2d '{"T": 8, "N": 16386, "s": 16, "B0": 8, "B1": 32}' 1 --temporal=3 > $D/t2.log 2>&1
echo rc=$?
