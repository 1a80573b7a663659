#!/bin/bash
# ncu full captures of the tuned Jacobi configurations (development aid)
D=gpurun_out/${OUT:-pj}
mkdir -p $D
P='python tools/profile_one.py'
ncu --set full --clock-control none --import-source on -k regex:jacobi2d_tma -s 3 -c 1 -o $D/jacobi2d -f \
    $P jacobi2d '{"T": 4, "N": 16386, "s": 16, "B0": 8, "B1": 32}' 1 > $D/jacobi2d.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi1d_tma -s 3 -c 1 -o $D/jacobi1d -f \
    $P jacobi '{"T": 4, "N": 268435458, "s": 8, "B": 256}' 1 > $D/jacobi1d.log 2>&1
