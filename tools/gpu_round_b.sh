#!/bin/bash
mkdir -p gpurun_out/b
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python tools/quick_bench.py jacobi jacobi2d matvec 2>&1 | tail -12
P='python tools/profile_one.py'
ncu --set full --clock-control none --import-source on -k regex:jacobi1d -s 3 -c 1 -o gpurun_out/b/jacobi1d -f \
    $P jacobi '{"T": 4, "N": 268435458, "s": 16, "B": 256}' 1 > gpurun_out/b/jacobi1d.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi2d -s 3 -c 1 -o gpurun_out/b/jacobi2d -f \
    $P jacobi2d '{"T": 4, "N": 16386, "s": 4, "B0": 8, "B1": 32}' 1 > gpurun_out/b/jacobi2d.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:matvec -s 1 -c 1 -o gpurun_out/b/matvec -f \
    $P matvec '{"N": 32768, "s": 1, "B": 128}' 2 > gpurun_out/b/matvec.log 2>&1
