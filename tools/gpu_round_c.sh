#!/bin/bash
mkdir -p gpurun_out/d
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or every_leaf" > gpurun_out/d/memcheck.log 2>&1; echo "memcheck rc=$?"
tail -5 gpurun_out/d/memcheck.log
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python tools/quick_bench.py jacobi jacobi2d matvec 2>&1 | tail -12
P='python tools/profile_one.py'
ncu --set full --clock-control none --import-source on -k regex:jacobi1d_tma -s 3 -c 1 -o gpurun_out/d/jacobi1d -f \
    $P jacobi '{"T": 4, "N": 268435458, "s": 16, "B": 256}' 1 > gpurun_out/d/jacobi1d.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi2d_tma -s 3 -c 1 -o gpurun_out/d/jacobi2d -f \
    $P jacobi2d '{"T": 4, "N": 16386, "s": 4, "B0": 8, "B1": 32}' 1 > gpurun_out/d/jacobi2d.log 2>&1
