#!/bin/bash
# bench + reference arm + ncu launch list + full captures of each family's kernel
set -x
mkdir -p gpurun_out/ncu
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ncu/launches_bench.log 2>&1
P='python tools/profile_one.py'
ncu --set full --clock-control none --import-source on -k regex:matmul_tiled -s 1 -c 1 -o gpurun_out/ncu/matmul8192 -f \
    $P matmul '{"n": 8192, "B0": 64, "ub1": 8, "s": 16}' 2 > gpurun_out/ncu/matmul.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:reverse -s 1 -c 1 -o gpurun_out/ncu/reverse -f \
    $P reverse '{"N": 1073741824, "s": 16, "B": 256}' 2 > gpurun_out/ncu/reverse.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:transpose -s 1 -c 1 -o gpurun_out/ncu/transpose -f \
    $P transpose '{"N": 32768, "s": 8, "B0": 64, "B1": 8}' 2 > gpurun_out/ncu/transpose.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi1d -s 3 -c 1 -o gpurun_out/ncu/jacobi1d -f \
    $P jacobi '{"T": 4, "N": 268435458, "s": 16, "B": 256}' 1 > gpurun_out/ncu/jacobi1d.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi2d -s 3 -c 1 -o gpurun_out/ncu/jacobi2d -f \
    $P jacobi2d '{"T": 4, "N": 16386, "s": 4, "B0": 8, "B1": 32}' 1 > gpurun_out/ncu/jacobi2d.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:matvec -s 1 -c 1 -o gpurun_out/ncu/matvec -f \
    $P matvec '{"N": 32768, "s": 1, "B": 128}' 2 > gpurun_out/ncu/matvec.log 2>&1
ls -la gpurun_out/ncu
