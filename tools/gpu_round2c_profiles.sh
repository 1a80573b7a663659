#!/bin/bash
# Round-2c evidence after the b-pair-major FFMA2 order and the Big1P tile:
# launch list of the bench command + one ncu --set full capture per FP32
# matmul leaf the tuners pick (numbers under ncu are evidence, never bench values).
D=gpurun_out/${OUT:-r02eprof}
mkdir -p $D
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file $D/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-tune > $D/bench_under_ncu.log 2>&1
echo "launch list rc=$?"
P='python tools/profile_one.py'
cap() {  # name regex skip args...
  local name=$1 re=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o $D/$name -f \
      $P "$@" > $D/$name.log 2>&1
  echo "$name rc=$?"
}
cap matmul_n8192 k_matmul_tma_sched 1 matmul '{"n": 8192, "B0": 128, "ub1": 8, "s": 16}' 3
cap matmul_n8192_t64 k_matmul_tma_sched 1 matmul '{"n": 8192, "B0": 128, "ub1": 8, "s": 8}' 3
cap matmul_n2048 k_matmul_tma_sched 1 matmul '{"n": 2048, "B0": 128, "ub1": 8, "s": 16}' 3
cap matmul_n2048_t64 k_matmul_tma_sched 1 matmul '{"n": 2048, "B0": 128, "ub1": 8, "s": 8}' 3
ls -la $D
