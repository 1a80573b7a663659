#!/bin/bash
# Round-2 evidence (names = the keys bench.py reads from profiles/ncu_traffic.json): launch list of the bench command + one ncu --set full
# capture per measured kernel (numbers under ncu are evidence, never bench values).
D=gpurun_out/${OUT:-r02fprof}
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
cap matmul_n8192_t64 k_matmul_tma_sched 1 matmul '{"n": 8192, "B0": 128, "ub1": 8, "s": 8}' 3
cap matmul_n2048 k_matmul_tma_sched 1 matmul '{"n": 2048, "B0": 128, "ub1": 8, "s": 16}' 3
cap tf32x3_n8192 k_tf32x3 1 matmul '{"n": 8192, "B0": 128, "ub1": 8, "s": 16}' 3 --tf32x3
cap jacobi1d_2p28 k_jacobi1d_reg 3 jacobi '{"T": 4, "N": 268435458, "s": 16, "B": 256}' 1
cap jacobi2d_16384 k_jacobi2d_reg 3 jacobi2d '{"T": 4, "N": 16386, "s": 32, "B0": 64, "B1": 4}' 1
cap jacobi1d_tma_2p28 k_jacobi1d_tma 3 jacobi '{"T": 4, "N": 268435458, "s": 16, "B": 256}' 1 --generic
cap jacobi2d_tma_16384 k_jacobi2d_tma 3 jacobi2d '{"T": 4, "N": 16386, "s": 32, "B0": 64, "B1": 4}' 1 --generic
cap jacobi2d_temporal_h7 k_jacobi2d_wavefront 0 jacobi2d '{"T": 8, "N": 16386, "s": 32, "B0": 64, "B1": 4}' 1 --temporal=7
cap reverse_2p30 k_reverse 1 reverse '{"N": 1073741824, "s": 16, "B": 256}' 3
cap transpose_32768 k_transpose 1 transpose '{"N": 32768, "s": 8, "B0": 64, "B1": 8}' 3
cap matvec_32768 k_matvec 1 matvec '{"N": 32768, "s": 1, "B": 512}' 3
cap matvec_f32_32768 k_matvec 1 matvec '{"N": 32768, "s": 1, "B": 512}' 3 --f32
cap addition_16384 k_addition_vec 1 addition '{"N": 16384, "B0": 8, "B1": 128}' 3
cap jacobi1d_temporal_h15 k_jacobi1d_rtemporal 0 jacobi '{"T": 16, "N": 268435458, "s": 16, "B": 256}' 1 --temporal=15
cap matmul_f64_n2048 k_matmul_exact_tiled 1 matmul '{"n": 2048, "B0": 32, "ub1": 8, "s": 4}' 3 --f64
cap matvec_f64_32768 k_matvec_exact 1 matvec '{"N": 32768, "s": 1, "B": 512}' 3 --f64
cap reverse_f64_2p29 k_reverse 1 reverse '{"N": 536870912, "s": 16, "B": 256}' 3 --f64
ls -la $D
