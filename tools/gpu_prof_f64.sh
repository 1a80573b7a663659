D=gpurun_out/r02prof; mkdir -p $D
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_matmul_exact_tiled -s 1 -c 1 -o $D/matmul_f64 -f python tools/profile_one.py matmul '{"n": 2048, "B0": 32, "ub1": 8, "s": 4}' 3 --f64 > $D/matmul_f64.log 2>&1; echo rc=$?
