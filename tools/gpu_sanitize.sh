#!/bin/bash
# compute-sanitizer passes over the GPU parity tests (development aid)
D=gpurun_out/san
mkdir -p $D
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py -x -q > $D/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 $D/memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "jacobi" > $D/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -4 $D/racecheck.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "jacobi or matmul" > $D/synccheck.log 2>&1; echo "synccheck rc=$?"; tail -4 $D/synccheck.log
