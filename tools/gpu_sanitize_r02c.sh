#!/bin/bash
# compute-sanitizer over the code changed late in round 2: the FP32 matmul
# tiles (b-pair-major FFMA2, Big1P with its producer warp, the ROWA tiles)
# and the generic path for programs outside the seven families (NVRTC).
D=gpurun_out/san2c
mkdir -p $D
run() {  # name tool args...
  local name=$1 tool=$2; shift 2
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 "$@" > $D/$name.log 2>&1
  echo "$name rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $D/$name.log | tail -2 | tr '\n' ' ')"
}
run mm_memcheck memcheck python -m pytest tests/test_gpu_parity.py -q -x -k "tile_options or mid_tile or matmul_split or tuned_and_generic or integer_valued_fp32"
run mm_racecheck racecheck --racecheck-report hazard python -m pytest tests/test_gpu_parity.py -q -x -k "tile_options and 2048"
run mm_synccheck synccheck python -m pytest tests/test_gpu_parity.py -q -x -k "tile_options and 2048"
run generic_memcheck memcheck python -m pytest tests/test_gpu_generic.py -q -x
