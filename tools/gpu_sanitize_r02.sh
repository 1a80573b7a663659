#!/bin/bash
# Round-2 compute-sanitizer passes over the code added this round: the 8-byte
# word kernels, binary64 / int64 arithmetic, the run_block kernels, the
# vectorised addition, the packed float32 mat-vec, the pageable staging path
# of pk_run_host_io, the coherent peer loads and the concurrent multi-stream
# sweeps.
D=gpurun_out/san2
mkdir -p $D
run() {  # name tool args...
  local name=$1 tool=$2; shift 2
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 "$@" > $D/$name.log 2>&1
  echo "$name rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $D/$name.log | tail -2 | tr '\n' ' ')"
}
run values_memcheck memcheck python -m pytest tests/test_gpu_values.py -q -x
run parity_memcheck memcheck python -m pytest tests/test_gpu_parity.py -q -x -k "not full_size"
run runblock_memcheck memcheck python -m pytest tests/test_gpu_run_block.py -q -x
run fuzz_memcheck memcheck python -m pytest tests/test_gpu_fuzz.py -q -x
run multi_memcheck memcheck --target-processes all python -m pytest tests/test_gpu_peer.py tests/test_gpu_partition.py -q -x -k "peer or launch_multi"
run values_racecheck racecheck --racecheck-report hazard python -m pytest tests/test_gpu_values.py -q -x -k "f64 or block"
run values_synccheck synccheck python -m pytest tests/test_gpu_values.py -q -x -k "f64 or block"
