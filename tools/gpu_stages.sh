#!/bin/bash
# TMA ring depth sweep for the Jacobi pipelines (development aid)
timeout 900 python -m pytest tests -m gpu -x -q -k "jacobi" 2>&1 | tail -5
for S in ${STAGES:-0 2 3 4}; do
  echo "== PK_TMA_STAGES=$S"
  PK_TMA_STAGES=$S timeout 600 python tools/quick_bench.py jacobi jacobi2d 2>&1 | grep -v "^machine\|^total"
done
