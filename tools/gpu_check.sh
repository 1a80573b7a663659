#!/bin/bash
# tests + bench + launch list (development aid)
D=gpurun_out/${OUT:-check}
mkdir -p $D
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
python bench.py > $D/bench.json 2> $D/bench.err; echo "bench rc=$?"
if [ -n "$LAUNCHES" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file $D/launches.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu --no-tune > $D/bench_under_ncu.log 2>&1
  echo "launch list rc=$?"
fi
