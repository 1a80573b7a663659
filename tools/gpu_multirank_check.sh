#!/bin/bash
# The N > 1 bench path on a one-GPU box: 2 ranks mapped onto device 0 over gloo
# (PK_BENCH_ONE_GPU=1; NCCL refuses two ranks on one device).  Exercises the
# row-shard headline, max-over-ranks timing, the partitioner's NCCL-style
# ghost-zone exchange (staged through host copies under gloo) and the fused
# peer sweeps through CUDA IPC.  Numbers are meaningless (two processes
# time-slice one GPU); the run must end rc=0 with one JSON line.
D=gpurun_out/${OUT:-multirank}
mkdir -p $D
PK_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 3 --warmup 3 \
    > $D/bench2.json 2> $D/bench2.err
echo "2-rank bench rc=$?"
