"""The N > 1 bench path end to end on the one GPU the box has: 2 ranks
mapped onto device 0 over gloo (PK_BENCH_ONE_GPU=1; NCCL refuses two ranks on
one device), launched the way the driver launches the scaling run
(torch.distributed.run, 127.0.0.1).  Exercises the row-shard headline with
its per-rank parity check, max-over-ranks timing, every family through the
partitioner with per-rank parity, the NCCL-style ghost-zone exchange (staged
through host copies under gloo) and the fused peer sweeps through CUDA IPC.
Numbers are meaningless (two processes time-slice one GPU); the run must end
rc = 0 with one JSON line whose parity verdicts are all ok."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_bench_line(cuda):
    env = dict(os.environ, PK_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(REPO, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-tune"]
    out = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["parity"].startswith("within")
    verdicts = {k: v[4] for k, v in d["summary"].items() if k != "cols" and v[4] is not None}
    assert verdicts and all(v == "ok" for v in verdicts.values()), verdicts
    assert "communicator ranks 2" in out.stderr
