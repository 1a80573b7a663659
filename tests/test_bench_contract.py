"""bench.py's reference arm on CPU: the oracle port timed on the host cores,
one JSON line with the driver's contract keys (the GPU arm is exercised by
tools/gpu_check.sh on a B200)."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*extra, env=None):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", *extra],
                         cwd=REPO, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    return [ln for ln in out.stdout.splitlines() if ln.strip()]


def test_reference_arm_prints_one_contract_line():
    lines = _run("--steps", "1", "--warmup", "0")
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    assert _run("--steps", "1", "--warmup", "0", "--gpus", "2", env=env) == []


def test_committed_ncu_traffic_covers_every_measured_kernel():
    """roofline.traffic and each family's traffic come from profiles/ncu_traffic.json
    under the keys bench.py looks up (a renamed capture would silently drop them)."""
    sys.path.insert(0, REPO)
    import bench

    with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as fh:
        recs = json.load(fh)
    for fam, key in bench.TRAFFIC_KEYS.items():
        assert key in recs, (fam, key)
    for n in (2048, 8192):
        for s in (8, 16):
            key = bench.matmul_traffic_key(n, {"B0": 128, "ub1": 8, "s": s})
            assert key in recs, key
    assert bench.matmul_traffic_key(1024, {"B0": 128, "ub1": 8, "s": 16}) is None
    for rec in recs.values():
        assert rec["dram_bytes"] > 0 and rec["kernel"] and rec["round"]
