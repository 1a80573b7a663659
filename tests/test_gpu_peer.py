"""Fused sweep + halo exchange over peer memory (pk_jacobi_sweep_peer,
partition.PeerStencil): 2 and 3 processes, each a rank with the whole
double buffer, exchanging ghost units through CUDA IPC mappings and device
counters.  The box has one GPU, so every rank maps the same device (the
kernels of the processes time-slice; the ordering protocol is the one
NVLink peers use).  The assembled result (each rank's own units, both
halves) must equal the CPU oracle bit for bit."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = {
    "jacobi": {"T": 7, "N": 20002, "s": 4, "B": 64},
    "jacobi2d": {"T": 5, "N": 130, "s": 2, "B0": 8, "B1": 16},
}


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, family, params, narrow, init_path, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1801_04348_b200 import _lib, binding, cases, partition, programs

    kind = programs.original(family)
    sel = cases.select(kind, params)
    L = binding.make_launch(kind, params, sel.applied, _lib.DTYPE_I32)
    if narrow:
        L.flags |= _lib.FLAG_NARROW
    a = torch.from_numpy(np.load(init_path)).cuda()
    ps = partition.PeerStencil(family, params, a, L)
    ps.run(params["T"])
    ps.close()
    np.savez(out_path % rank, a=a.cpu().numpy(), lo=ps.lo, hi=ps.hi)
    dist.destroy_process_group()


def _run(tmp_path, family, params, world, narrow, lim):
    import torch.multiprocessing as mp

    rng = np.random.default_rng(world * 7 + len(family))
    N = params["N"]
    n = 2 * N if family == "jacobi" else 2 * N * N
    init = rng.integers(-lim, lim, size=n, dtype=np.int64).astype(np.int32)
    init_path = str(tmp_path / "init.npy")
    np.save(init_path, init)
    out_path = str(tmp_path / "out_%d.npz")
    ctx = mp.get_context("spawn")
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, family, params, narrow, init_path, out_path))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    got = None
    row = 1 if family == "jacobi" else N
    half = N * row
    for r in range(world):
        z = np.load(out_path % r)
        if got is None:
            got = z["a"].copy()
        lo, hi = int(z["lo"]), int(z["hi"])
        for h in (0, half):
            got[h + lo * row:h + hi * row] = z["a"][h + lo * row:h + hi * row]
    return init, got


@pytest.mark.parametrize("family", sorted(CASES))
@pytest.mark.parametrize("world", [2, 3])
def test_peer_stencil_matches_oracle(cuda, oracle_mod, tmp_path, family, world):
    params = CASES[family]
    init, got = _run(tmp_path, family, params, world, True, 1 << 20)
    want = oracle_mod.run(family, params, {"a": init if family == "jacobi" else init.reshape(2 * params["N"], -1)})
    assert np.array_equal(got.reshape(-1), np.asarray(want["a"]).reshape(-1))


def test_peer_stencil_wide_values(cuda, oracle_mod, tmp_path):
    """Full-range int32: 64-bit sums inside the fused sweep."""
    params = CASES["jacobi2d"]
    init, got = _run(tmp_path, "jacobi2d", params, 2, False, 2**31 - 1)
    want = oracle_mod.run("jacobi2d", params, {"a": init.reshape(2 * params["N"], -1)})
    assert np.array_equal(got.reshape(-1), np.asarray(want["a"]).reshape(-1))


@pytest.mark.parametrize("family,params", [
    ("jacobi", {"T": 600, "N": 20002, "s": 4, "B": 64}),
    ("jacobi2d", {"T": 500, "N": 130, "s": 2, "B0": 8, "B1": 16}),
])
def test_peer_stencil_long_runs(cuda, oracle_mod, tmp_path, family, params):
    """PeerStencil for hundreds of steps (2 processes): the counters keep the
    edge blocks in step through T >= 500 exchanges."""
    init, got = _run(tmp_path, family, params, 2, True, 1 << 20)
    want = oracle_mod.run(family, params, {"a": init if family == "jacobi" else init.reshape(2 * params["N"], -1)})
    assert np.array_equal(got.reshape(-1), np.asarray(want["a"]).reshape(-1))
